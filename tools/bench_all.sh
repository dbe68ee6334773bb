#!/bin/bash
# All bench workloads + the N=2 one-GPU (gloo) path on one box: tools/bench_all.sh <tag>
T=${1:-r2}; mkdir -p gpurun_out/$T
run() { local name=$1; shift; timeout 900 "$@" > gpurun_out/$T/$name.json 2> gpurun_out/$T/$name.err; echo "$name rc=$?"; }
run bench python bench.py
run bench_esdf_stress python bench.py --workload esdf_stress --steps 5
run bench_mav python bench.py --workload mav --steps 2 --warmup 1
run bench_incremental python bench.py --workload incremental --steps 5
run bench_reference python bench.py --impl reference --steps 2 --warmup 1
CVX_BENCH_ONE_GPU=1 CVX_BENCH_BACKEND=gloo run bench_n2_onegpu_gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline
CVX_BENCH_ONE_GPU=1 CVX_BENCH_BACKEND=gloo run bench_mav_n2_onegpu_gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --workload mav --gpus 2 --steps 1 --warmup 1
for w in $EXTRA; do run bench_$w python bench.py --workload $w --steps 5; done
