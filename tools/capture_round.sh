#!/bin/bash
# One GPU session of evidence for profiles/: default bench line, ncu launch list of our kernels, and one
# `ncu --set full` capture per hot kernel.  usage: tools/capture_round.sh <tag> [what...]
T=${1:-r1}; shift
mkdir -p gpurun_out/$T
cap() {  # <regex on the base function name> <name> <skip>
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s $3 -c 1 -o gpurun_out/$T/$2 \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/$T/$2.log 2>&1; echo "ncu $2 rc=$?"
}
capw() {  # <regex> <name> <skip> <workload>: as cap, on another bench workload
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s $3 -c 1 -o gpurun_out/$T/$2 \
    python bench.py --workload $4 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/$T/$2.log 2>&1; echo "ncu $2 rc=$?"
}
WHAT=${@:-bench launches walk block_walk prepare fold esdf_pass_x esdf_pass_y esdf_pass_z query}
for w in $WHAT; do case $w in
  bench) timeout 600 python bench.py > gpurun_out/$T/bench.json 2> gpurun_out/$T/bench.err; echo "bench rc=$?";;
  launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled \
      -k regex:_ZN3cvx --csv --log-file gpurun_out/$T/launches.csv python bench.py --steps 1 --warmup 1 \
      --no-cpu-baseline --no-e2e > gpurun_out/$T/launches_bench.json 2>&1; echo "launches rc=$?";;
  walk) cap "^walk_dw_kernel" walk 2;;   # one walk launch per configs[1] submap (dense window, R19)
  walk_cw) CVX_DENSE=0 cap "^walk_(cw_)?kernel" walk_cw 2;;
  dense_fold) cap "^dense_fold_kernel" dense_fold 2;;
  block_walk) cap "^block_walk[23]?_kernel" block_walk 2;;
  prepare) cap "^prepare_kernel" prepare 2;;
  fold) cap "^fold_kernel" fold 1;;
  esdf_pass_x) cap "^pass_x_kernel" esdf_pass_x 1;;
  esdf_pass_y) cap "^(link|pba|ring)_line_kernel" esdf_pass_y 2;;
  esdf_pass_z) cap "^(link|pba|ring)_line_kernel" esdf_pass_z 3;;
  query) cap "^query_kernel" query 0;;
  project) capw "^project_kernel" project 2 rgbd;;
  inc_window) capw "^inc_window" inc_window 3 incremental;;
  mav) timeout 900 python bench.py --workload mav --steps 3 --warmup 1 > gpurun_out/$T/bench_mav.json 2> gpurun_out/$T/bench_mav.err; echo "mav rc=$?";;
  reference) timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$T/bench_reference.json 2> gpurun_out/$T/bench_reference.err; echo "reference rc=$?";;
  color) timeout 900 python bench.py --workload color --steps 10 > gpurun_out/$T/bench_color.json 2> gpurun_out/$T/bench_color.err; echo "color rc=$?";;
  voxel_sweep) timeout 900 python bench.py --workload voxel_sweep --steps 5 > gpurun_out/$T/bench_voxel_sweep.json 2> gpurun_out/$T/bench_voxel_sweep.err; echo "voxel_sweep rc=$?";;
  n2) CVX_BENCH_ONE_GPU=1 CVX_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$T/bench_n2_onegpu_gloo.json 2> gpurun_out/$T/bench_n2_onegpu_gloo.err; echo "n2 rc=$?";;
  stress_x) capw "^pass_x_kernel" stress_pass_x 0 esdf_stress;;
  stress_y) capw "^(link|pba|ring)_line_kernel" stress_pass_y 0 esdf_stress;;
  stress_z) capw "^(link|pba|ring)_line_kernel" stress_pass_z 1 esdf_stress;;
  rgbd) timeout 900 python bench.py --workload rgbd --steps 5 > gpurun_out/$T/bench_rgbd.json 2> gpurun_out/$T/bench_rgbd.err; echo "rgbd rc=$?";;
  incremental) timeout 900 python bench.py --workload incremental --steps 5 > gpurun_out/$T/bench_incremental.json 2> gpurun_out/$T/bench_incremental.err; echo "incremental rc=$?";;
  gputest) timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/$T/gputest.log 2>&1; echo "gputest rc=$?";;
  stress) timeout 900 python bench.py --workload esdf_stress --steps 5 > gpurun_out/$T/bench_esdf_stress.json 2> gpurun_out/$T/bench_esdf_stress.err; echo "stress rc=$?";;
esac; done
