#!/bin/bash
# A/B of library variants on configs[1] (device + e2e) and the MAV workload: tools/ab_libs_all.sh v1 v2 ...
cd "$(dirname "$0")/.."
cp paper_2410_21149_b200/libcvx.so /tmp/libcvx_orig.so
for r in 1 2; do for v in "$@"; do
  cp variants/libcvx_$v.so paper_2410_21149_b200/libcvx.so
  a=$(CVX_NO_BUILD=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'walk', round(d['kernel_ms_per_step']['ray_walk_update'],3))")
  b=$(CVX_NO_BUILD=1 python bench.py --workload mav --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2))")
  echo "$v lidar $a mav $b"
done; done
cp /tmp/libcvx_orig.so paper_2410_21149_b200/libcvx.so
