#!/bin/bash
# A/B of library variants on the ESDF stress workload: tools/ab_stress.sh v1 v2 ...
cd "$(dirname "$0")/.."
cp paper_2410_21149_b200/libcvx.so /tmp/libcvx_orig.so
for v in "$@"; do
  cp variants/libcvx_$v.so paper_2410_21149_b200/libcvx.so
  python bench.py --workload esdf_stress --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2), {k: round(x,2) for k,x in d['kernel_ms_per_step'].items()})"
done
cp /tmp/libcvx_orig.so paper_2410_21149_b200/libcvx.so
