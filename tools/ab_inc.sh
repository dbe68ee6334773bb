#!/bin/bash
# A/B of library variants on the incremental workload: tools/ab_inc.sh v1 v2 ...
cd "$(dirname "$0")/.."
cp paper_2410_21149_b200/libcvx.so /tmp/libcvx_orig.so
for r in 1 2; do for v in "$@"; do
  cp variants/libcvx_$v.so paper_2410_21149_b200/libcvx.so
  python bench.py --workload incremental --steps 3 --warmup 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],3), round(d['exact_finalize_ms_per_update'],3), {k: round(x,3) for k,x in d['inc_kernel_ms_per_update'].items()})"
done; done
cp /tmp/libcvx_orig.so paper_2410_21149_b200/libcvx.so
