#!/bin/bash
# On the GPU box: one bench workload's value per variants/libcvx_<name>.so, R rounds interleaved.
# usage: W=incremental R=2 tools/ab_workload.sh name1 name2 ...
cd "$(dirname "$0")/.."
R=${R:-2}; W=${W:-lidar}
cp paper_2410_21149_b200/libcvx.so /tmp/libcvx_orig.so
for r in $(seq $R); do for v in "$@"; do
  cp variants/libcvx_$v.so paper_2410_21149_b200/libcvx.so; touch paper_2410_21149_b200/libcvx.so
  CVX_NO_BUILD=1 python bench.py --workload $W --steps 10 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['value'],4), d['unit'], {k: round(v,3) for k, v in (d.get('inc_kernel_ms_per_update') or {}).items()})"
done; done
cp /tmp/libcvx_orig.so paper_2410_21149_b200/libcvx.so
