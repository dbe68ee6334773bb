#!/bin/bash
# On the GPU box: device and host-frame (e2e) step time per variants/libcvx_<name>.so, R rounds interleaved.
# usage: R=2 tools/ab_e2e.sh name1 name2 ...
cd "$(dirname "$0")/.."
R=${R:-2}
cp paper_2410_21149_b200/libcvx.so /tmp/libcvx_orig.so
for r in $(seq $R); do for v in "$@"; do
  cp variants/libcvx_$v.so paper_2410_21149_b200/libcvx.so; touch paper_2410_21149_b200/libcvx.so
  CVX_NO_BUILD=1 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3))"
done; done
cp /tmp/libcvx_orig.so paper_2410_21149_b200/libcvx.so
