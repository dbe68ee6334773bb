#!/bin/bash
# A/B of env knobs on the default bench (interleaved): tools/ab_knobs.sh "K=V,K2=V2" "K=V" ...
cd "$(dirname "$0")/.."
for r in 1 2; do for spec in "$@"; do
  env ${spec//,/ } python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step_serial']
print('$spec', round(d['ms_per_step'],3), {a: round(k[a],3) for a in ('ray_prepare','block_walk_allocate','ray_walk_update','esdf_pass_y')})"
done; done
