#!/bin/bash
# A/B of env knobs on the mav workload (kernel breakdown): tools/ab_mav.sh "K=V" "K=V,K2=V2" ...
cd "$(dirname "$0")/.."
for spec in "$@"; do
  env CVX_BENCH_MAV_PROFILE=1 ${spec//,/ } python bench.py --workload mav --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$spec', round(d['ms_per_step'],2), {k: round(x,2) for k,x in d.get('kernel_ms_per_step',{}).items()})"
done
