#!/bin/bash
# A/B of env settings on the configs[1] bench (2 interleaved rounds): tools/ab_env_bench.sh "ENV=a" "ENV=b" ...
cd "$(dirname "$0")/.."
for r in 1 2; do for spec in "$@"; do
  env ${spec//,/ } python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step_serial']
print('$spec', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3) if d.get('e2e') else None, {a: round(k[a],3) for a in k if k[a] > 0.02})"
done; done
