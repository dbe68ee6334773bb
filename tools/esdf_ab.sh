#!/bin/bash
# A/B of the ESDF line-pass kernels (CVX_EDT_KERNEL: 0 = ring (default), 2 = link, 1 = band hulls) on
# configs[4] and configs[1]: tools/esdf_ab.sh [kernels...]
cd "$(dirname "$0")/.."
for k in ${@:-0 2}; do
  CVX_EDT_KERNEL=$k python bench.py --workload esdf_stress --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stress k=$k', round(d['ms_per_step'],2), {a: round(v,2) for a,v in d['kernel_ms_per_step'].items()})"
  CVX_EDT_KERNEL=$k python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step_serial']; print('lidar k=$k', round(d['ms_per_step'],3), {a:round(k[a],3) for a in k if 'esdf' in a})"
done
