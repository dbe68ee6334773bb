#!/bin/bash
# A/B of library variants (variants/libcvx_<v>.so) with optional env: tools/ab_libs.sh v1[:K=V,..] v2 ...
cd "$(dirname "$0")/.."
cp paper_2410_21149_b200/libcvx.so /tmp/libcvx_orig.so
for r in 1 2; do for spec in "$@"; do
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=${spec#*:}
  cp variants/libcvx_$v.so paper_2410_21149_b200/libcvx.so
  env ${envs//,/ } python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step_serial']
print('$spec', round(d['ms_per_step'],3), {a: round(k[a],3) for a in ('ray_prepare','block_walk_allocate','ray_walk_update','esdf_pass_x','esdf_pass_y','esdf_pass_z') if a in k})"
done; done
cp /tmp/libcvx_orig.so paper_2410_21149_b200/libcvx.so
