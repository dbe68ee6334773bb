#!/bin/bash
# On the GPU box: time ray_walk_update (and the step) for each variants/libcvx_*.so given, R rounds interleaved.
cd "$(dirname "$0")/.."
R=${R:-2}
cp paper_2410_21149_b200/libcvx.so /tmp/libcvx_orig.so
for r in $(seq $R); do
  for v in "$@"; do
    cp variants/libcvx_$v.so paper_2410_21149_b200/libcvx.so
    touch paper_2410_21149_b200/libcvx.so
    out=$(CVX_NO_BUILD=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} 2>&1 | tail -1)
    KEYS="${KEYS}" python - "$v" "$out" <<'PY'
import json, sys
v, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    k = d.get("kernel_ms_per_step", {})
    import os, re
    keys = os.environ.get("KEYS", "ray_walk_update|block_walk_allocate|ray_prepare")
    ks = "  ".join(f"{n} {t:.3f}" for n, t in k.items() if re.search(keys, n))
    print(f"{v:10s} step {d['ms_per_step']:.3f} ms  {ks}", flush=True)
except Exception as e:
    print(v, "ERR", line[-300:])
PY
  done
done
cp /tmp/libcvx_orig.so paper_2410_21149_b200/libcvx.so
