cd "$(dirname "$0")/.."
for r in 1 2; do for o in 1 0; do
CVX_BENCH_ORDER=$o python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('order=$o', round(d['ms_per_step'],3), round(d['one_submap_in_flight']['ms_per_step'],3))"
done; done
