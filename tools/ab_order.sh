cd "$(dirname "$0")/.."
for r in 1 2; do for spec in "1 1" "0 1" "0 0"; do set -- $spec
CVX_BENCH_ORDER=$1 CVX_WALK_ORDER=$2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench_order=$1 walk_order=$2', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'one', round(d['one_submap_in_flight']['ms_per_step'],3))"
done; done
