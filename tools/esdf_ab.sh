cd $GRAFT_REPO_ROOT
for k in 0 1; do
  CVX_EDT_KERNEL=$k python bench.py --workload esdf_stress --steps 3 --warmup 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stress k=$k', d['ms_per_step'], d['kernel_ms_per_step'])"
  CVX_EDT_KERNEL=$k python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step_serial']; print('lidar k=$k', d['ms_per_step'], {a:round(k[a],3) for a in k if 'esdf' in a})"
done
CVX_EDT_KERNEL=0 python -m pytest tests/test_gpu_parity.py tests/test_gpu_esdf_incremental.py -x -q -m gpu -k "esdf or incremental" 2>&1 | tail -2
