cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "pool" 2>&1 | tail -2
for v in 0 1 0 1; do
  PARAGAN_POOL_FUSE=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d38_bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d38_bench_$v.log').read().strip().splitlines()[-1]);print('pool=$v', round(d['value'],1), d['losses']['d'], d['losses']['g'])"
done
timeout 1500 python -m pytest tests/test_gpu_step.py tests/test_gpu_ops.py tests/test_gpu_guard.py -q -x 2>&1 | tail -1
