cd $GRAFT_REPO_ROOT
for v in 0 1 0 1; do
  PARAGAN_DGRAD_UP2=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d42_bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d42_bench_$v.log').read().strip().splitlines()[-1]);print('dgup2=$v', round(d['value'],1), round(d['roofline']['achieved_executed'],1), d['losses']['d'], d['losses']['g'], d['losses'].get('d_grad_norm_last'))"
done
timeout 1800 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_boundary.py tests/test_gpu_async.py -q -x 2>&1 | tail -3
