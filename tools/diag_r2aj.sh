cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_attn.py -q -x 2>&1 | tail -2
for v in 0 1 0 1; do
  PARAGAN_ATTN_FLAT=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d36_bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d36_bench_$v.log').read().strip().splitlines()[-1]);print('flat=$v', round(d['value'],1), d['roofline']['other_kernels_ms_per_step'], d['losses']['d'], d['losses']['g'])"
done
timeout 1200 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -1
