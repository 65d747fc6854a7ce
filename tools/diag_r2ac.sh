cd $GRAFT_REPO_ROOT
for v in 0 1 0 1; do
  PARAGAN_GRAPHS=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/d30_bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d30_bench_$v.log').read().strip().splitlines()[-1]);print('graphs=$v', round(d['value'],1), round(d['e2e']['value'],1), d['gpu_launches'], d['losses']['d'], d['losses']['g'], d['losses']['d_per_step_e2e'][:3])"
done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/d30_tests.log 2>&1; tail -3 gpurun_out/d30_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
