cd $GRAFT_REPO_ROOT
# R38 A/B (pooled D forward as a stride-2 phase conv) + the step / full-size / boundary tests
for v in 0 1 0 1; do
  PARAGAN_POOL_FWD=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d43_bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d43_bench_$v.log').read().strip().splitlines()[-1]);print('poolfwd=$v', round(d['value'],1), d['losses']['d'], d['losses']['g'], d['losses'].get('d_grad_norm_last'))" || tail -5 gpurun_out/d43_bench_$v.log
done
for v in 0 1; do
  PARAGAN_POOL_FWD=$v PARAGAN_PROFILE_VERBOSE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --repeats 1 > /dev/null 2> gpurun_out/d43_layers_$v.err
  python tools/prof_layers.py gpurun_out/d43_layers_$v.err 60 2 > gpurun_out/d43_layers_$v.md; grep -iE "pool|->192|->384|->768|->1536" gpurun_out/d43_layers_$v.md | head -24
done
timeout 1800 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_boundary.py tests/test_gpu_async.py -q -x 2>&1 | tail -8
