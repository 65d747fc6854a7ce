cd $GRAFT_REPO_ROOT
# relu(x) + avgpool2(x) from one read of x for R38 blocks: bit-identical losses expected (d 1.4008493423461914,
# g 1.3385354280471802 at the default bench), throughput, then the step / boundary / full-size tests
for i in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d46_bench_$i.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d46_bench_$i.log').read().strip().splitlines()[-1]);print('fused', round(d['value'],1), d['losses']['d'], d['losses']['g'], d['gpu_launches'])" || tail -5 gpurun_out/d46_bench_$i.log
done
timeout 1800 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_boundary.py -q -x 2>&1 | tail -3
