# thin output layer on the tensor cores (R36): op tests, guard, step parity, smoke, A/B bench
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "out_conv_split or thin" > gpurun_out/d15_ops.log 2>&1
timeout 300 python -m pytest tests/test_gpu_guard.py -q -k "out_conv or thin" >> gpurun_out/d15_ops.log 2>&1
tail -3 gpurun_out/d15_ops.log
timeout 1500 python -m pytest tests/test_gpu_step.py -q -x > gpurun_out/d15_step.log 2>&1
tail -3 gpurun_out/d15_step.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d15_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/d15_smoke.log
for v in 0 1 0 1; do
  PARAGAN_THIN_TC=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d15_bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d15_bench_$v.log').read().strip().splitlines()[-1]);print('thin_tc=$v', round(d['value'],1), d['roofline']['other_kernels_ms_per_step'], d['losses']['d'], d['losses']['g'])" >> gpurun_out/d15_summary.txt
done
cat gpurun_out/d15_summary.txt
