cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "out_conv_split or thin" > gpurun_out/d20_ops.log 2>&1; tail -2 gpurun_out/d20_ops.log
timeout 300 python -m pytest tests/test_gpu_guard.py -q -k "out_conv or thin" >> gpurun_out/d20_ops.log 2>&1; tail -1 gpurun_out/d20_ops.log
timeout 300 python tools/check_outconv.py > gpurun_out/d20_check.log 2>&1; cat gpurun_out/d20_check.log
timeout 300 python tools/bench_thin.py 10 > gpurun_out/d20_thin.log 2>&1; cat gpurun_out/d20_thin.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/d20_ncu_thin.csv python tools/bench_thin.py 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/d20_ncu_thin.csv --iters 1 > gpurun_out/d20_ncu_thin.md 2>&1; head -20 gpurun_out/d20_ncu_thin.md
timeout 1500 python -m pytest tests/test_gpu_step.py -q > gpurun_out/d20_step.log 2>&1; tail -3 gpurun_out/d20_step.log
for v in 0 1 0 1; do
  PARAGAN_THIN_TC=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d20_bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d20_bench_$v.log').read().strip().splitlines()[-1]);print('thin_tc=$v', round(d['value'],1), d['roofline']['other_kernels_ms_per_step'])" >> gpurun_out/d20_summary.txt
done
cat gpurun_out/d20_summary.txt
