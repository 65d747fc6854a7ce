cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "out_conv_split or thin" > gpurun_out/d16_ops.log 2>&1; tail -2 gpurun_out/d16_ops.log
timeout 300 python tools/bench_thin.py 10 > gpurun_out/d16_thin.log 2>&1; cat gpurun_out/d16_thin.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d16_ncu_thin.csv python tools/bench_thin.py 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/d16_ncu_thin.csv --iters 1 > gpurun_out/d16_ncu_thin.md 2>&1; head -30 gpurun_out/d16_ncu_thin.md
for v in 0 1; do
PARAGAN_THIN_TC=$v PARAGAN_PROFILE_VERBOSE=1 PARAGAN_ALLOW_SHORT_WARMUP=1 timeout 600 python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/d16_layers_$v.err
grep "kind=6" gpurun_out/d16_layers_$v.err
done
