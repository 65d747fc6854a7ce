cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py -q -k "out_conv_split or thin" > gpurun_out/d19_ops.log 2>&1; tail -2 gpurun_out/d19_ops.log
timeout 300 python -m pytest tests/test_gpu_guard.py -q -k "out_conv or thin" >> gpurun_out/d19_ops.log 2>&1; tail -1 gpurun_out/d19_ops.log
timeout 300 python tools/check_outconv.py > gpurun_out/d19_check.log 2>&1; cat gpurun_out/d19_check.log
timeout 300 python tools/bench_thin.py 10 > gpurun_out/d19_thin.log 2>&1; cat gpurun_out/d19_thin.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/d19_ncu_thin.csv python tools/bench_thin.py 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/d19_ncu_thin.csv --iters 1 > gpurun_out/d19_ncu_thin.md 2>&1; head -20 gpurun_out/d19_ncu_thin.md
