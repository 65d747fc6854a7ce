cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_guard.py -q > gpurun_out/d12_guard.log 2>&1
timeout 300 python tools/bench_thin.py 20 > gpurun_out/d12_thin.log 2>&1
echo done
