cd $GRAFT_REPO_ROOT
timeout 300 python tools/bench_conv.py 2>&1 | tail -10
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_guard.py -q -x 2>&1 | tail -2
