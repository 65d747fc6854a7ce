cd $GRAFT_REPO_ROOT
timeout 300 python tools/bench_conv.py "k1" 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_guard.py tests/test_gpu_attn.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
