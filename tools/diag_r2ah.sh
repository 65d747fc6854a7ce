cd $GRAFT_REPO_ROOT
PARAGAN_RESB=0 timeout 300 python tools/bench_conv.py "96->96@128k3" 2>&1 | tail -1 | sed 's/^/resb0 /'
timeout 300 python tools/bench_conv.py "96->96@128k3" 2>&1 | tail -1 | sed 's/^/resb1 /'
PARAGAN_RESB=0 timeout 300 python tools/bench_conv.py "96->96@128k3" 2>&1 | tail -1 | sed 's/^/resb0 /'
timeout 300 python tools/bench_conv.py "96->96@128k3" 2>&1 | tail -1 | sed 's/^/resb1 /'
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
