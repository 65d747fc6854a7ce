cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_ops.py -q -x -k "attn or thin" > gpurun_out/d9_attn_thin.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_step.py -q -s -k "micro or bitwise or bf16_biggan128_subpixel" > gpurun_out/d9_step.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/d9_bench.log 2>&1
PARAGAN_PROFILE_VERBOSE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --repeats 1 > /dev/null 2> gpurun_out/d9_layers.err
echo done
