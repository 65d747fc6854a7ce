cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_ops.py tests/test_gpu_attn.py tests/test_gpu_boundary.py tests/test_gpu_optim.py tests/test_gpu_async.py -q -x > gpurun_out/d4_tests.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_step.py -q -s -k "micro or sndcgan or reproducible or f32_biggan or order or nonfinite or replicas" > gpurun_out/d4_step.log 2>&1
timeout 300 python tools/parity_report.py --bf16 --batch 8 --summary > gpurun_out/d4_micro_sub.log 2>&1
PARAGAN_SUBPIXEL=0 timeout 300 python tools/parity_report.py --bf16 --batch 8 --summary > gpurun_out/d4_micro_nosub.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/d4_bench.log 2>&1
echo done
