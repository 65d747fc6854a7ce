cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/d5_smi.txt
timeout 900 python -m pytest tests/test_gpu_async.py tests/test_gpu_checkpoint.py tests/test_gpu_optim.py tests/test_gpu_boundary.py -q -s > gpurun_out/d5_async_ck.log 2>&1
timeout 900 python -m pytest tests/test_gpu_step.py -q -s -k "bf16_micro" > gpurun_out/d5_micro.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d5_smoke.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -s > gpurun_out/d5_dist.log 2>&1
echo done
