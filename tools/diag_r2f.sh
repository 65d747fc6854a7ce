cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d6_smoke.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_step.py -q -s -k "f32_biggan or isolated or micro" > gpurun_out/d6_step.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -s > gpurun_out/d6_dist.log 2>&1
echo done
