cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -s -x > gpurun_out/d7_dist.log 2>&1
echo dist_rc=$? >> gpurun_out/d7_dist.log
for ov in 1 0; do
PARAGAN_OVERLAP=$ov timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29511 bench.py --gpus 2 --steps 10 --warmup 3 --repeats 2 --no-e2e > gpurun_out/d7_bench2_ov$ov.log 2>&1
done
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d7_smoke.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_step.py -q -s -k "not b64" > gpurun_out/d7_step.log 2>&1
echo done
