cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_boundary.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/d33_n1.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/d33_n1.log').read().strip().splitlines()[-1]);print('n1', round(d['value'],1), d['e2e'], d['losses']['d_per_step_e2e'][:4])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29651 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/d33_n4.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/d33_n4.log').read().strip().splitlines()[-1]);print('n4', round(d['value'],1), d['e2e'])"
