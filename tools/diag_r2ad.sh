cd $GRAFT_REPO_ROOT
run() {  # name env...
  local name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
      --master-port=$((29600 + RANDOM % 300)) bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e > gpurun_out/d31_$name.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d31_$name.log').read().strip().splitlines()[-1]);print('$name', round(d['value'],1), d['losses']['d'], d['losses']['g'], d.get('roofline',{}).get('collectives'))" 2>&1 | tail -1
}
run ov1_g0 PARAGAN_OVERLAP=1 PARAGAN_GRAPHS=0
run ov0_g2 PARAGAN_OVERLAP=0 PARAGAN_GRAPHS=2
run ov1_g0b PARAGAN_OVERLAP=1 PARAGAN_GRAPHS=0
run ov0_g2b PARAGAN_OVERLAP=0 PARAGAN_GRAPHS=2
run ov0_g0 PARAGAN_OVERLAP=0 PARAGAN_GRAPHS=0
PARAGAN_OVERLAP=0 PARAGAN_GRAPHS=2 timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -2
