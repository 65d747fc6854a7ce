# A12 overlap tuning at 4 GPUs: (G blocks capped, SMs left free) for D's all-reduce
cd $GRAFT_REPO_ROOT
for v in "0 0 0" "1 3 16" "1 5 16" "1 5 8" "1 2 32" "1 5 24"; do
  set -- $v
  PARAGAN_OVERLAP=$1 PARAGAN_OVERLAP_BLOCKS=$2 PARAGAN_OVERLAP_SMS=$3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 \
     --master-addr=127.0.0.1 --master-port=$((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-profile \
     > gpurun_out/ov_$1_$2_$3.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ov_$1_$2_$3.log').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), d['repeats_ms_per_step'])" >> gpurun_out/ov_summary.txt
done
echo done
