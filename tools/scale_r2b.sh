# 4-GPU measurements with the final round-2 code (third pass) (gpurun --gpus 4 -- bash tools/scale_r2b.sh): weak scaling with
# the CUDA-graph step cache (default) and with the overlapped all-reduce instead, config 3 literal, configs 4/5,
# the asynchronous scheme, the 2-GPU tests.  Lines land in gpurun_out/s7_*.log
cd $GRAFT_REPO_ROOT
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$np --master-addr=127.0.0.1 \
      --master-port=$((29600 + RANDOM % 300)) bench.py --gpus $np "$@" > gpurun_out/s7_$name.log 2>&1
  echo "$name rc=$?"
}
nvidia-smi -L > gpurun_out/s7_smi.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s7_n1.log 2>&1
run n4 4 --steps 10 --warmup 3
PARAGAN_OVERLAP=1 run n4_ov 4 --steps 10 --warmup 3 --no-e2e
run n2 2 --steps 10 --warmup 3 --no-e2e
run c3lit 4 --steps 5 --warmup 3 --batch 512 --no-e2e
run c4 4 --steps 5 --warmup 3 --res 256 --batch 128 --d-steps 2 --no-e2e
run c5 4 --steps 5 --warmup 3 --res 512 --batch 32 --no-e2e
run async 4 --steps 10 --warmup 3 --async
timeout 600 python bench.py --steps 5 --warmup 3 --res 256 --batch 128 --d-steps 2 --no-e2e --no-cpu-baseline > gpurun_out/s7_c4_n1.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --res 512 --batch 32 --no-e2e --no-cpu-baseline > gpurun_out/s7_c5_n1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/s7_dist_tests.log 2>&1; tail -1 gpurun_out/s7_dist_tests.log
for f in gpurun_out/s7_*.log; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('n_gpus'), round(d['value'],1), d['config'].get('global_batch'), d['config'].get('workload','')[:40], (d.get('e2e') or {}).get('value'))
except Exception as e: print('$f', 'no line', e)
"; done
