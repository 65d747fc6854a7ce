# Final round-2 multi-GPU lines with R38 (gpurun --gpus 4 -- bash tools/scale_r2c.sh): 1 / 2 / 4 GPUs weak scaling
# with the CUDA-graph step cache (default), the 2-rank tests.  Lines land in gpurun_out/s8_*.log
cd $GRAFT_REPO_ROOT
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$np --master-addr=127.0.0.1 \
      --master-port=$((29600 + RANDOM % 300)) bench.py --gpus $np "$@" > gpurun_out/s8_$name.log 2>&1
  echo "$name rc=$?"
}
nvidia-smi -L > gpurun_out/s8_smi.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s8_n1.log 2>&1
run n2 2 --steps 10 --warmup 3
run n4 4 --steps 10 --warmup 3
timeout 900 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/s8_dist_tests.log 2>&1; tail -1 gpurun_out/s8_dist_tests.log
for f in gpurun_out/s8_*.log; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d.get('n_gpus'), round(d['value'],1), round(d['ms_per_step'],2), d['config'].get('global_batch'), (d.get('e2e') or {}).get('value'), d.get('clocks'))
except Exception as e: print('$f', 'no line', e)
"; done
