# 4-GPU measurements (gpurun --gpus 4 -- bash tools/scale_r2.sh): weak scaling, overlap on/off, config 3
# literal, configs 4 and 5, the asynchronous scheme.  Lines land in gpurun_out/s4_*.log
cd $GRAFT_REPO_ROOT
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$np --master-addr=127.0.0.1 \
      --master-port=$((29600 + RANDOM % 300)) bench.py --gpus $np "$@" > gpurun_out/s4_$name.log 2>&1
  echo "$name rc=$?"
}
nvidia-smi -L > gpurun_out/s4_smi.txt
run n4 4 --steps 10 --warmup 3
PARAGAN_OVERLAP=0 run n4_noov 4 --steps 10 --warmup 3 --no-e2e
run n2 2 --steps 10 --warmup 3 --no-e2e
run c3lit 4 --steps 5 --warmup 3 --batch 512 --no-e2e
run c4 4 --steps 5 --warmup 3 --res 256 --batch 128 --d-steps 2 --no-e2e
run c5 4 --steps 5 --warmup 3 --res 512 --batch 32 --no-e2e
run async 4 --steps 10 --warmup 3 --async
run async_g512 4 --steps 10 --warmup 3 --async --g-batch 512 --batch 256
timeout 600 python bench.py --steps 5 --warmup 3 --res 256 --batch 128 --d-steps 2 --no-e2e --no-cpu-baseline > gpurun_out/s4_c4_n1.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --res 512 --batch 32 --no-e2e --no-cpu-baseline > gpurun_out/s4_c5_n1.log 2>&1
echo done
