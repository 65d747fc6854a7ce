# NCCL environment sweep for the 4-GPU step (gpurun --gpus 4 -- bash tools/nccl_sweep.sh)
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 4 --no-cpu-baseline --no-e2e > gpurun_out/ns_$name.log 2>&1
  echo "rc=$?" >> gpurun_out/ns_$name.log
}
run default NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING
run ring NCCL_ALGO=Ring
run nvls NCCL_ALGO=NVLS
run nonvls NCCL_NVLS_ENABLE=0
run ch32 NCCL_MIN_NCHANNELS=32
run ll128 NCCL_PROTO=LL128
