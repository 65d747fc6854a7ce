# Table 3 precision toggle re-run on one B200: the same BigGAN-128 iteration through the
# bf16 tcgen05 path and through the fp32 SIMT parity engine (gpurun -- bash tools/table3_precision.sh).
export PARAGAN_ALLOW_SHORT_WARMUP=1
for B in 64 256; do
  for c in bf16 f32; do
    timeout 600 python bench.py --compute $c --batch $B --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-profile \
      > gpurun_out/t3_${c}_b${B}.log 2>&1; echo "rc=$?" >> gpurun_out/t3_${c}_b${B}.log
  done
done
