cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_attn.py -q > gpurun_out/d14_attn.log 2>&1
for lib in base new base new; do
  if [ $lib = base ]; then export PARAGAN_LIB=$GRAFT_REPO_ROOT/paper_2411_03999_b200/libparagan_base.so; else unset PARAGAN_LIB; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d14_bench_$lib.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d14_bench_$lib.log').read().strip().splitlines()[-1]);print('$lib', round(d['value'],1), d['roofline']['other_kernels_ms_per_step'])" >> gpurun_out/d14_summary.txt
done
unset PARAGAN_LIB
echo done
