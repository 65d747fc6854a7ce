cd $GRAFT_REPO_ROOT
BASE=$GRAFT_REPO_ROOT/paper_2411_03999_b200/libparagan_base.so
PARAGAN_LIB=$BASE timeout 300 python tools/bench_conv.py 2>&1 | tail -10 | sed 's/^/base /'
timeout 300 python tools/bench_conv.py 2>&1 | tail -10 | sed 's/^/new  /'
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_guard.py tests/test_gpu_attn.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for lib in base new base new; do
  if [ $lib = base ]; then export PARAGAN_LIB=$BASE; else unset PARAGAN_LIB; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d28_bench_$lib.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d28_bench_$lib.log').read().strip().splitlines()[-1]);print('$lib', round(d['value'],1), round(d['roofline']['achieved_executed'],1), round(d['roofline']['wgrad']['achieved_executed'],1))"
done
