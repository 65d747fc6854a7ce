cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_ops.py -q -x 2>&1 | tail -1
BASE=$GRAFT_REPO_ROOT/paper_2411_03999_b200/libparagan_base.so
PARAGAN_LIB=$BASE timeout 300 python tools/bench_attn.py 10 2>&1 | sed "s/^/base /"
timeout 300 python tools/bench_attn.py 10 2>&1 | sed "s/^/new  /"
for lib in base new base new; do
  if [ $lib = base ]; then export PARAGAN_LIB=$BASE; else unset PARAGAN_LIB; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d26_bench_$lib.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d26_bench_$lib.log').read().strip().splitlines()[-1]);print('$lib', round(d['value'],1), d['roofline']['achieved_executed'], d['roofline']['other_kernels_ms_per_step'])"
done
