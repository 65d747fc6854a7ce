cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py -q -x > gpurun_out/d29_step.log 2>&1; tail -2 gpurun_out/d29_step.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
BASE=$GRAFT_REPO_ROOT/paper_2411_03999_b200/libparagan_base.so
for lib in base new base new; do
  if [ $lib = base ]; then export PARAGAN_LIB=$BASE; else unset PARAGAN_LIB; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d29_bench_$lib.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d29_bench_$lib.log').read().strip().splitlines()[-1]);print('$lib', round(d['value'],1), d['gpu_launches'], d['losses']['d'], d['losses']['g'])"
done
