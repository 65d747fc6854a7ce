cd $GRAFT_REPO_ROOT
BASE=$GRAFT_REPO_ROOT/paper_2411_03999_b200/libparagan_base.so
for lib in base new base new; do
  if [ $lib = base ]; then export PARAGAN_LIB=$BASE; else unset PARAGAN_LIB; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d34_bench_$lib.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d34_bench_$lib.log').read().strip().splitlines()[-1]);print('$lib', round(d['value'],1), d['losses']['d'], d['losses']['g'])"
done
unset PARAGAN_LIB
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_bn_ -c 120 --csv --log-file gpurun_out/d34_bn.csv env PARAGAN_ALLOW_SHORT_WARMUP=1 python bench.py --steps 1 --warmup 1 --repeats 1 --reals uniform --no-cpu-baseline --no-e2e --no-profile > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/d34_bn.csv --iters 1 2>&1 | head -10
