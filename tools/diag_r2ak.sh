cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_attn.py -q -x 2>&1 | tail -1
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d37_bench_$i.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/d37_bench_$i.log').read().strip().splitlines()[-1]);print('new', round(d['value'],1), d['roofline']['other_kernels_ms_per_step'], d['losses']['d'], d['losses']['g'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rowmaxnorm -c 16 --csv --log-file gpurun_out/d37_ncu.csv env PARAGAN_GRAPHS=0 PARAGAN_ALLOW_SHORT_WARMUP=1 python bench.py --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline --no-e2e --no-profile > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/d37_ncu.csv --iters 1 2>&1 | head -6
timeout 1200 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -1
