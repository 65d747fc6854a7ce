cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d43_bench_$i.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/d43_bench_$i.log').read().strip().splitlines()[-1]);print('new', round(d['value'],1), d['losses']['d'], d['losses']['g'])"; done
for i in 1 2; do PARAGAN_DGRAD_UP2=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d43_off_$i.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/d43_off_$i.log').read().strip().splitlines()[-1]);print('off', round(d['value'],1))"; done
timeout 1500 python -m pytest tests/test_gpu_step.py tests/test_gpu_boundary.py -q -x 2>&1 | tail -1
