cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d39_bench.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/d39_bench.log').read().strip().splitlines()[-1]);print('new', round(d['value'],1), d['losses']['d'], d['losses']['g'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:im2col -c 4 --csv --log-file gpurun_out/d39_ncu.csv env PARAGAN_GRAPHS=0 PARAGAN_ALLOW_SHORT_WARMUP=1 python bench.py --steps 1 --warmup 1 --repeats 1 --no-cpu-baseline --no-e2e --no-profile > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/d39_ncu.csv --iters 1 2>&1 | head -6
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "bf16" 2>&1 | tail -1
