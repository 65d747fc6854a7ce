cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d32_bench.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/d32_bench.log').read().strip().splitlines()[-1]);print(round(d['value'],1), d['losses']['d'], d['losses']['g'], d['gpu_launches'])"
timeout 900 python -m pytest tests/test_gpu_step.py -q -x -k "bf16 or sn" 2>&1 | tail -1
