cd $GRAFT_REPO_ROOT
# R38 for D's first block (96 channels at 128^2): A/B and per-layer times
for v in 0 1 0 1; do
  PARAGAN_POOL_FWD0=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d45_bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d45_bench_$v.log').read().strip().splitlines()[-1]);print('poolfwd0=$v', round(d['value'],1), d['losses']['d'], d['losses']['g'])" || tail -5 gpurun_out/d45_bench_$v.log
done
PARAGAN_POOL_FWD0=1 PARAGAN_PROFILE_VERBOSE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --repeats 1 > /dev/null 2> gpurun_out/d45_layers.err
python tools/prof_layers.py gpurun_out/d45_layers.err 80 2 > gpurun_out/d45_layers.md; grep -E "128x128|fwd-pool" gpurun_out/d45_layers.md
PARAGAN_POOL_FWD0=1 timeout 1800 python -m pytest tests/test_gpu_step.py tests/test_gpu_boundary.py -q -x 2>&1 | tail -3
