cd $GRAFT_REPO_ROOT
# R38 + half-resolution shortcut wgrad: A/B, then the full round-end check
for v in 0 1; do
  PARAGAN_POOL_FWD=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d44_bench_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/d44_bench_$v.log').read().strip().splitlines()[-1]);print('poolfwd=$v', round(d['value'],1), d['losses']['d'], d['losses']['g'])" || tail -5 gpurun_out/d44_bench_$v.log
done
bash tools/full_check.sh
python -c "import json;d=json.loads(open('gpurun_out/fc_bench.log').read().strip().splitlines()[-1]);print('default', d['value'], d['e2e']['value'], d['roofline'])"
