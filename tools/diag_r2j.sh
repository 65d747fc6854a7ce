cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_ops.py -q -k "attn or thin" > gpurun_out/d10_attn_thin.log 2>&1
for single in 1 0 1 0; do
PARAGAN_ATTN_SINGLE=$single timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/d10_bench_s$single.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/d10_bench_s$single.log').read().strip().splitlines()[-1]);print($single, d['value'], d['roofline']['other_kernels_ms_per_step'])" >> gpurun_out/d10_summary.txt
done
echo done
