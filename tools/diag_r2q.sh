cd $GRAFT_REPO_ROOT
for v in 0 1; do
  PARAGAN_THIN_TC=$v timeout 600 python bench.py --trace 40 > gpurun_out/d18_trace_$v.log 2>&1
done
paste <(grep trace_step gpurun_out/d18_trace_0.log | python -c "import sys,json;[print('%d %.5f %.5f'%(d['trace_step'],d['d_loss'],d['g_loss'])) for d in map(json.loads,sys.stdin)]") <(grep trace_step gpurun_out/d18_trace_1.log | python -c "import sys,json;[print('%.5f %.5f'%(d['d_loss'],d['g_loss'])) for d in map(json.loads,sys.stdin)]")
