# The driver's round-end checks on one GPU (gpurun -- bash tools/full_check.sh): the whole -m gpu suite,
# smoke(), the default bench line; logs in gpurun_out/fc_*.log
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/fc_tests.log 2>&1
echo "tests rc=$? after ${SECONDS}s" >> gpurun_out/fc_summary.txt
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fc_summary.txt
timeout 900 python bench.py > gpurun_out/fc_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/fc_summary.txt
for im in 0 1; do
  PARAGAN_IM2COL=$im timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/fc_bench_im2col$im.log 2>&1
done
echo done
