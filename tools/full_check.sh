# The driver's round-end checks on one GPU (gpurun -- bash tools/full_check.sh): the whole -m gpu suite,
# smoke(), the default bench line, the reference arm; logs in gpurun_out/fc_*.log
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/fc_summary.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/fc_tests.log 2>&1
echo "tests rc=$? after ${SECONDS}s: $(tail -1 gpurun_out/fc_tests.log)" >> gpurun_out/fc_summary.txt
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fc_summary.txt
timeout 900 python bench.py > gpurun_out/fc_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/fc_summary.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fc_reference.log 2>&1
echo "reference rc=$?" >> gpurun_out/fc_summary.txt
PARAGAN_GRAPHS=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/fc_bench_eager.log 2>&1
echo "eager bench rc=$?" >> gpurun_out/fc_summary.txt
cat gpurun_out/fc_summary.txt
