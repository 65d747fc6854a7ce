set -x
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/d1_nproc.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=15 > gpurun_out/d1_fullsize.log 2>&1
timeout 600 python -m pytest tests/test_gpu_step.py -q -s -k "isolated" > gpurun_out/d1_isolated.log 2>&1
timeout 300 python tools/parity_report.py --bf16 --batch 8 > gpurun_out/d1_micro_bf16.log 2>&1
timeout 600 python tools/parity_report.py --res 128 --ch 96 --attn 64 --classes 1000 --shared 128 --zc 20 --batch 8 --seed 24 --bf16 > gpurun_out/d1_b128_bf16.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/d1_bench.log 2>&1
echo done
