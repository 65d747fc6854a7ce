cd $GRAFT_REPO_ROOT
B128="--res 128 --ch 96 --attn 64 --classes 1000 --shared 128 --zc 20"
timeout 600 python -m pytest tests/test_gpu_optim.py -q -s > gpurun_out/d2_optim.log 2>&1
timeout 600 python tools/parity_report.py $B128 --batch 2 --seed 24 --g-isolated > gpurun_out/d2_giso_f32.log 2>&1
timeout 600 python tools/parity_report.py $B128 --batch 2 --seed 24 --summary > gpurun_out/d2_b128_f32.log 2>&1
timeout 300 python tools/parity_report.py --bf16 --batch 8 --summary > gpurun_out/d2_micro_bf16.log 2>&1
timeout 900 python tools/parity_report.py $B128 --batch 16 --seed 24 --bf16 > gpurun_out/d2_b128_bf16_b16.log 2>&1
echo done
