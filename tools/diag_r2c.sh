cd $GRAFT_REPO_ROOT
B128="--res 128 --ch 96 --attn 64 --classes 1000 --shared 128 --zc 20"
timeout 600 python -m pytest tests/test_gpu_optim.py tests/test_gpu_boundary.py -q -s > gpurun_out/d3_optim_boundary.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_step.py -q -s -k "f32_biggan128 or isolated" > gpurun_out/d3_f32.log 2>&1
PARAGAN_SUBPIXEL=0 timeout 900 python tools/parity_report.py $B128 --batch 16 --seed 24 --bf16 --summary > gpurun_out/d3_b16_nosub.log 2>&1
echo done
