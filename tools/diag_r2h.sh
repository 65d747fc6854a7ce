cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py -q -s -k "isolated_bf16" > gpurun_out/d8_giso.log 2>&1
export ROUND=r2
timeout 2400 bash tools/profile_round.sh attn_fwd attn_bwd thin_fwd thin_wgrad wgrad3_96 cg2_96_0 bn_bwd_apply_bulk > gpurun_out/d8_profile.log 2>&1
echo done
