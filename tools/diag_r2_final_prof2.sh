cd $GRAFT_REPO_ROOT
ROUND=r2c timeout 2400 bash tools/profile_round.sh cg2_192_1 cg2_96_3 cg2_256_2 attn_fwd attn_bwd wgrad3_96 out_conv_fwd out_conv_bwd bn_bwd_apply_bulk > gpurun_out/f2_prof.log 2>&1
tail -12 gpurun_out/f2_prof.log
