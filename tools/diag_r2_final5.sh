cd $GRAFT_REPO_ROOT
# End-of-round profile with R38 (launch list + per-layer table + ncu --set full of k_conv_fprop_cg2<256, 2>)
ROUND=r2f timeout 2400 bash tools/profile_round.sh cg2_256_2 > gpurun_out/f5_prof.log 2>&1
tail -3 gpurun_out/f5_prof.log
head -30 gpurun_out/launches_summary.md
