cd $GRAFT_REPO_ROOT
bash tools/full_check.sh
ROUND=r2d timeout 2400 bash tools/profile_round.sh attn_fwd cg2_96_3 > gpurun_out/f3_prof.log 2>&1
tail -4 gpurun_out/f3_prof.log
head -8 gpurun_out/launches_summary.md
