cd $GRAFT_REPO_ROOT
ROUND=r2e timeout 2400 bash tools/profile_round.sh cg2_96_2 > gpurun_out/f4_prof.log 2>&1
tail -3 gpurun_out/f4_prof.log
head -30 gpurun_out/launches_summary.md
