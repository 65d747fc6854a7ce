cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_guard.py -q -k "thin" > gpurun_out/d13_thin_tests.log 2>&1
for cpt in 1 2; do PARAGAN_THIN_DG_CPT=$cpt timeout 300 python tools/bench_thin.py 20 >> gpurun_out/d13_thin.log 2>&1; done
export ROUND=r2
timeout 2400 bash tools/profile_round.sh cg2_192_1 cg2_96_0 cg2_256_2 wgrad3_96 wgrad_cg2_256 attn_fwd attn_bwd thin_fwd thin_dgrad thin_wgrad bn_apply_bulk bn_bwd_apply_bulk > gpurun_out/d13_profile.log 2>&1
echo done
