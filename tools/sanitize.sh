# compute-sanitizer over a cross-section of the GPU tests (gpurun -- bash tools/sanitize.sh): memcheck on
# every kernel family (layout, tcgen05 fprop in all three variants / wgrad / sub-pixel, fused attention,
# fp32 SIMT step, bf16 step, optimiser); racecheck and synccheck on a smaller set (they serialise every
# shared-memory access).  Logs: gpurun_out/san_<tool>.log, exit codes in gpurun_out/san_summary.txt
cd $GRAFT_REPO_ROOT
T=tests/test_gpu_ops.py
MEM="$T::test_layout_pack_bit_exact $T::test_tc_conv_fprop_integer_exact[shape0] $T::test_tc_conv_fprop_integer_exact[shape10] $T::test_tc_conv_fprop_integer_exact[shape13] $T::test_tc_conv_fprop_integer_exact[shape17] $T::test_tc_conv_wgrad_integer_exact[shape1] $T::test_tc_conv_wgrad_integer_exact[shape18] $T::test_tc_conv_wgrad_integer_exact[shape20] $T::test_conv_up2_phase_decomposition_integer_exact[shape0] $T::test_conv_up2_wgrad_integer_exact[shape5] $T::test_thin_conv_f32_fwd_dgrad_wgrad tests/test_gpu_attn.py tests/test_gpu_step.py::test_step_parity_f32_micro tests/test_gpu_step.py::test_step_parity_bf16_micro tests/test_gpu_optim.py::test_policy_update_matches_oracle"
SMALL="$T::test_tc_conv_fprop_integer_exact[shape0] $T::test_tc_conv_fprop_integer_exact[shape13] $T::test_tc_conv_wgrad_integer_exact[shape1] $T::test_conv_up2_phase_decomposition_integer_exact[shape0] tests/test_gpu_attn.py::test_attn_bwd_deterministic"
rm -f gpurun_out/san_summary.txt
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 50 \
    python -m pytest $MEM -q -p no:cacheprovider > gpurun_out/san_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/san_summary.txt
for tool in racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 50 \
      python -m pytest $SMALL -q -p no:cacheprovider > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_summary.txt
done
echo done
