# Capture ncu --set full reports of the top kernels of one bench step and summarise them on
# the GPU box (gpurun -- bash tools/profile_top_kernels.sh [name ...]); summaries land in
# gpurun_out/${ROUND}_<name>.md (the .ncu-rep files are deleted unless KEEP_REP=1: gpurun returns
# at most 64 MiB).
export PARAGAN_ALLOW_SHORT_WARMUP=1
export PARAGAN_GRAPHS=0   # ncu profiles eager launches (graph replays are not listed per kernel)
CMD="python bench.py --steps 1 --warmup 1 --repeats 1 --reals uniform --no-cpu-baseline --no-e2e --no-profile"
$CMD > gpurun_out/plain_prof.log 2>&1 || exit 1
SPECS="cg2_192_1:k_conv_fprop_cg2<.int.192, .int.1>:4 cg2_96_0:k_conv_fprop_cg2<.int.96, .int.0>:2 cg2_256_2:k_conv_fprop_cg2<.int.256, .int.2>:6 wgrad_192:k_conv_wgrad<.int.192>:4 wgrad_256:k_conv_wgrad<.int.256>:4 thin_fwd:k_thin_fwd:1 thin_wgrad:k_thin_wgrad:0 thin_dgrad:k_thin_dgrad:0 attn_fwd:k_attn_fwd:1 attn_bwd:k_attn_bwd:0"
want="$*"
IFS=' '
for spec in $SPECS; do :; done
python - "$want" <<'PY' > /tmp/specs.txt
import sys
specs = """cg2_192_1|k_conv_fprop_cg2<.int.192, .int.1>|4
cg2_96_0|k_conv_fprop_cg2<.int.96, .int.0>|2
cg2_256_2|k_conv_fprop_cg2<.int.256, .int.2>|6
wgrad_192|k_conv_wgrad<.int.192>|4
wgrad_256|k_conv_wgrad<.int.256>|4
thin_fwd|k_thin_fwd|1
thin_wgrad|k_thin_wgrad|0
thin_dgrad|k_thin_dgrad|0
attn_fwd|k_attn_fwd|1
attn_bwd|k_attn_bwd|0
wgrad3_96|k_conv_wgrad3<.int.96>|2
wgrad_cg2_256|k_conv_wgrad_cg2<.int.256>|2
bn_apply_bulk|k_bn_apply_relu_bulk|4
bn_bwd_apply_bulk|k_bn_bwd_apply_bulk|2
bn_bwd_reduce_bulk|k_bn_bwd_reduce_bulk|2
cg2_96_3|k_conv_fprop_cg2<.int.96, .int.3>|1
cg2_96_2|k_conv_fprop_cg2<.int.96, .int.2>|2
out_conv_fwd|k_out_conv_fwd|1
out_conv_bwd|k_out_conv_bwd|0""".splitlines()
want = sys.argv[1].split()
for s in specs:
    if not want or s.split("|")[0] in want:
        print(s)
PY
while IFS='|' read -r name kre skip; do
  rep=gpurun_out/${ROUND:-r2}_$name
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$kre" -s $skip -c 1 -o $rep $CMD > gpurun_out/ncu_$name.log 2>&1
  echo "$name $?"
  if [ -f $rep.ncu-rep ]; then
    python tools/ncu_report.py $rep.ncu-rep > $rep.md 2>&1
    short=$(echo "$kre" | sed 's/<.*//')
    python tools/ncu_pcs.py $rep.ncu-rep "$short" 40 >> $rep.md 2>&1
    [ "$KEEP_REP" = "1" ] || rm -f $rep.ncu-rep
  fi
done < /tmp/specs.txt
