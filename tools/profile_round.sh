# One GPU box: the round's profile set (run from the repo root: gpurun -- bash tools/profile_round.sh).
#   gpurun_out/launches_compact.csv  one row per launch (ncu, cold cache, serialised), two iterations
#   gpurun_out/launches_summary.md   per-kernel shares
#   gpurun_out/layers.md             per-layer tcgen05 conv table from CUDA events inside a bench step
#   gpurun_out/r1_<name>.md          ncu --set full summaries of the top kernels
export PARAGAN_ALLOW_SHORT_WARMUP=1
export PARAGAN_GRAPHS=0   # ncu profiles eager launches (graph replays are not listed per kernel)
CMD="python bench.py --steps 1 --warmup 1 --repeats 1 --reals uniform --no-cpu-baseline --no-e2e --no-profile"
$CMD > gpurun_out/plain_round.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_raw.csv $CMD > gpurun_out/ncu_launches.log 2>&1
python tools/ncu_compact.py gpurun_out/launches_raw.csv > gpurun_out/launches_compact.csv
python tools/ncu_summary.py gpurun_out/launches_raw.csv --iters 2 > gpurun_out/launches_summary.md 2>&1
rm -f gpurun_out/launches_raw.csv
PARAGAN_PROFILE_VERBOSE=1 python bench.py --steps 1 --warmup 3 --repeats 1 --reals uniform --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/layers.err
python tools/prof_layers.py gpurun_out/layers.err 70 2 > gpurun_out/layers.md
bash tools/profile_top_kernels.sh "$@"
