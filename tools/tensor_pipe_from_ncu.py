"""Tensor-pipe utilisation of the profiled conv / attention kernels from the `--set full` summaries
(tools/ncu_report.py output, gpurun_out/<round>_<name>.md), for bench.py's conv_tensor_pipe_util.

    python tools/tensor_pipe_from_ncu.py gpurun_out/r2_*.md > profiles/round2_tensor_pipe.json
"""
import json
import re
import sys


def main():
    out = {"note": "ncu --set full --clock-control none, one launch per kernel (cold cache, serialised): "
                   "sm__pipe_tensor... utilisation as reported in the summary tables"}
    for path in sys.argv[1:]:
        for line in open(path):
            if not line.startswith("| `"):
                continue
            cols = [c.strip() for c in line.strip().strip("|").split("|")]
            name = re.sub(r"^`(unnamed>::)?|`$", "", cols[0])
            m = re.match(r"([0-9.]+)", cols[6])
            if m:
                out[name] = {"tensor_pipe_pct": float(m.group(1)), "time": cols[2], "source": path}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
