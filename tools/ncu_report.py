"""Key metrics of an `ncu --set full` report, one row per captured launch (markdown).

    python tools/ncu_report.py gpurun_out/prof.ncu-rep [--flops F1,F2,...] > profiles/<name>.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1tex %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem LSU %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem TC %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("launch__registers_per_thread", "regs"),
]


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full: {rep}\n")
    print("| kernel | grid | " + " | ".join(m[1] for m in METRICS) + " |")
    print("|---|---|" + "---|" * len(METRICS))
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
        cells = []
        for m, _ in METRICS:
            i = idx.get(m)
            if i is None:   # section-prefixed names (e.g. "TPC.TriageCompute.<metric>")
                i = next((j for h, j in idx.items() if h.endswith("." + m)), None)
            cells.append(f"{r[i]} {units[i]}".strip() if i is not None else "-")
        print(f"| `{name}` | {r[idx.get('Grid Size', 0)]} | " + " | ".join(cells) + " |")
    stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    print("\nTop warp-stall samples (all warps, incl. idle producer/MMA/epilogue waits):\n")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void ", "")
        vals = sorted(((float(r[idx[h]] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stall),
                      reverse=True)[:6]
        print(f"- `{name}`: " + ", ".join(f"{n} {int(v)}" for v, n in vals))


if __name__ == "__main__":
    main()
