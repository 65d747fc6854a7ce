"""Per-launch DRAM traffic of the kernel families bench.py reports, from a compact ncu launch
list (tools/ncu_compact.py output).  Written to profiles/<round>_traffic.json and read by bench.py
for roofline.traffic (cold-cache, serialised ncu replay: an upper bound on the in-step traffic).

    python tools/traffic_from_launches.py profiles/round1_launches.csv > profiles/round1_traffic.json
"""
import csv
import json
import re
import sys

GROUPS = {"conv_fprop": r"^k_conv_fprop", "conv_wgrad": r"^k_conv_wgrad", "attn_fwd": r"^k_attn_fwd",
          "attn_bwd": r"^k_attn_bwd"}


def main():
    rows = list(csv.DictReader(open(sys.argv[1])))
    out = {"source": sys.argv[1], "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
           "dram__bytes_write.sum --clock-control none; per launch averages over every launch of the family"}
    for g, pat in GROUPS.items():
        sel = [r for r in rows if re.search(pat, r["kernel"])]
        if not sel:
            continue
        b = [1e6 * (float(r["dram_read_mb"]) + float(r["dram_write_mb"])) for r in sel]
        t = [float(r["time_us"]) for r in sel]
        out[g] = {"launches": len(sel), "dram_bytes_per_launch": sum(b) / len(b), "time_us_per_launch": sum(t) / len(t),
                  "dram_GBps": sum(b) / (sum(t) * 1e3)}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
