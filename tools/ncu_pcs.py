"""Top stall PCs of one kernel in an ncu --set full report (source page, SASS).

    python tools/ncu_pcs.py REPORT KERNEL_REGEX [N] [--launch K]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else 40
    launch = sys.argv[sys.argv.index("--launch") + 1] if "--launch" in sys.argv else "0"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-skip", launch, "--launch-count", "1", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    hdr = rows[hi[0]]
    end = hi[1] if len(hi) > 1 else len(rows)
    data = [r for r in rows[hi[0] + 1:end] if r and len(r) == len(hdr)]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iw, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = sum(f(r[iw]) for r in data) or 1.0
    print(f"# {kern}: {tot:.0f} samples, {len(data)} SASS instructions")
    for r in sorted(sorted(data, key=lambda r: -f(r[iw]))[:n], key=lambda r: r[ia]):
        print(f"{100 * f(r[iw]) / tot:5.1f}% {r[ia][-5:]} {f(r[ie]):10.0f}  {r[isrc][:100]}")


if __name__ == "__main__":
    main()
