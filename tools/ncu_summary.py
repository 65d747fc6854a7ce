"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/ncu_summary.py gpurun_out/launches.csv [--iters N] > profiles/<round>_launches.md

ncu times are cold-cache and serialised: compare each kernel's SHARE of the
step, not the absolute numbers.
"""
import collections
import csv
import io
import re
import sys


def load(path):
    with open(path) as f:
        txt = f.read()
    # ncu prefixes the CSV with its own log lines; keep from the header on
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    out = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        out.append((r["Kernel Name"], v * scale))
    return out


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    return name[:90]


def main():
    path = sys.argv[1]
    iters = 1
    if "--iters" in sys.argv:
        iters = int(sys.argv[sys.argv.index("--iters") + 1])
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, ms in rows:
        a = agg[short(n)]
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list summary: {len(rows)} launches, {tot:.2f} ms total ({tot / iters:.2f} ms per iteration)\n")
    print("| kernel | launches | ms (sum) | share |")
    print("|---|---|---|---|")
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {ms:.3f} | {100 * ms / tot:.1f}% |")


if __name__ == "__main__":
    main()
