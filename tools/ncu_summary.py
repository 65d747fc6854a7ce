"""Summarise an ncu launch list per kernel.

    ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --csv --log-file L <cmd>
    python tools/ncu_summary.py L [--iters N] > profiles/<round>_launches.md

ncu times are cold-cache and serialised: compare each kernel's SHARE of the
step, not the absolute numbers.
"""
import collections
import csv
import io
import re
import sys

TIME = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    """-> list of (kernel name, ms, dram bytes or None) in launch order."""
    with open(path) as f:
        txt = f.read()
    i = txt.find('"ID"')
    per = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO(txt[i:])):
        key = (r["ID"], r["Kernel Name"])
        d = per.setdefault(key, {})
        v = float(r["Metric Value"].replace(",", ""))
        u = r.get("Metric Unit", "")
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["ms"] = v * TIME.get(u, 1e-6)
        elif r["Metric Name"].startswith("dram__bytes"):
            d["bytes"] = d.get("bytes", 0.0) + v * BYTES.get(u, 1.0)
    return [(k[1], d.get("ms", 0.0), d.get("bytes")) for k, d in per.items()]


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    return name.replace("pg::<unnamed>::", "")[:80]


def main():
    path = sys.argv[1]
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 1
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, False])
    for n, ms, b in rows:
        a = agg[short(n)]
        a[0] += 1
        a[1] += ms
        if b is not None:
            a[2] += b
            a[3] = True
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list: {len(rows)} launches, {tot:.2f} ms total, {tot / iters:.2f} ms per iteration "
          f"({iters} iterations captured)\n")
    print("| kernel | launches/iter | ms/iter | share | DRAM GB/s |")
    print("|---|---|---|---|---|")
    for k, (c, ms, b, hb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        bw = f"{b / (ms * 1e6):.0f}" if hb and ms > 0 else "-"
        print(f"| `{k}` | {c / iters:g} | {ms / iters:.3f} | {100 * ms / tot:.1f}% | {bw} |")


if __name__ == "__main__":
    main()
