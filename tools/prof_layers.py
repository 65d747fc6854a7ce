"""Per-layer conv table from a PARAGAN_PROFILE_VERBOSE=1 bench log (PROF lines).

    python tools/prof_layers.py LOG [rows] [dup]     # dup: how often each conv launch is printed

bench.py queries the profile for kinds 0/1 (algorithmic flops) and again for 3/4 (executed flops), and
each query prints the kind-0/1 records, so one step's conv launches appear `dup` = 2 times; the other
kinds (5 attention, 6 thin) are printed once.

TFLOP/s columns: algorithmic (G's sub-pixel conv1 counted over the upsampled tensor) and
executed (the flops issued to the tensor cores).
"""
import collections
import re
import sys

rows = []
for l in open(sys.argv[1]):
    m = re.match(r"PROF kind=(\d) ms=([\d.]+) tflops=([\d.]+)(?: exec_tflops=([\d.]+))? (.*)", l.strip())
    if m:
        rows.append((int(m[1]), float(m[2]), float(m[3]), float(m[4]) if m[4] else float(m[3]), m[5]))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for k, ms, tf, etf, w in rows:
    a = agg[(k, w)]
    a[0] += 1
    a[1] += ms
    a[2] += ms * tf
    a[3] += ms * etf
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
dup = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
tot = {k: sum(v[1] for kk, v in agg.items() if kk[0] == k) / (dup if k < 2 else 1.0) for k in (0, 1, 2)}
print(f"# per-layer device time (ms per step): fprop/dgrad {tot[0]:.2f}, wgrad {tot[1]:.2f}, collectives {tot[2]:.2f}\n")
print("| launch | launches/step | ms/step | TFLOP/s (algorithmic) | TFLOP/s (executed) |")
print("|---|---|---|---|---|")
norm = {kw: v[1] / (dup if kw[0] < 2 else 1.0) for kw, v in agg.items()}
for (k, w), (c, ms, ft, eft) in sorted(agg.items(), key=lambda kv: -norm[kv[0]])[:n]:
    steps = dup if k < 2 else 1.0
    if k < 2:
        print(f"| {w} | {c / steps:g} | {ms / steps:.3f} | {ft / ms:.0f} | {eft / ms:.0f} |")
    else:
        print(f"| {w} | {c / steps:g} | {ms / steps:.3f} | - | - |")
