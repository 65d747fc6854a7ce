"""Per-layer conv table from a PARAGAN_PROFILE_VERBOSE=1 bench log (PROF lines)."""
import collections
import re
import sys

rows = []
for l in open(sys.argv[1]):
    m = re.match(r"PROF kind=(\d) ms=([\d.]+) tflops=([\d.]+)(?: exec_tflops=[\d.]+)? (.*)", l.strip())
    if m:
        rows.append((int(m[1]), float(m[2]), float(m[3]), m[4]))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for k, ms, tf, w in rows:
    a = agg[(k, w)]
    a[0] += 1
    a[1] += ms
    a[2] += ms * tf
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = {k: sum(v[1] for kk, v in agg.items() if kk[0] == k) for k in (0, 1, 2)}
print(f"# per-layer device time (ms per step): fprop/dgrad {tot[0]:.2f}, wgrad {tot[1]:.2f}, collectives {tot[2]:.2f}\n")
print("| launch | count | ms | TFLOP/s |")
print("|---|---|---|---|")
for (k, w), (c, ms, ft) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
    print(f"| {w} | {c} | {ms:.3f} | {ft / ms:.0f} |" if k < 2 else f"| {w} | {c} | {ms:.3f} | - |")
