"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of
bench.py: split into steps at k_validate (first kernel of xm_build_Q) and print
per-kernel launches / time / share for one step (default: the 4th = the timed
step).  usage: python tools/launch_summary.py launches.csv [step]"""
import csv, sys
from collections import defaultdict

path = sys.argv[1]
want = int(sys.argv[2]) if len(sys.argv) > 2 else 3
steps, cur = [], None
with open(path) as f:
    rows = [r for r in csv.reader(f) if len(r) > 5 and r[-3] == "gpu__time_duration.sum"]
for r in rows:
    name = r[4].split("(")[0]
    if name.startswith("xm::k_validate"):
        cur = []
        steps.append(cur)
    if cur is not None:
        cur.append((name, float(r[-1]) / 1e3))  # µs
step = steps[want]
agg = defaultdict(lambda: [0, 0.0])
for n, us in step:
    agg[n][0] += 1
    agg[n][1] += us
tot = sum(v[1] for v in agg.values())
print(f"steps found: {len(steps)}; step {want}: {len(step)} launches, sum of kernel durations {tot / 1e3:.2f} ms")
print(f"{'kernel':46s} {'launches':>8s} {'sum ms':>9s} {'share':>6s} {'avg us':>9s}")
for n, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{n:46s} {c:8d} {us / 1e3:9.2f} {100 * us / tot:5.1f}% {us / c:9.2f}")
