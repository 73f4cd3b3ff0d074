"""Aggregate an ncu --csv launch list: total / share / count / average per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    k = r[ki].split("(")[0][:70]
    agg[k][0] += 1
    agg[k][1] += float(r[vi]) / 1e3
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1]:9.1f} us {100 * v[1] / tot:5.1f}% n={v[0]:4d} avg={v[1] / v[0]:7.2f}  {k}")
