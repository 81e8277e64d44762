#!/usr/bin/env python
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv):
  python scripts/launch_table.py gpurun_out/launches_c4.csv [steps]"""
import collections
import csv
import sys

path = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
h = rows[0]
agg = collections.OrderedDict()
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    n = d["Kernel Name"].split("(")[0]
    unit = d.get("Metric Unit", "ns")
    v = float(d["Metric Value"]) * (1e3 if unit == "us" else (1e6 if unit == "ms" else 1.0))
    agg.setdefault(n, [0, 0.0])
    agg[n][0] += 1
    agg[n][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'ms/step':>9} {'launches':>8} {'share':>6}  kernel")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / 1e6 / steps:9.3f} {c:8d} {100 * t / tot:5.1f}%  {n}")
print(f"{tot / 1e6 / steps:9.3f} total")
