"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3, "ms": 1e3}
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0][-60:]
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(v[1] for v in agg.values())
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{v / 1e3:9.3f} ms {n:5d}x {100 * v / tot:5.1f}%  {k}")
print(f"total {tot / 1e3:.3f} ms")
