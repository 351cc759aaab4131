"""Per-launch durations of one bench step from an ncu launch-list CSV."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
gi = h.index("Grid Size") if "Grid Size" in h else None
L = [(r[ki].split("(")[0][-44:], float(r[vi].replace(",", "")), r[gi] if gi is not None else "")
     for r in rows[hi + 1:]]
idx = [i for i, l in enumerate(L) if "chunk_count" in l[0]]
a, b = idx[-2], idx[-1]
tot = 0.0
for name, ns, grid in L[a:b]:
    tot += ns
    if ns > 20000:
        print(f"{name:46s} {ns / 1000:8.1f} us {grid}")
print(f"step total {tot / 1e6:.3f} ms (ncu, serialized)")
