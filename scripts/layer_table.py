"""Per-launch table (time, DRAM bytes, tensor-pipe %) of the second refine
call in an ncu --csv launch list written by scripts/cnn_once.py."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
launches = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = int(d["ID"])
    e = launches.setdefault(k, {"name": d["Kernel Name"].split("(")[0]
                                .replace("void ", "").replace("ts::<unnamed>::", "")})
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    m = d["Metric Name"]
    if m == "gpu__time_duration.sum":
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(u, 1)
        e["us"] = v
    elif m.startswith("dram__bytes"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        e["dram"] = e.get("dram", 0) + v
    else:
        e["tc"] = v
L = list(launches.values())
L = L[len(L) // 2:]
tot = sum(e["us"] for e in L)
print(f"{len(L)} launches, {tot:.1f} us, DRAM {sum(e.get('dram', 0) for e in L) / 1e9:.2f} GB")
for e in L:
    print(f"  {e['us']:8.1f} us  {e.get('dram', 0) / 1e6:8.1f} MB  tc {e.get('tc', 0):5.1f}%  {e['name']}")
