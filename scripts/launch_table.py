"""Print the per-launch times of the last refine call in an ncu --csv
launch list (scripts/cnn_once.py runs two; the second is printed)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                     "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
            out.append((d["Kernel Name"].split("(")[0].replace("ts::<unnamed>::", "")
                        .replace("void ", ""),
                        float(d["Metric Value"].replace(",", "")) * scale))
n = len(out) // 2
run = out[n:]
print(f"{len(run)} launches, total {sum(v for _, v in run):.1f} us")
for k, v in run:
    print(f"  {v:8.1f}  {k}")
