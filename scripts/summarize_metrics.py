"""Summarise an ncu --csv launch list with time/DRAM/tensor metrics into
markdown + a small JSON (per-step DRAM traffic of the CNN and bake)."""
import collections
import csv
import json
import sys

path, out_md, out_json = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"),
                  h.index("Metric Value"), h.index("Metric Unit"))
idi = h.index("ID")
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    d = launch.setdefault(r[idi], {"name": r[ki].split("(")[0].split("::")[-1]})
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0}.get(u, 1.0)
    d[r[mi]] = v * scale
# one bench step = from the first chunk_count launch to the refine epilogue
ids = list(launch)
start = next(i for i, k in enumerate(ids) if "chunk_count" in launch[k]["name"])
end = next(i for i, k in enumerate(ids[start:], start)
           if "refine_epilogue" in launch[k]["name"])
step = [launch[k] for k in ids[start:end + 1]]
agg = collections.OrderedDict()
for d in step:
    a = agg.setdefault(d["name"], [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    a[3] += d.get("gpu__time_duration.sum", 0.0) * \
        d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
tot = sum(a[1] for a in agg.values())
lines = ["| kernel | launches | time (us, ncu serialized) | share | DRAM bytes | "
         "tensor pipe active (time-weighted) |", "|---|---|---|---|---|---|"]
for name, (n, t, b, tw) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| {name} | {n} | {t:.1f} | {100 * t / tot:.1f}% | {b / 1e6:.1f} MB | "
                 f"{tw / t if t else 0:.1f}% |")
cnn = [d for d in step if "conv" in d["name"] or "upsample" in d["name"] or
       "copy_inputs" in d["name"] or "refine_epilogue" in d["name"]]
cnn_bytes = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
                for d in cnn)
cnn_time = sum(d.get("gpu__time_duration.sum", 0) for d in cnn)
bake = [d for d in launch.values() if "bake" in d["name"]]
bake_bytes = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
                 for d in bake[-2:])
open(out_md, "w").write("\n".join(lines) + "\n")
json.dump({"cnn_dram_bytes_per_step": cnn_bytes, "cnn_ncu_us_per_step": cnn_time,
           "step_ncu_us": tot, "bake_dram_bytes_per_launch": bake_bytes,
           "source": path}, open(out_json, "w"), indent=1)
print("\n".join(lines))
print(f"CNN DRAM {cnn_bytes / 1e9:.3f} GB/step; CNN ncu time {cnn_time / 1e3:.2f} ms; "
      f"bake DRAM {bake_bytes / 1e9:.3f} GB (20M-pt capture)")
