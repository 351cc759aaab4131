"""Turn the scripts/profile_round.sh outputs into the committed profiles/
summaries: step kernel table (markdown), traffic JSON read by bench.py, and
the key ncu --set full metrics of the two captured kernels."""
import collections
import csv
import json
import os
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = "gpurun_out", "profiles"


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ii = (h.index("Kernel Name"), h.index("Metric Name"),
                      h.index("Metric Value"), h.index("ID"))
    out = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = out.setdefault(r[ii], {"name": r[ki].split("(")[0].split("::")[-1]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return list(out.values())


L = launches(f"{G}/{R}_launch_metrics.csv")
start = next(i for i, d in enumerate(L) if "chunk_count" in d["name"])
end = next(i for i in range(start, len(L)) if "refine_epilogue" in L[i]["name"])
step = L[start:end + 1]
agg = collections.OrderedDict()
for d in step:
    a = agg.setdefault(d["name"], [0, 0.0, 0.0, 0.0])
    t = d.get("gpu__time_duration.sum", 0.0) / 1e3
    a[0] += 1
    a[1] += t
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    a[3] += t * d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
tot = sum(a[1] for a in agg.values())
md = [f"# {R}: one bench step (1,024 tiles), ncu launch list "
      "(--clock-control none, serialized, cold L2 per launch)", "",
      "| kernel | launches | time (us) | share | DRAM bytes | tensor pipe active (time-weighted) |",
      "|---|---|---|---|---|---|"]
for name, (n, t, b, tw) in sorted(agg.items(), key=lambda x: -x[1][1]):
    md.append(f"| {name} | {n} | {t:.1f} | {100 * t / tot:.1f}% | {b / 1e6:.1f} MB | "
              f"{tw / t if t else 0:.1f}% |")
cnn = [d for d in step if any(k in d["name"] for k in ("conv", "copy_inputs", "epilogue"))]
cnn_b = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in cnn)
cnn_t = sum(d.get("gpu__time_duration.sum", 0) for d in cnn) / 1e3
md += ["", f"step total {tot / 1e3:.3f} ms; CNN launches {cnn_t / 1e3:.3f} ms "
       f"({100 * cnn_t / tot:.1f}%), CNN DRAM {cnn_b / 1e9:.3f} GB"]
B = launches(f"{G}/{R}_bake_launches.csv")
splat = [d for d in B if "bake_splat" in d["name"]][-1]
fin = [d for d in B if "bake_finalize" in d["name"]][-1]
bake_b = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
             for d in (splat, fin))
md += ["", "splat (configs[2], 200M points, 4,096 heightmaps): "
       f"bake_splat {splat['gpu__time_duration.sum'] / 1e6:.3f} ms, "
       f"{(splat['dram__bytes_read.sum'] + splat['dram__bytes_write.sum']) / 1e9:.2f} GB; "
       f"bake_finalize {fin['gpu__time_duration.sum'] / 1e6:.3f} ms"]
open(f"{P}/{R}_step_kernels.md", "w").write("\n".join(md) + "\n")
json.dump({"cnn_dram_bytes_per_step": cnn_b, "cnn_ncu_us_per_step": cnn_t,
           "step_ncu_us": tot, "bake_dram_bytes_per_launch": bake_b,
           "source": f"profiles/{R}_step_kernels.md (ncu launch lists of bench.py)"},
          open(f"{P}/{R}_traffic.json", "w"), indent=1)
for cap in ("fuse0", "splat", "raster", "delaunay"):
    rep = f"{G}/{R}_{cap}.ncu-rep"
    if not os.path.exists(rep):
        continue
    txt = subprocess.run([sys.executable, "scripts/ncu_details.py", rep],
                         capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    keep = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active")
    extra = [f"   {k:60s} {v}" for k, v in zip(r[0], r[2]) if k in keep]
    open(f"{P}/{R}_ncu_{cap}.txt", "w").write(
        f"ncu --set full --clock-control none --import-source on ({rep})\n" + txt +
        "\n".join(extra) + "\n")
print("\n".join(md))
