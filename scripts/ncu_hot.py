"""Top SASS instructions by warp-stall samples for one launch of an .ncu-rep
(with the CUDA source line when -lineinfo is present)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kid = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kid:
    cmd += ["--launch-skip", kid, "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
body = [r for r in rows[hi + 1:] if len(r) > si and r[si].isdigit()]
tot = sum(int(r[si]) for r in body)
print(f"samples {tot}, warp instructions {sum(int(r[ie] or 0) for r in body)}")
for r in sorted(body, key=lambda r: -int(r[si]))[:n]:
    print(f"{int(r[si]) / tot * 100:5.1f}% {r[ie]:>10s}  {r[1].strip()[:90]}")
