"""Per-CUDA-source-line warp-stall samples (all + not-issued) of one launch."""
import csv
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = []
fname = None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0].isdigit() and len(r) > 6:
        try:
            lines.append((int(r[4]), int(r[5]), int(r[7] or 0), f"{fname}:{r[0]}", r[1].strip()[:80]))
        except ValueError:
            pass
tot = sum(x[0] for x in lines) or 1
print(f"total samples {tot}")
for a, ni, ex, loc, src in sorted(lines, reverse=True)[:n]:
    print(f"{100 * a / tot:5.1f}% (not-issued {100 * ni / tot:5.1f}%) {ex:>10d}  {loc:18s} {src}")
