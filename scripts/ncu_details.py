"""Print the key --page details metrics of every launch in an .ncu-rep."""
import csv
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Issue Slots Busy", "Executed Ipc Active",
        "Registers Per Thread", "Achieved Occupancy", "Dynamic Shared Memory Per Block",
        "Warp Cycles Per Issued Instruction", "No Eligible")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ii, ki, mi, ui, vi = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"),
                      h.index("Metric Unit"), h.index("Metric Value"))
cur = None
for r in rows[1:]:
    if len(r) <= vi:
        continue
    if r[ii] != cur:
        cur = r[ii]
        print(f"== launch {cur}: {r[ki][:80]}")
    if r[mi] in KEYS:
        print(f"   {r[mi]:40s} {r[vi]:>12s} {r[ui]}")
