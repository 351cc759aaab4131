"""Key counters of one ncu --set full report: python scripts/ncu_summary.py X.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Block Limit Registers", "Block Limit Shared Mem", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "Warp Cycles Per Issued Instruction",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    R = list(csv.reader(io.StringIO(out)))
    h = R[0]
    print(f"== {path}: {R[1][h.index('Kernel Name')][:80]}")
    seen = set()
    for r in R[1:]:
        n = r[h.index("Metric Name")]
        if n in KEYS and n not in seen:
            seen.add(n)
            print(f"  {n:40s} {r[h.index('Metric Value')]} {r[h.index('Metric Unit')]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    R = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = R[0], R[1], R[2]
    want = ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio",
            "smsp__inst_executed.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w[:78]:78s} {vals[i]} {units[i]}")
