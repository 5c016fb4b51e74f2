"""Key metrics of an ncu report's details page: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEEP = ["Duration", "Elapsed Cycles", "SM Active Cycles", "SM Frequency", "DRAM Throughput",
        "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Avg. Active Threads Per Warp", "Achieved Active Warps Per SM", "Theoretical Occupancy",
        "Executed Instructions", "Registers Per Thread", "No Eligible",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block", "Block Size",
        "Grid Size", "Local Memory Spilling"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
mi, ui, vi, ki = (h.index(c) for c in ("Metric Name", "Metric Unit", "Metric Value", "Kernel Name"))
for row in rows[1:]:
    if any(row[mi].startswith(k) for k in KEEP):
        print(f"{row[ki][:30]:30s} {row[mi][:42]:42s} {row[ui]:10s} {row[vi]}")
