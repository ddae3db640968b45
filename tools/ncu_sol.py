"""Key SOL / occupancy / stall metrics from an ncu report (details page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
ki, si, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Section Name", "Metric Name", "Metric Value", "Metric Unit"))
want = {"Duration", "Elapsed Cycles", "SM Active Cycles", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Avg. Not Predicated Off Threads Per Warp", "Block Limit Registers", "Block Limit Shared Mem"}
seen = set()
for r in rows[1:]:
    if r[mi] in want and (r[ki], r[mi]) not in seen:
        seen.add((r[ki], r[mi]))
        print(f"{r[ki][:24]:24s} {r[mi]:42s} {r[vi]:>14s} {r[ui]}")
