"""Export ncu evidence into profiles/ (tracked):

  python tools/ncu_export.py <round-tag> [gpurun_out] [out dir, default profiles/]

writes
  profiles/<tag>_launches.csv        kernel, grid, block, duration_ns (one row per launch)
  profiles/<tag>_launch_shares.md    per-kernel totals and share of the profiled run
  profiles/<tag>_<kernel>_full.txt   SOL/occupancy/stall summary + SASS opcode mix +
                                     top stall instructions of each full capture
  profiles/<tag>_traffic.json        dram bytes read+write per launch of each captured kernel
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "profiles")
os.makedirs(out, exist_ok=True)


def short(name):
    m = re.search(r"(k\d+\w*?)(?:<|\(|$)", name)
    if "pf::" in name and m:
        return m.group(1)
    return re.sub(r"\(.*", "", name)[:60]


# ---- launch list ----------------------------------------------------------
lp = os.path.join(src, "launches.csv")
if os.path.exists(lp):
    lines = open(lp).read().splitlines()
    k = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[k:]))
    h = rows[0]
    ik, ig, ib, iv = (h.index(x) for x in ("Kernel Name", "Grid Size", "Block Size", "Metric Value"))
    tot = defaultdict(lambda: [0, 0.0])
    with open(os.path.join(out, f"{tag}_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["launch", "kernel", "grid", "block", "duration_ns"])
        for n, r in enumerate(rows[1:]):
            kn = short(r[ik])
            d = float(r[iv])
            w.writerow([n, kn, r[ig], r[ib], int(d)])
            tot[kn][0] += 1
            tot[kn][1] += d
    allns = sum(v[1] for v in tot.values())
    pf = {k: v for k, v in tot.items() if k.startswith("k")}
    pfns = sum(v[1] for v in pf.values())
    with open(os.path.join(out, f"{tag}_launch_shares.md"), "w") as f:
        f.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
        f.write("Command: `ncu --metrics gpu__time_duration.sum --clock-control none python bench.py "
                "--steps 2 --warmup 1 --no-e2e --no-cpu` (cold-cache, serialised launches: "
                "compare shares, not absolutes).\n\n")
        f.write("| kernel | launches | total ms | mean us | share of libpowerfoam time |\n|---|---|---|---|---|\n")
        for kn, (c, d) in sorted(pf.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {kn} | {c} | {d / 1e6:.3f} | {d / c / 1e3:.1f} | {100 * d / pfns:.1f}% |\n")
        f.write(f"\nOther (torch) kernels: {(allns - pfns) / 1e6:.3f} ms of {allns / 1e6:.3f} ms.\n")

# ---- full captures --------------------------------------------------------
WANT = ["Duration", "Elapsed Cycles", "SM Active Cycles", "Compute (SM) Throughput",
        "Memory Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Avg. Not Predicated Off Threads Per Warp"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "smsp__thread_inst_executed_per_inst_executed.ratio",
       "smsp__inst_executed.sum", "sm__inst_executed.sum.pct_of_peak_sustained_elapsed",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum"]
traffic = OrderedDict()
workloads = {}
for rep in sorted(f for f in os.listdir(src) if f.startswith("prof_") and f.endswith(".ncu-rep")):
    path = os.path.join(src, rep)
    name = rep[5:-8]
    if "@" in name:                     # prof_<kernel>@<workload>.ncu-rep
        name, wl = name.split("@", 1)
        workloads[name] = wl
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    sass = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_sass_summary.py"), path],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    lines = [f"# {tag}: ncu --set full capture `{rep}`", ""]
    if rows:
        h = rows[0]
        ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                               "Metric Unit"))
        kname = rows[1][ki] if len(rows) > 1 else "?"
        lines.append(f"kernel: {kname}")
        seen = set()
        for r in rows[1:]:
            if r[mi] in WANT and r[mi] not in seen:
                seen.add(r[mi])
                lines.append(f"  {r[mi]:45s} {r[vi]:>14s} {r[ui]}")
    rr = list(csv.reader(io.StringIO(raw)))
    vals = {}
    if len(rr) > 2:
        h = rr[0]
        lines.append("")
        lines.append("raw metrics:")
        for m in RAW:
            if m in h:
                i = h.index(m)
                lines.append(f"  {m:62s} {rr[2][i]:>14s} {rr[1][i]}")
                vals[m] = (rr[2][i], rr[1][i])
    lines.append("")
    lines.append(sass)
    open(os.path.join(out, f"{tag}_{name}_full.txt"), "w").write("\n".join(lines) + "\n")

    def tobytes(v):
        x, unit = float(v[0].replace(",", "")), v[1]
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)

    if "dram__bytes_read.sum" in vals:
        traffic[name] = {"dram_read_bytes": tobytes(vals["dram__bytes_read.sum"]),
                         "dram_write_bytes": tobytes(vals["dram__bytes_write.sum"]),
                         "source": f"profiles/{tag}_{name}_full.txt (ncu --set full, 1 launch)",
                         # the bench workload tag of the capture (bench.py matches on it);
                         # prof_<kernel>[@<workload>].ncu-rep, default the bench default
                         "workload": workloads.get(name, "train8_1m")}
        traffic[name]["traffic_bytes"] = (traffic[name]["dram_read_bytes"]
                                          + traffic[name]["dram_write_bytes"])
        if "smsp__inst_executed.sum" in vals:
            traffic[name]["warp_inst"] = float(vals["smsp__inst_executed.sum"][0].replace(",", ""))
        if "sm__inst_executed.sum.pct_of_peak_sustained_elapsed" in vals:
            traffic[name]["issue_pct_of_peak"] = float(
                vals["sm__inst_executed.sum.pct_of_peak_sustained_elapsed"][0].replace(",", ""))
json.dump(traffic, open(os.path.join(out, f"{tag}_traffic.json"), "w"), indent=1)
print("wrote", sorted(os.listdir(out)))
