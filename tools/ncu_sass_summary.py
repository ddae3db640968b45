"""Summarise an ncu source page (SASS) : top stall lines and opcode mix.
usage: python tools/ncu_sass_summary.py report.ncu-rep [kernel-regex] [launch-index]"""
import csv, io, re, subprocess, sys
from collections import Counter, defaultdict

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
blocks = re.split(r'^"Kernel Name",', txt, flags=re.M)
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if not re.search(kre, name):
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    hdr = rows[0]
    ia, isrc, ist, iex = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                  "Instructions Executed"))
    tot_s = sum(int(r[ist] or 0) for r in rows[1:])
    tot_i = sum(int(r[iex] or 0) for r in rows[1:])
    print(f"== {name[:90]}  samples={tot_s} warp-inst={tot_i:.3e}")
    ops = Counter(); opsamp = Counter()
    for r in rows[1:]:
        op = r[isrc].strip().split()[0] if r[isrc].strip() else "?"
        if op.startswith("@"):
            op = r[isrc].strip().split()[1]
        op = op.split(".")[0]
        ops[op] += int(r[iex] or 0); opsamp[op] += int(r[ist] or 0)
    print("opcode mix (warp-inst %, stall-sample %):")
    for op, n in ops.most_common(25):
        print(f"  {op:10s} {100*n/tot_i:5.1f}%  {100*opsamp[op]/max(tot_s,1):5.1f}%")
    top = sorted(rows[1:], key=lambda r: -int(r[ist] or 0))[:25]
    print("top stall instructions:")
    for r in top:
        print(f"  {r[ia][-5:]} {int(r[ist]):7d} {int(r[iex]):10d}  {r[isrc].strip()[:70]}")
    break
