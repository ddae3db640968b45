"""Per-CUDA-source-line instructions executed and stall samples of an ncu report
(source page, cuda+sass correlation).  usage: python tools/ncu_cuda_lines.py rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
res = []
fname = "?"
h = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        h = r; ist = h.index("Warp Stall Sampling (All Samples)"); iex = h.index("Instructions Executed")
        continue
    if h and r and r[0].isdigit() and r[2] == "-":
        s = int(r[ist] or 0); e = int(r[iex] or 0)
        if s or e:
            res.append((e, s, fname, int(r[0]), r[1].strip()[:78]))
te = sum(x[0] for x in res); ts = sum(x[1] for x in res)
print(f"total warp-inst {te:.3e}, stall samples {ts}")
for e, s, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100*e/te:5.1f}% inst {100*s/max(ts,1):5.1f}% stall  {f}:{ln:4d}  {src}")
