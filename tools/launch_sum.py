"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_sum.py gpurun_out/launches.csv [top]"""
import csv, sys
from collections import defaultdict
lines = open(sys.argv[1]).read().splitlines()
k = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[k:]))
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
t = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    n = r[ik].split('(')[0][:60]
    t[n][0] += 1
    t[n][1] += float(r[iv].replace(",", "")) / 1e6
for n, (c, ms) in sorted(t.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{ms:9.3f} ms {c:4d} launches  {n}")
