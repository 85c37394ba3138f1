"""Top SASS lines by warp-stall samples from an ncu report: python tools/ncu_hot.py rep.ncu-rep [n]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
data = []
for r in rows[1:]:
    try:
        data.append((float(r[si]), int(float(r[ie] or 0)), r[0], r[1]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for v, ex, a, s in sorted(data, key=lambda x: -x[0])[:n]:
    print(f"{100 * v / tot:5.1f}%  exec={ex:8d}  {a[-5:]}  {s.strip()[:100]}")
