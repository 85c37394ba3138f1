"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list.
Usage: python tools/launch_summary.py launches.csv [fraction_to_skip]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
data = [r for r in rows[1:] if len(r) > vi]
skip = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
data = data[int(len(data) * skip):]
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    name = r[ki].split("(")[0]
    name = name.replace("rn::", "").replace("(anonymous namespace)::", "")[:70]
    v = float(r[vi].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
print(f"launches {len(data)}  total {s / 1e3:.1f} us (ncu: serialised, cold-cache)")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:30]:
    print(f"{v / 1e3:9.1f} us {100 * v / s:5.1f}% {cnt[k]:4d}  {k}")
