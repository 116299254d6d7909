"""Per-kernel table of an `ncu --metrics gpu__time_duration.sum --csv` launch list (last step).
usage: python profiles/launch_table.py launches.csv [marker-kernel]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else "k_group_table"
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
data = []
for r in rows[1:]:
    if len(r) <= vi or r[0] == "ID":
        continue
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
    data.append((r[ki], float(r[vi].replace(",", "")) * scale))
idx = [i for i, (k, v) in enumerate(data) if marker in k]
last = data[idx[-1]:] if idx else data
tot = sum(v for _, v in last)
print(f"launches in last step: {len(last)}, kernel time {tot:.1f} us")
agg, cnt = defaultdict(float), defaultdict(int)
for k, v in last:
    kk = k.split("(")[0].replace("void ", "")[:48]
    agg[kk] += v
    cnt[kk] += 1
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k:50s} n={cnt[k]:3d} {v:9.1f} us  {100 * v / tot:5.1f}%")
