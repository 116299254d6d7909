"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum, from an
`ncu --set full` capture) per JIT kernel family, recorded for bench.py's roofline "traffic".
usage: python profiles/ncu_traffic.py REPORT.ncu-rep WORKLOAD_NAME M [ROWS_SCALE] [ROWS]
ROWS_SCALE rescales the captured bytes (default 1); ROWS = rows per launch of the capture, recorded
as "<workload>|rows" so bench.py scales the figure to its own rows per launch (micro-batches)."""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402

rep, workload, M = sys.argv[1], sys.argv[2], int(sys.argv[3])
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
cap_rows = int(sys.argv[5]) if len(sys.argv) > 5 else None
names = {0: "forward", 1: "turnaround", 2: "adjoint"}
fam: dict = {}
for k in load(rep):
    m = re.match(r"lsq_jit_p(\d+)_m(\d)", k["kernel"])
    if not m:
        continue
    mode = int(m.group(2))
    label = "lsq_jit_p*_m%d (%s, M=%d)" % (mode, names[mode], M)
    fam.setdefault(label, []).append((k["dram_read"] + k["dram_write"]) * scale)
out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
data = json.load(open(out_path)) if os.path.exists(out_path) else {}
for label, v in fam.items():
    data[f"{workload}|{label}"] = round(sum(v) / len(v))
    print(workload, label, len(v), "launches, mean bytes/launch", round(sum(v) / len(v)))
if cap_rows:
    data[f"{workload}|rows"] = cap_rows
json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
