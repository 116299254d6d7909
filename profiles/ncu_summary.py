"""Summarise an ncu report: per kernel duration, DRAM bytes/throughput, pipe utilisation,
occupancy, top stall reasons. usage: python profiles/ncu_summary.py REPORT.ncu-rep [--json OUT]"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "shared_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        stalls = {}
        for i, h in enumerate(hdr):
            v = row[i].replace(",", "")
            if h in KEYS:
                try:
                    d[KEYS[h]] = float(v)
                except ValueError:
                    pass
                if KEYS[h] in ("dram_read", "dram_write"):
                    u = units[i]
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    d[KEYS[h]] = float(v) * scale
                if KEYS[h] == "duration_us":
                    u = units[i]
                    d[KEYS[h]] = float(v) * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
            m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", h)
            if m:
                try:
                    stalls[m.group(1)] = float(v)
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        d["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
        if "dram_read" in d and "duration_us" in d:
            d["dram_GBps"] = round((d["dram_read"] + d.get("dram_write", 0)) / (d["duration_us"] * 1e-6) / 1e9, 1)
        res.append(d)
    return res


if __name__ == "__main__":
    res = load(sys.argv[1])
    for d in res:
        print(json.dumps(d))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)
