"""Executed FP32 work of the pass kernels from ncu source counters (SASS view).

usage: python profiles/ncu_fp32.py REPORT.ncu-rep CFG ROWS_PER_LAUNCH [--json profiles/ncu_fp32.json]

Per kernel: flops = 32 lanes x sum over SASS instructions of executed warp instructions x flops
per lane (FFMA2 4, FMUL2/FADD2 2, FFMA 2, FMUL/FADD 1), divided by the rows of the launch ->
flops per row, the deterministic unit bench.py multiplies by its own rows and divides by its
own CUDA-event launch times (the FP32-pipe view of the roofline)."""
import csv
import io
import json
import subprocess
import sys

FLOPS = {"FFMA2": 4, "FMUL2": 2, "FADD2": 2, "FFMA": 2, "FMUL": 1, "FADD": 1}


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", "gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ik, it = hdr.index("Kernel Name"), hdr.index("gpu__time_duration.sum")
    unit = rows[1][it]
    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1e-9)
    return [(r[ik], float(r[it]) * scale) for r in rows[2:]]


def flops_of(rep, name, launch_idx):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", name, "--launch-skip", str(launch_idx), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    tot = 0.0
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[ix].split():
            continue
        t = r[ix].split()
        op = t[1] if t[0].startswith("@") else t[0]
        base = op.split(".")[0]
        key = base + ("2" if "F32x2" in r[ix] and not base.endswith("2") else "")
        tot += FLOPS.get(key, 0) * 32 * float(r[iex] or 0)
    return tot


def main():
    rep, cfg, rows = sys.argv[1], sys.argv[2], int(sys.argv[3])
    out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    seen = {}
    res = {}
    for name, dur in kernels(rep):
        k = seen.get(name, 0)
        seen[name] = k + 1
        if k:
            continue
        f = flops_of(rep, name, 0)
        res[f"cfg{cfg}|{name}"] = {"flops_per_row": f / rows, "ncu_tflops": f / dur / 1e12, "ncu_us": dur * 1e6}
        print(f"{name:16s} {dur * 1e6:9.1f} us  {f / dur / 1e12:6.1f} TFLOP/s  {f / rows / 1e9:.3f} GFLOP/row")
    if out:
        try:
            cur = json.load(open(out))
        except Exception:
            cur = {}
        cur.update(res)
        json.dump(cur, open(out, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
