"""Markdown table of the GPU parity log pytest writes to $LSQ_PARITY_OUT (tests/conftest.py).
usage: python profiles/parity_table.py profiles/r02/parity_<tag>.json > profiles/r02/parity_table.md"""
import json
import os
import sys

path = sys.argv[1]
rows = json.load(open(path))
print(f"# GPU parity table (round 2, `pytest -m gpu` on one B200, {os.path.relpath(path)})\n")
print("A2 = worst |g - g_ref| / max(|g_ref|, 1e-2 * max|g_ref|) over the compared array of angle gradients\n"
      "(per-row trainable + encoding gradients; `_sum` = the batch-summed loss gradient). Per-row floor =\n"
      "the same with 1e-2 * each row's own max (recorded, not asserted: below the complex64 floor, DESIGN §4).\n"
      "Normwise = max|dg| / max|g_ref|. <Z_q> errors are absolute.\n")
print("| test | compared | worst A2 | per-row-floor A2 | normwise | bound |")
print("|---|---|---|---|---|---|")
zq = []
for r in rows:
    if "a2_rel" in r:
        prf = r.get("a2_rel_per_row_floor")
        print(f"| {r['test']} | {r['what']} | {r['a2_rel']:.2e} | {'' if prf is None else f'{prf:.2e}'} | "
              f"{r.get('normwise', float('nan')):.2e} | {r['tol']:.1e} |")
    else:
        zq.append(r)
print("\n| test | compared | worst abs error | bound |")
print("|---|---|---|---|")
for r in zq:
    print(f"| {r['test']} | {r['what']} | {r['abs']:.2e} | {r['tol']:.1e} |")
a2 = [r["a2_rel"] / r["tol"] for r in rows if "a2_rel" in r]
ab = [r["abs"] / r["tol"] for r in zq]
print(f"\n{len(rows)} checks; worst gradient error at {100 * max(a2):.0f}% of its bound, worst <Z> / value error at "
      f"{100 * max(ab):.1f}% of its bound.")
