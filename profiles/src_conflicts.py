"""Shared-memory bank conflicts and stall samples per SASS instruction from an ncu source page
(SASS view). usage: python profiles/src_conflicts.py SRC.csv[.gz] [N]"""
import csv
import gzip
import io
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
c = {h: i for i, h in enumerate(hdr)}
recs = []
tot_ex = tot_wf = tot_samp = 0
for idx, r in enumerate(rows[2:]):
    if len(r) < len(hdr):
        continue
    num = lambda k: float(r[c[k]] or 0) if r[c[k]] not in ("-", "") else 0.0  # noqa: E731
    ex, wf, samp = num("L1 Wavefronts Shared Excessive"), num("L1 Wavefronts Shared"), num("Warp Stall Sampling (All Samples)")
    tot_ex += ex
    tot_wf += wf
    tot_samp += samp
    recs.append((ex, wf, samp, idx, r[c["Source"]].strip()))
print(f"shared wavefronts {tot_wf:.3e}, excessive {tot_ex:.3e} ({100 * tot_ex / max(tot_wf, 1):.1f}%), stall samples {tot_samp:.0f}")
print("top excessive-wavefront instructions:")
for ex, wf, samp, idx, src in sorted(recs, reverse=True)[:n]:
    if ex <= 0:
        break
    print(f"  #{idx:5d} excess {ex:10.0f} of {wf:10.0f}  samples {samp:6.0f}  {src}")
