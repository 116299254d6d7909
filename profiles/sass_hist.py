"""Per-opcode histogram of an ncu source page (SASS view): executed warp instructions and
warp-stall samples per opcode. usage: ncu -i REP --page source --csv --print-source sass -k K
> x.csv; python profiles/sass_hist.py x.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix, iss, iex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ex = collections.Counter()
st = collections.Counter()
why = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[ix].split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0] + ("2" if ".F32x2" in r[ix] or "F32x2" in r[ix] else "")
    ex[o] += int(r[iex] or 0)
    st[o] += int(r[iss] or 0)
    for i, h in stall_cols:
        v = int(r[i] or 0)
        if v:
            why[o][h[6:]] += v
tex, tst = sum(ex.values()), sum(st.values())
print(f"{'op':10s} {'exec%':>7s} {'stall%':>7s}  top stalls")
for o, v in ex.most_common(30):
    tops = ", ".join(f"{k}:{100 * c / tst:.1f}" for k, c in why[o].most_common(3))
    print(f"{o:10s} {100 * v / tex:7.2f} {100 * st[o] / tst:7.2f}  {tops}")
