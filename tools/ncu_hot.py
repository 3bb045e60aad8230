"""Summarise an ncu --page source --csv --print-source sass dump: top instructions by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ci = hdr.index("Warp Stall Sampling (All Samples)")
si = hdr.index("Source")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[ci] or 0) for r in data)
print("total samples", tot)
agg = {}
for r in data:
    for i in stall_cols:
        agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
print(sorted(((round(v / tot * 100, 1), k) for k, v in agg.items() if v), reverse=True)[:10])
top = sorted(data, key=lambda r: -float(r[ci] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    st = sorted(((float(r[i] or 0), hdr[i]) for i in stall_cols), reverse=True)[:2]
    print(f"{float(r[ci] or 0) / tot * 100:5.1f}%  {r[0]:>6} {r[si][:70]:70s} {st}")
