"""Summarise an ncu source-page CSV (--page source --print-source sass): top
instructions by warp-stall samples with their dominant stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
agg = {h: 0 for h in stall_cols}
for r in data:
    for h in stall_cols:
        agg[h] += int(r[idx[h]] or 0)
print("by reason:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:10])
top = sorted(data, key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for r in top:
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    reasons = sorted(((int(r[idx[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:3]
    print(f"{r[0][-5:]} {s:6d} {100*s/tot:5.1f}%  {r[1].strip()[:60]:60s} {reasons}")
