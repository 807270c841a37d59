"""Split an ncu source-page CSV (sass) into regions bounded by marker opcodes and
sum the stall samples per region: python ncu_regions.py src.csv [window]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = rows[2:]
tot = sum(int(r[idx[S]] or 0) for r in data)
ex = [i for i, r in enumerate(data) if "MUFU.EX2" in r[1]]
lo, hi = ex[0], ex[-1]
w = int(sys.argv[2]) if len(sys.argv) > 2 else 200
def agg(a, b):
    s = sum(int(r[idx[S]] or 0) for r in data[a:b])
    rs = {h[6:]: sum(int(r[idx[h]] or 0) for r in data[a:b]) for h in stall_cols}
    n = b - a
    return s, n, sorted(((v, k) for k, v in rs.items() if v), reverse=True)[:6]
print("total", tot, "instructions", len(data))
for name, a, b in (("before-softmax", max(0, lo - w), lo), ("ex2 span", lo, hi + 1), ("after", hi + 1, min(len(data), hi + 1 + w))):
    s, n, rs = agg(a, b)
    print(f"{name:15s} [{a},{b}) n={n} samples={s} ({100*s/tot:.1f}%) {rs}")
