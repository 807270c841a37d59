"""Debug T=2 on the tcgen05 path: compare the hand-off tensor hat_alpha_R and the
column statistics in the workspace with the oracle (1 head, SF shape)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2602_12271_b200 as pk  # noqa: E402
from paper_2602_12271_b200 import ops  # noqa: E402
from oracle import monarch_oracle as orc  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device="cpu").manual_seed(2)
f, h, w, d = 3, 30, 52, 128
q, k, v = (torch.randn(1, 1, f * h * w, d, generator=g).to(dev, torch.bfloat16) for _ in range(3))
s = pk.VideoShape(f, h, w)
plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, h, w))
low = pk.lower_square(plan)
ws = torch.zeros(1 << 28, dtype=torch.uint8, device=dev)
out = ops.forward(q, k, v, low, 2, workspace=ws)
torch.cuda.synchronize()
gq, gk, s1, s2 = 3, 3, 30, 52
nkeys = gk * s1
ncols = gq * s2
rows = ncols * nkeys
al = lambda x: (x + 255) // 256 * 256
ckey = (nkeys + 31) // 32 * 32
off_wc = al(rows * 512)
off_cnt = off_wc + al(ncols * ckey * 4)
off_ar = off_cnt + al(1 * 4)
off_st = off_ar + al(rows * 256)
wsh = ws.cpu().numpy()
AR = torch.from_numpy(wsh[off_ar:off_ar + rows * 256].copy()).view(torch.bfloat16).float().numpy()
AR = AR.reshape(gq, nkeys, s2, d)
ST = wsh[off_st:off_st + ncols * 64 * 4].view(np.float32).reshape(ncols, 64)
# oracle iteration 0
scale = 1 / np.sqrt(d)
qn, kn, vn = (x[0, 0].float().cpu().numpy().astype(np.float64) for x in (q, k, v))
qs = qn * scale
qt = qs.reshape(gq, s1, s2, d)
kt = kn.reshape(gk, s1, s2, d)
beta = np.matmul(np.broadcast_to(qt[:, None], (gq, gk, s1, s2, d)), np.swapaxes(kt, -1, -2)[None])
R = orc._softmax_last(beta)
alpha_l = np.matmul(R, kt[None])
ent = (R * np.log(np.maximum(R, 1e-300))).sum(-1)
qcol = qt.transpose(0, 2, 1, 3)
acol = alpha_l.transpose(0, 3, 1, 2, 4).reshape(gq, s2, gk * s1, d)
ccol = ent.transpose(0, 3, 1, 2).reshape(gq, s2, gk * s1)
S = np.matmul(qcol, np.swapaxes(acol, -1, -2)) - ccol[:, :, None, :]
P = orc._softmax_last(S)
Pk = P.reshape(gq, s2, s1, gk, s1)
alpha_r = np.einsum("ajlck,aljv->ackjv", Pk, qt)
c_r = Pk.sum(axis=2).transpose(0, 2, 3, 1)
ahat = alpha_r / c_r[..., None]                  # (gq, gk, s1, s2, d), scaled units
ahat_ws = AR.reshape(gq, gk, s1, s2, d) * scale  # workspace is in unscaled Q units
print("hat_alpha_R rel_l2", orc.rel_l2(ahat_ws, ahat))
print(" sample ws", ahat_ws[0, 0, 0, 0, :4], "oracle", ahat[0, 0, 0, 0, :4])
print(" per (a,c) rel", [[round(orc.rel_l2(ahat_ws[a, c], ahat[a, c]), 4) for c in range(gk)] for a in range(gq)])
# statistics: L row sums from m, 1/sum (log2 units): check sum_k 2^(x - m) * inv = 1 using oracle S
log2e = 1.4426950408889634
Sx = S * log2e                                   # x = S log2e  (S already includes scale and -c_L)
col = 0
m, inv = ST[col, :32], ST[col, 32:]
tot = (np.exp2(Sx[0, 0, :s1, :] - m[:s1, None]) * inv[:s1, None]).sum(-1)
print("stats: row sums with oracle logits (should be ~1):", tot[:6])
ref = orc.forward_phi(qn, kn, vn, np.arange(f * h * w), np.arange(f * h * w), 3, 3, 1, s1, s2, 2)[2]
print("out rel_l2 T=2", orc.rel_l2(out[0, 0].float().cpu().numpy(), ref))
for col in (0, 52, 104, 130):
    a, j = col // s2, col % s2
    m, inv = ST[col, :32], ST[col, 32:]
    tot = (np.exp2(Sx[a, j, :s1, :] - m[:s1, None]) * inv[:s1, None]).sum(-1)
    print("stats col", col, "a", a, "row sums", np.round(tot[:4], 4), "m", m[:3], "inv", inv[:3])
e = np.abs(ahat_ws[2] - ahat[2]).mean(-1)     # (gk, s1, s2)
print("a=2 err by j (k=0,c=0):", np.round(e[0, 0, :10], 4))
print("a=2 err by k (j=0,c=0):", np.round(e[0, :10, 0], 4))
e2 = np.abs(ahat_ws[2] - ahat[2]).mean(-1)   # (gk, s1, s2)
bad = np.argwhere(e2 > 1e-3)
print("a=2 bad count", len(bad), "of", e2.size, "first", bad[:8].tolist())
print("by j:", np.round(e2.mean(axis=(0, 1)), 4))
