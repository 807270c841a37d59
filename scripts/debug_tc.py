"""Inspect the tcgen05 path's workspace (row-stage output) against torch fp32."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_12271_b200 as pk  # noqa: E402
from paper_2602_12271_b200 import _lib, ops  # noqa: E402

dev = torch.device("cuda", 0)
torch.manual_seed(0)
f, h, w, d = int(sys.argv[1]) if len(sys.argv) > 1 else 3, 30, 52, 128
shape = pk.VideoShape(f, h, w)
plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), (1, h, w))
low = pk.lower_square(plan)
q, k, v = (torch.randn(1, 1, shape.n, d, device=dev, dtype=torch.bfloat16) for _ in range(3))
ws = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
print("path", ops.selected_path(q, k, v, low))
out = ops.forward(q, k, v, low, workspace=ws)
torch.cuda.synchronize()
gq = gk = f
s1, s2 = h, w
nkeys = gk * s1
rows = gq * s2 * nkeys
W = ws[: rows * 512].view(torch.bfloat16).view(gq, s2, nkeys, 256).float()
off = (rows * 512 + 255) // 256 * 256
Wc = ws[off: off + rows * 4].view(torch.float32).view(gq, s2, nkeys)

scale = d ** -0.5
Q = (q[0, 0].float() * scale).view(gq, s1, s2, d)
K = k[0, 0].float().view(gk, s1, s2, d)
V = v[0, 0].float().view(gk, s1, s2, d)
z = torch.einsum("akjd,ckid->ackji", Q, K)
R = torch.softmax(z, -1)
aL = torch.einsum("ackji,ckid->ajckd", R, K).reshape(gq, s2, nkeys, d)
Y = torch.einsum("ackji,ckid->ajckd", R, V).reshape(gq, s2, nkeys, d)
cL = (R * torch.log(R)).sum(-1).permute(0, 3, 1, 2).reshape(gq, s2, nkeys)


def rel(x, y):
    return float((x - y).norm() / y.norm())


print("aL rel", rel(W[..., :128], aL), "Y rel", rel(W[..., 128:], Y), "cL rel", rel(Wc, cL))
print("aL sample", W[0, 0, 0, :4].tolist(), aL[0, 0, 0, :4].tolist())
print("Y sample", W[0, 0, 0, 128:132].tolist(), Y[0, 0, 0, :4].tolist())
print("cL sample", Wc[0, 0, :4].tolist(), cL[0, 0, :4].tolist())
# per (a, j) error map of aL
err = (W[..., :128] - aL).norm(dim=-1) / aL.norm(dim=-1)
print("aL err by a", err.mean(dim=(1, 2)).tolist())
print("aL err by j (first 8, last 4)", err.mean(dim=(0, 2))[:8].tolist(), err.mean(dim=(0, 2))[-4:].tolist())
print("aL err by key (first 4)", err.mean(dim=(0, 1))[:4].tolist())
# column stage given the device W
S = torch.einsum("aljd,ajkd->ajlk", Q, W[..., :128]) - Wc[:, :, None, :]
L = torch.softmax(S, -1)
O = torch.einsum("ajlk,ajkd->aljd", L, W[..., 128:]).reshape(-1, d)
print("out vs column-stage(W_device) rel", rel(out[0, 0].float(), O))
S = torch.einsum("aljd,ajkd->ajlk", Q, aL) - cL[:, :, None, :]
L = torch.softmax(S, -1)
Oref = torch.einsum("ajlk,ajkd->aljd", L, Y).reshape(-1, d)
print("out vs full ref rel", rel(out[0, 0].float(), Oref))
