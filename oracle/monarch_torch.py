"""Differentiable float64 torch restatement of the tiled MonarchAttention forward
-- TEST INFRASTRUCTURE ONLY (the backward pass's oracle).

Same algorithm, notation and index order as ``oracle/monarch_oracle.py``
(``tiled_forward``, which is pinned to the unmodified reference's golden
vectors): the reference package has no backward pass (SPEC.md:8 puts it out of
scope; the paper's finetuning backward is PAPER.md:135-136, 644), so gradients
of q, k, v are those of this restatement computed by torch autograd in float64.
``tests/test_backward_oracle.py`` checks that its forward equals the numpy
oracle to 1e-12 on the golden cases, and that its gradients pass
``torch.autograd.gradcheck``.  Only ``tests/`` may import this module.

Reference lines followed (solver.py of /root/reference/pkg/src/monarchbench):
scale applied to q before the solver (:104), identity L init (:180), R update
(:187-189), c_L = sum R log R (:191, evaluated as sum R z - lse), joint L
softmax over all key tiles (:193-195), alpha_R / c_R hand-off (:185-186),
Y = R V and O = L Y (factors.py:123-124).
"""

from __future__ import annotations

import torch


def tiled_forward_torch(qs, ks, vs, c1q, c1k, c2, s1, s2, iterations=1, eps_div=1e-30):
    """Differentiable counterpart of monarch_oracle.tiled_forward on slot-ordered,
    already-scaled inputs; returns (L', R', O) in the same layouts."""
    d = qs.shape[1]
    dv = vs.shape[1]
    gq, gk = c1q * c2, c1k * c2
    qt = qs.reshape(c1q, s1, c2, s2, d).permute(0, 2, 1, 3, 4).reshape(gq, s1, s2, d)
    kt = ks.reshape(c1k, s1, c2, s2, d).permute(0, 2, 1, 3, 4).reshape(gk, s1, s2, d)
    vt = vs.reshape(c1k, s1, c2, s2, dv).permute(0, 2, 1, 3, 4).reshape(gk, s1, s2, dv)
    alpha_r = qt[:, None].expand(gq, gk, s1, s2, d)
    c_r = torch.ones((gq, gk, s1, s2), dtype=qs.dtype, device=qs.device)
    R = L = None
    for _ in range(iterations):
        beta = torch.matmul(alpha_r, kt.transpose(-1, -2)[None])             # (gq,gk,s1,s2,s2)
        z = beta / torch.clamp(c_r, min=eps_div)[..., None]
        lse = torch.logsumexp(z, dim=-1)
        R = torch.softmax(z, dim=-1)
        alpha_l = torch.matmul(R, kt[None])                                   # (gq,gk,s1,s2,d)
        ent = (R * z).sum(-1) - lse                                           # = sum R log R
        qcol = qt.permute(0, 2, 1, 3)                                         # (gq, s2, s1, d)
        acol = alpha_l.permute(0, 3, 1, 2, 4).reshape(gq, s2, gk * s1, d)
        ccol = ent.permute(0, 3, 1, 2).reshape(gq, s2, gk * s1)
        S = torch.matmul(qcol, acol.transpose(-1, -2)) - ccol[:, :, None, :]
        P = torch.softmax(S, dim=-1)                                          # (gq, s2, s1, gk*s1)
        L = P
        Pk = P.reshape(gq, s2, s1, gk, s1)
        alpha_r = torch.einsum("ajlck,aljv->ackjv", Pk, qt)
        c_r = Pk.sum(dim=2).permute(0, 2, 3, 1)
    Y = torch.matmul(R, vt[None])
    ycol = Y.permute(0, 3, 1, 2, 4).reshape(gq, s2, gk * s1, dv)
    O = torch.matmul(L, ycol)
    O = O.reshape(c1q, c2, s2, s1, dv).permute(0, 3, 1, 2, 4).reshape(-1, dv)
    Rf = R.reshape(c1q, c2, c1k, c2, s1, s2, s2)
    Lf = L.reshape(c1q, c2, s2, s1, c1k, c2, s1).permute(0, 1, 4, 5, 2, 3, 6)
    return Lf, Rf, O


def forward_phi_torch(q, k, v, order_q, order_k, c1q, c1k, c2, s1, s2, iterations=1, scale=None):
    """Row-major (phi order) in and out, like monarch_oracle.forward_phi; differentiable."""
    if scale is None:
        scale = 1.0 / q.shape[1] ** 0.5
    oq = torch.as_tensor(order_q, dtype=torch.long, device=q.device)
    ok = torch.as_tensor(order_k, dtype=torch.long, device=q.device)
    _, _, Oo = tiled_forward_torch((q * scale)[oq], k[ok], v[ok], c1q, c1k, c2, s1, s2, iterations)
    out = torch.empty_like(Oo)
    out = out.index_copy(0, oq, Oo)
    return out


def grads(q, k, v, dout, order_q, order_k, c1q, c1k, c2, s1, s2, iterations=1, scale=None):
    """(dq, dk, dv) of sum(out * dout) in float64."""
    q, k, v = (torch.as_tensor(x, dtype=torch.float64).clone().requires_grad_(True) for x in (q, k, v))
    out = forward_phi_torch(q, k, v, order_q, order_k, c1q, c1k, c2, s1, s2, iterations, scale)
    out.backward(torch.as_tensor(dout, dtype=torch.float64))
    return q.grad.detach(), k.grad.detach(), v.grad.detach()
