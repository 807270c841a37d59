"""CPU oracle for the tiled MonarchAttention forward — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The shipped operator
(``paper_2602_12271_b200``) never calls into ``oracle/`` and fails loudly when
its CUDA library is missing.

It restates, in float64 numpy, the algorithm of the reference package
``monarchbench`` (/root/reference/pkg/src/monarchbench) in the *kernel
oriented* form the CUDA path uses: a row stage per
(query tile, key tile, in-tile row) and a column stage per (query tile,
in-tile column) with a joint softmax over all key tiles.  Every function
cites the reference lines it follows.

Parity is pinned: ``tests/test_oracle_golden.py`` checks this restatement
against golden vectors produced by the unmodified reference
(``tests/golden/make_goldens.py`` imports /root/reference in the build
container; the vectors are committed as ``tests/golden/*.npz``).

Notation (tensorops.py:253-255): query tile a = (l1, j1), key tile c = (k1, i1),
in-tile row l2/k2 in [s1], in-tile column j2/i2 in [s2].  A rectangular
problem (chunked-KV) has c1_q query tile-rows and c1_k key tile-rows; the
square reference is the c1_q == c1_k case.
"""

from __future__ import annotations

import numpy as np

# --------------------------------------------------------------------------
# Token orderings (layout.py:55-114, 168-239, 279-351)
# --------------------------------------------------------------------------


def _axis_sizes(shape):
    f, h, w = shape
    return {"f": f, "h": h, "w": w}


def order_aligned(shape, g1):
    """order[p] = phi index for the aligned config whose b1 slot holds the
    axes ``g1`` (layout.py:111-114, 204-208, 218-221).  Slow digits are the g1
    axes, fast digits the remaining axes, each in (f, h, w) order."""
    sizes = _axis_sizes(shape)
    g2 = tuple(a for a in "fhw" if a not in g1)
    perm = ["fhw".index(a) for a in tuple(g1) + g2]
    grid = np.arange(int(np.prod(shape))).reshape(shape)
    del sizes
    return grid.transpose(perm).reshape(-1).astype(np.int64)


def order_phi(shape):
    """Row-major flattening (layout.py:97-101); used by raw configs (:208)."""
    return np.arange(int(np.prod(shape)), dtype=np.int64)


def order_neighborhood(shape, nbhd):
    """Neighborhood tile-plan ordering (layout.py:319-332): digits
    (f/n_f, h/n_h, n_f, n_h, w/n_w, n_w), coarse above fine."""
    f, h, w = shape
    nf, nh, nw = nbhd
    grid = np.arange(f * h * w).reshape(f // nf, nf, h // nh, nh, w // nw, nw)
    return grid.transpose(0, 2, 1, 3, 4, 5).reshape(-1).astype(np.int64)


# --------------------------------------------------------------------------
# Numerics helpers (tensorops.py:22-39)
# --------------------------------------------------------------------------


def _softmax_last(z):
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


# --------------------------------------------------------------------------
# Tiled forward (solver.py:161-217, factors.py:110-125)
# --------------------------------------------------------------------------


def tiled_forward(qs, ks, vs, c1q, c1k, c2, s1, s2, iterations=1,
                  eps_div=1e-30, eps_log=1e-300):
    """Run T alternating R/L refinements and apply the factors to V.

    ``qs`` (c1q*s1*c2*s2, d) is already scaled by the logit scale and in the
    plan's slot order (solver.py:103-106, 173-174); ``ks``/``vs`` likewise
    ordered (c1k*s1*c2*s2, d|dv).  Returns (L', R', O) with
    L' shape (c1q, c2, c1k, c2, s2, s1, s1) indexed [l1,j1,k1,i1,j2,l2,k2],
    R' shape (c1q, c2, c1k, c2, s1, s2, s2) indexed [l1,j1,k1,i1,k2,j2,i2]
    (factors.py:57-79) and O (c1q*s1*c2*s2, dv) in slot order.
    """
    d = qs.shape[1]
    dv = vs.shape[1]
    gq, gk = c1q * c2, c1k * c2
    # tile views: [tile, row, col, feature]  (solver.py:178-179 reshape)
    qt = qs.reshape(c1q, s1, c2, s2, d).transpose(0, 2, 1, 3, 4).reshape(gq, s1, s2, d)
    kt = ks.reshape(c1k, s1, c2, s2, d).transpose(0, 2, 1, 3, 4).reshape(gk, s1, s2, d)
    vt = vs.reshape(c1k, s1, c2, s2, dv).transpose(0, 2, 1, 3, 4).reshape(gk, s1, s2, dv)

    # L' starts as stacked identities (solver.py:180) => alpha_R = Q, c_R = 1
    # qrow[a, c, k, j, :] is alpha_R / c_R's numerator; cr its column mass.
    alpha_r = np.broadcast_to(qt[:, None], (gq, gk, s1, s2, d)).copy()
    c_r = np.ones((gq, gk, s1, s2))
    R = L = None
    for _ in range(iterations):
        # ---- row stage: per (a, c, k) a (s2 x s2) softmax over i2 ----
        # beta_R = alpha_R . K  (t_beta_r, tensorops.py:268); z = beta/max(c_R, eps)
        beta = np.matmul(alpha_r, np.swapaxes(kt, -1, -2)[None])        # (gq,gk,s1,s2,s2)
        z = beta / np.maximum(c_r, eps_div)[..., None]                  # solver.py:188
        R = _softmax_last(z)                                            # solver.py:189
        alpha_l = np.matmul(R, kt[None])                                # t_alpha_l :269 (gq,gk,s1,s2,d)
        ent = (R * np.log(np.maximum(R, eps_log))).sum(-1)              # t_c_l :270, solver.py:191
        # ---- column stage: per (a, j) joint softmax over keys (c, k) ----
        # S[a, j, l, (c,k)] = Q[a,l,j] . alpha_L[a,c,k,j] - c_L   (t_beta_l :271, solver.py:194)
        qcol = qt.transpose(0, 2, 1, 3)                                  # (gq, s2, s1, d)
        acol = alpha_l.transpose(0, 3, 1, 2, 4).reshape(gq, s2, gk * s1, d)
        ccol = ent.transpose(0, 3, 1, 2).reshape(gq, s2, gk * s1)
        S = np.matmul(qcol, np.swapaxes(acol, -1, -2)) - ccol[:, :, None, :]
        P = _softmax_last(S)                                             # softmax_axes (2,3,6) :195
        L = P                                                            # (gq, s2, s1, gk*s1)
        # next row stage: alpha_R = sum_l L Q, c_R = sum_l L  (t_alpha_r/t_c_r :266-267)
        Pk = P.reshape(gq, s2, s1, gk, s1)                               # [a, j, l, c, k]
        alpha_r = np.einsum("ajlck,aljv->ackjv", Pk, qt)
        c_r = Pk.sum(axis=2).transpose(0, 2, 3, 1)                       # (gq, gk, s1, s2) [a,c,k,j]
    # ---- apply (factors.py:121-125): Y = R V, O = L Y ----
    Y = np.matmul(R, vt[None])                                           # (gq,gk,s1,s2,dv) [a,c,k,j,:]
    ycol = Y.transpose(0, 3, 1, 2, 4).reshape(gq, s2, gk * s1, dv)
    O = np.matmul(L, ycol)                                               # (gq, s2, s1, dv) [a,j,l,:]
    # back to slot order [l1, l2, j1, j2]
    O = O.reshape(c1q, c2, s2, s1, dv).transpose(0, 3, 1, 2, 4).reshape(-1, dv)
    # factor containers in the reference layout
    Rf = R.reshape(c1q, c2, c1k, c2, s1, s2, s2)
    Lf = L.reshape(c1q, c2, s2, s1, c1k, c2, s1).transpose(0, 1, 4, 5, 2, 3, 6)
    return np.ascontiguousarray(Lf), np.ascontiguousarray(Rf), O


def forward_phi(q, k, v, order_q, order_k, c1q, c1k, c2, s1, s2, iterations=1,
                scale=None, eps_div=1e-30, eps_log=1e-300):
    """Row-major in, row-major out (solver.py:207-217): gather by ``order``,
    run :func:`tiled_forward`, scatter the output back to phi order."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if scale is None:
        scale = 1.0 / np.sqrt(q.shape[1])                                # solver.py:58-60
    L, R, Oo = tiled_forward((q * scale)[order_q], k[order_k], v[order_k],
                             c1q, c1k, c2, s1, s2, iterations, eps_div, eps_log)
    out = np.empty_like(Oo)
    out[order_q] = Oo
    return L, R, out


def dense_attention(q, k, v, scale=None):
    """Exact softmax(scale Q K^T) V (baselines.py:51-58) — dense-degenerate check."""
    q = np.asarray(q, dtype=np.float64)
    if scale is None:
        scale = 1.0 / np.sqrt(q.shape[1])
    a = _softmax_last((q * scale) @ np.asarray(k, dtype=np.float64).T)
    return a @ np.asarray(v, dtype=np.float64)


def rel_l2(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(x - ref) / (den if den > 0 else 1.0))
