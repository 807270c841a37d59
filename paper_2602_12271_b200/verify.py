"""Verification path on the GPU: factor containers, dense
materialisation of small factorizations and the solver's per-iteration traces.

* ``save_factors`` / ``load_factors`` -- the reference's MNR1 container
  (factors.py:244-298): magic ``b"MNR1"``, five little-endian ``uint32``
  (kind, b1, b2, c1, c2), then L and R as raw float64.  Same bytes, same
  ``FactorError`` conditions; a deserialized tiled plan carries the canonical
  (1, b1, b2) video shape, as in the reference.
* ``densify`` / ``densify_tiled`` / ``approx_attention_matrix`` (factors.py:93-107,
  solver.py:218-225): the N x N matrix of a factorization, N <= 4096, computed
  on the device in float64 (a verification path: it is exact, not fast).
* ``objective`` (solver.py:228-254) and ``frobenius_mse`` (tensorops.py:42-49).
* ``solve_traced`` -- what ``SolverConfig(trace_objective / trace_mse)`` records:
  the objective / MSE after every refinement t = 1..T.  The fused kernels keep
  no per-iteration state, so iteration t is re-run with ``iterations = t``
  (factor export, fp32) and densified.
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .layout import BlockConfig, TilePlan, VideoShape
from .solver import FactorError, MonarchFactors, SolverError, TiledMonarchFactors

DENSIFY_LIMIT = 4096   # factors.py:24
MNR_MAGIC = b"MNR1"
_HEAD = struct.Struct("<5I")


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise SolverError("the verification path runs on the GPU (no CUDA device)")
    return torch.device("cuda", torch.cuda.current_device())


def _t(a) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=_dev())


def _check_size(n: int) -> None:
    if n > DENSIFY_LIMIT:
        raise FactorError(f"densify is a verification path, refusing N = {n} > {DENSIFY_LIMIT}")


def _dense_slot_order(factors) -> torch.Tensor:
    """N x N matrix in slot (ordered) index space, float64 on the device."""
    _check_size(factors.n)
    L, R = _t(factors.l_blocks), _t(factors.r_blocks)
    if isinstance(factors, MonarchFactors):
        # M[(l, j), (k, i)] = L[j, l, k] R[k, j, i]
        return torch.einsum("jlk,kji->ljki", L, R).reshape(factors.n, factors.n)
    # M[(a, l, b, j), (c, k, e, i)] = L'[a, b, c, e, j, l, k] R'[a, b, c, e, k, j, i]
    return torch.einsum("abcejlk,abcekji->albjckei", L, R).reshape(factors.n, factors.n)


def identity_factors(b1: int, b2: int) -> MonarchFactors:
    """Factors whose densification is the N x N identity (factors.py:86-90)."""
    return MonarchFactors(b1, b2, np.tile(np.eye(b1), (b2, 1, 1)), np.tile(np.eye(b2), (b1, 1, 1)))


def densify(factors: MonarchFactors) -> np.ndarray:
    """factors.py:98-101 -- slot order."""
    return _dense_slot_order(factors).cpu().numpy()


def densify_tiled(factors: TiledMonarchFactors) -> np.ndarray:
    """factors.py:104-107 -- slot order."""
    return _dense_slot_order(factors).cpu().numpy()


def _dense_token_order(factors) -> torch.Tensor:
    m = _dense_slot_order(factors)
    if factors.order is None:
        return m
    order = torch.as_tensor(np.asarray(factors.order, dtype=np.int64), device=m.device)
    out = torch.empty_like(m)
    out[order[:, None], order[None, :]] = m
    return out


def approx_attention_matrix(factors) -> np.ndarray:
    """solver.py:218-225 -- densified approximation in row-major token order."""
    return _dense_token_order(factors).cpu().numpy()


def _objective(approx: torch.Tensor, logits: torch.Tensor) -> float:
    if float(approx.min()) < 0:
        raise SolverError("objective needs a non-negative approximation")
    ent = torch.where(approx > 0, approx * torch.log(approx.clamp_min(1e-300)), torch.zeros_like(approx))
    return float((approx * logits).sum() - ent.sum())


def objective(factors, q, k, scale: float | None = None) -> float:
    """<A', scale Q K^T> + H(A') of the densified factors (solver.py:235-254)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    if scale is None:
        scale = 1.0 / np.sqrt(q.shape[1])
    if factors.order is not None:
        q, k = q[factors.order], k[factors.order]
    qt, kt = _t(q), _t(k)
    return _objective(_dense_slot_order(factors), (qt * scale) @ kt.T)


def frobenius_mse(a, b) -> float:
    """Mean squared entrywise difference (tensorops.py:42-49)."""
    from .solver import ShapeError

    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ShapeError(f"shape mismatch: {a.shape} vs {b.shape}")
    d = _t(a) - _t(b)
    return float((d * d).mean())


def solve_traced(problem, plan_or_config, solver):
    """(factors, SolverTrace) with ``objectives`` / ``mses`` filled per refinement, as
    the reference's solve / solve_tiled record them (solver.py:150-157, 196-203)."""
    from dataclasses import replace

    from . import solver as sv

    tiled = isinstance(plan_or_config, TilePlan)
    run = sv._solve_tiled_untraced if tiled else sv._solve_untraced
    trace = sv.SolverTrace()
    base = replace(solver, trace_objective=False, trace_mse=False)
    n = problem.n
    _check_size(n)
    order = plan_or_config.ordering().to_phi()
    qs = (problem.q * problem.logit_scale)[order]
    ks = problem.k[order]
    logits = _t(qs) @ _t(ks).T
    dense_ref = None
    if solver.trace_mse:
        dense_ref = torch.softmax(logits, dim=1)   # dense attention in slot order (solver.py:109-111)
    fac = None
    for t in range(1, solver.iterations + 1):
        fac, _ = run(problem, plan_or_config, replace(base, iterations=t))
        approx = _dense_slot_order(fac)
        if solver.trace_objective:
            trace.objectives.append(_objective(approx, logits))
        if dense_ref is not None:
            d = approx - dense_ref
            trace.mses.append(float((d * d).mean()))
    return fac, trace


def save_factors(factors, path) -> None:
    """MNR1 container (factors.py:244-262)."""
    if isinstance(factors, MonarchFactors):
        head = _HEAD.pack(0, factors.b1, factors.b2, 1, 1)
    else:
        p = factors.plan
        head = _HEAD.pack(1, p.config.b1, p.config.b2, p.c1, p.c2)
    blob = MNR_MAGIC + head + np.ascontiguousarray(factors.l_blocks, dtype="<f8").tobytes() + \
        np.ascontiguousarray(factors.r_blocks, dtype="<f8").tobytes()
    if hasattr(path, "write"):
        path.write(blob)
    else:
        with open(path, "wb") as fh:
            fh.write(blob)


def load_factors(path):
    """Inverse of ``save_factors`` (factors.py:265-298)."""
    if hasattr(path, "read"):
        data = path.read()
    else:
        with open(path, "rb") as fh:
            data = fh.read()
    if data[:4] != MNR_MAGIC:
        raise FactorError(f"bad magic {data[:4]!r}, expected {MNR_MAGIC!r}")
    if len(data) < 4 + _HEAD.size:
        raise FactorError(f"truncated header: {len(data)} bytes")
    kind, b1, b2, c1, c2 = _HEAD.unpack_from(data, 4)
    if kind == 0:
        l_shape, r_shape = (b2, b1, b1), (b1, b2, b2)
    elif kind == 1:
        s1, s2 = b1 // c1, b2 // c2
        l_shape, r_shape = (c1, c2, c1, c2, s2, s1, s1), (c1, c2, c1, c2, s1, s2, s2)
    else:
        raise FactorError(f"unknown kind tag {kind}")
    nl, nr = int(np.prod(l_shape)), int(np.prod(r_shape))
    need = 4 + _HEAD.size + 8 * (nl + nr)
    if len(data) != need:
        raise FactorError(f"container has {len(data)} bytes, expected {need}")
    body = np.frombuffer(data, dtype="<f8", offset=4 + _HEAD.size)
    lb, rb = body[:nl].reshape(l_shape).copy(), body[nl:].reshape(r_shape).copy()
    if kind == 0:
        return MonarchFactors(b1, b2, lb, rb)
    cfg = BlockConfig(VideoShape(1, b1, b2), b1, b2, ("f", "h"), ("w",))
    return TiledMonarchFactors(TilePlan(cfg, c1, c2), lb, rb)


__all__ = ["DENSIFY_LIMIT", "identity_factors", "densify", "densify_tiled", "approx_attention_matrix", "objective",
           "frobenius_mse", "solve_traced", "save_factors", "load_factors"]
