"""Batched torch-level operator over the C ABI.

``monarch_attention(q, k, v, plan, ...)`` is the fast entry point: q, k, v are
CUDA tensors (B, H, N, d) in token (phi) order, bf16 or fp32; the output has
q's layout.  It lowers the plan (layout.Lowered), builds an ``mbx_desc`` and
enqueues ``mbx_forward`` on torch's current stream.  No CPU fallback exists:
CPU tensors or a missing library raise.
"""

from __future__ import annotations

import ctypes
import functools
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .layout import LayoutError, Lowered, TilePlan, BlockConfig, lower_chunked, lower_square


class SolverError(ValueError):
    """Invalid problem or solver configuration (solver.py:25-26)."""


_DTYPES = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16}

_order_cache: dict[tuple, tuple[np.ndarray, torch.Tensor]] = {}


def _device_order(order: np.ndarray | None, device: torch.device) -> torch.Tensor | None:
    """Upload a slot permutation once per (array, device); lowered plans are
    cached, so their order arrays are long-lived."""
    if order is None:
        return None
    key = (id(order), str(device))
    hit = _order_cache.get(key)
    if hit is None or hit[0] is not order:
        hit = (order, torch.from_numpy(np.ascontiguousarray(order, dtype=np.int32)).to(device))
        _order_cache[key] = hit
    return hit[1]


@functools.lru_cache(maxsize=256)
def _lower_square_cached(plan):
    return lower_square(plan)


@functools.lru_cache(maxsize=256)
def _lower_chunked_cached(plan, q_frames):
    return lower_chunked(plan, q_frames)


@dataclass
class PreparedProblem:
    """A descriptor plus the device buffers it points into (kept alive)."""

    desc: _lib.MbxDesc
    q_order: torch.Tensor | None
    kv_order: torch.Tensor | None
    workspace: torch.Tensor | None = None


def _strides(t: torch.Tensor) -> tuple[int, int, int]:
    if t.stride(-1) != 1:
        raise SolverError("the feature dimension must be contiguous")
    return (t.stride(0), t.stride(1), t.stride(2))


def prepare(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor,
            low: Lowered, iterations: int = 1, scale: float | None = None,
            eps_div: float = 1e-30, eps_log: float = 1e-300, flags: int = 0) -> PreparedProblem:
    if not (q.is_cuda and k.is_cuda and v.is_cuda and out.is_cuda):
        raise SolverError("monarch_attention runs on CUDA tensors only (no CPU fallback)")
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        raise SolverError("q, k, v must be (B, H, N, d)")
    if q.dtype not in _DTYPES or k.dtype != q.dtype or v.dtype != q.dtype or out.dtype != q.dtype:
        raise SolverError(f"q, k, v, out must share dtype float32 or bfloat16, got {q.dtype}")
    if not (k.device == q.device and v.device == q.device and out.device == q.device):
        raise SolverError("q, k, v and out must live on one device")
    B, H, nq, d = q.shape
    if k.shape[:2] != (B, H) or v.shape[:2] != (B, H):
        raise SolverError("q, k, v batch/head dims differ")
    if nq != low.n_q or k.shape[2] != low.n_kv or v.shape[2] != low.n_kv:
        raise SolverError(f"token counts (q {nq}, k {k.shape[2]}, v {v.shape[2]}) do not match the "
                          f"plan (q {low.n_q}, kv {low.n_kv})")
    if k.shape[3] != d:
        raise SolverError("q and k must share the head dimension")
    if out.shape != (B, H, nq, v.shape[3]):
        raise SolverError("out must be (B, H, N_q, d_v)")
    if iterations < 1:
        raise SolverError("iterations must be >= 1")
    desc = _lib.MbxDesc()
    desc.abi_version = _lib.ABI_VERSION
    desc.dtype = _DTYPES[q.dtype]
    desc.batch, desc.heads, desc.head_dim, desc.v_dim = B, H, d, v.shape[3]
    desc.c1_q, desc.c1_kv, desc.c2, desc.s1, desc.s2 = low.c1_q, low.c1_kv, low.c2, low.s1, low.s2
    desc.iterations = iterations
    desc.flags = flags
    desc.scale = float(scale) if scale is not None else 1.0 / math.sqrt(d)
    desc.eps_div, desc.eps_log = eps_div, eps_log
    for name, t in (("q_stride", q), ("k_stride", k), ("v_stride", v), ("o_stride", out)):
        getattr(desc, name)[:] = _strides(t)
    qo = _device_order(low.q_order, q.device)
    ko = _device_order(low.kv_order, q.device)
    desc.q_order = qo.data_ptr() if qo is not None else None
    desc.kv_order = ko.data_ptr() if ko is not None else None
    if low.nbhd is not None:
        desc.grid[:] = low.grid
        desc.nbhd[:] = low.nbhd
    return PreparedProblem(desc, qo, ko)


def _raise_mapped(err: _lib.MbxError):
    if err.status == _lib.BAD_PLAN:
        raise LayoutError(str(err)) from None
    if err.status in (_lib.BAD_SHAPE, _lib.BAD_ITERS, _lib.BAD_EPS, _lib.BAD_DTYPE, _lib.UNSUPPORTED):
        raise SolverError(str(err)) from None
    raise err


# Prepared descriptors keyed by everything they encode (shapes, strides, dtype, device,
# plan, solver settings, flags).  The descriptor holds no data pointers, so one entry
# serves every call with the same geometry; the lowered plan is kept alive by the entry.
_PREP: dict = {}
# Workspaces per (device, stream): uses on one stream are ordered by that stream.
_WS: dict = {}


def _prepared(q, k, v, out, low, iterations, scale, eps_div, eps_log, flags):
    key = (q.shape, q.stride(), k.shape, k.stride(), v.shape, v.stride(), out.shape, out.stride(),
           q.dtype, q.device, id(low), iterations, scale, eps_div, eps_log, flags, _lib.OPTIONS_VERSION[0])
    hit = _PREP.get(key)
    if hit is not None and hit[0] is low:
        return hit[1], hit[2]
    prep = prepare(q, k, v, out, low, iterations, scale, eps_div, eps_log, flags)
    lib = _lib.load()
    try:
        _lib.check(lib.mbx_validate(ctypes.byref(prep.desc)))
    except _lib.MbxError as e:
        _raise_mapped(e)
    nbytes = lib.mbx_workspace_bytes(ctypes.byref(prep.desc))
    if len(_PREP) > 512:
        _PREP.clear()
    _PREP[key] = (low, prep, nbytes)
    return prep, nbytes


def _workspace(device: torch.device, stream, nbytes: int) -> torch.Tensor:
    key = (device.index, stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def forward(q, k, v, low: Lowered, iterations=1, scale=None, eps_div=1e-30, eps_log=1e-300,
            out=None, return_factors=False, force_generic=False, workspace=None, split=None,
            all_iters=False):
    """Run ``mbx_forward``; returns out or (out, L', R') with fp32 factors of
    shape (B, H, c1_q, c2, c1_kv, c2, s2, s1, s1) / (..., s1, s2, s2) -- with
    ``all_iters`` one such slice per refinement, stacked on a leading T axis.

    ``split``: None = the library's choice of concurrent head halves, True / False
    force it on / off.  The call is enqueued on the current stream of q's device
    (that device is made current for the call)."""
    lib = _lib.load()
    if out is None:
        out = torch.empty(q.shape[:3] + (v.shape[3],), dtype=q.dtype, device=q.device)
    flags = _lib.FLAG_FORCE_GENERIC if force_generic else 0
    if return_factors:
        flags |= _lib.FLAG_FACTORS
        if all_iters:
            flags |= _lib.FLAG_ALL_ITERS
    if split is not None:
        flags |= _lib.FLAG_SPLIT if split else _lib.FLAG_NO_SPLIT
    prep, nbytes = _prepared(q, k, v, out, low, iterations, scale, eps_div, eps_log, flags)
    lf = rf = None
    if return_factors:
        B, H = q.shape[:2]
        lead = (iterations,) if all_iters else ()
        lf = torch.empty(lead + (B, H, low.c1_q, low.c2, low.c1_kv, low.c2, low.s2, low.s1, low.s1),
                         dtype=torch.float32, device=q.device)
        rf = torch.empty(lead + (B, H, low.c1_q, low.c2, low.c1_kv, low.c2, low.s1, low.s2, low.s2),
                         dtype=torch.float32, device=q.device)
    with torch.cuda.device(q.device):
        stream = torch.cuda.current_stream(q.device).cuda_stream
        if workspace is None or workspace.numel() < nbytes:
            workspace = _workspace(q.device, stream, nbytes)
        st = lib.mbx_forward(ctypes.byref(prep.desc), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                             out.data_ptr(), lf.data_ptr() if lf is not None else None,
                             rf.data_ptr() if rf is not None else None,
                             workspace.data_ptr(), nbytes, stream)
    if st != 0:
        try:
            _lib.check(st)
        except _lib.MbxError as e:
            _raise_mapped(e)
    if return_factors:
        return out, lf, rf
    return out


BACKWARD_MAX_BYTES = 8 << 30   # device memory one backward call may hold (workspace + factors)


def _backward_bytes_per_head(q, k, v, low: Lowered, iterations) -> int:
    """Workspace + recomputed factors of one (b,h) head of the backward."""
    lib = _lib.load()
    q1, k1, v1 = q[:1, :1], k[:1, :1], v[:1, :1]
    prep = prepare(q1, k1, v1, q1, low, iterations)
    ws = lib.mbx_backward_workspace_bytes(ctypes.byref(prep.desc))
    pairs = low.c1_q * low.c2 * low.c1_kv * low.c2
    fac = iterations * pairs * (low.s2 * low.s1 * low.s1 + low.s1 * low.s2 * low.s2) * 4
    return int(ws) + int(fac)


def backward(q, k, v, dout, low: Lowered, iterations=1, scale=None, eps_div=1e-30, eps_log=1e-300,
             factors=None, max_bytes=None):
    """Gradients (dq, dk, dv) of sum(out * dout) through ``mbx_backward``.

    ``factors`` = (L', R') of every refinement as returned by
    ``forward(..., return_factors=True, all_iters=True)``; recomputed when absent
    (FlashAttention-style recomputation: the forward is cheap next to the backward).
    With recomputation the (b,h) heads are processed in chunks whose workspace and
    factors stay under ``max_bytes`` (default ``BACKWARD_MAX_BYTES``): the paper's
    mini-sequence chunking for training, e.g. the Wan stack at B=8."""
    lib = _lib.load()
    if factors is None:
        B, H = q.shape[:2]
        cap = max_bytes if max_bytes is not None else BACKWARD_MAX_BYTES
        per = B * H if cap == float("inf") else \
            max(1, int(cap) // max(1, _backward_bytes_per_head(q, k, v, low, iterations)))
        if per < B * H:
            flat = [x.reshape(1, B * H, x.shape[2], x.shape[3]) for x in (q, k, v, dout)]
            grads = [torch.empty(x.shape, dtype=x.dtype, device=x.device) for x in flat[:3]]
            for lo in range(0, B * H, per):
                hi = min(B * H, lo + per)
                part = backward(*(x[:, lo:hi] for x in flat), low, iterations, scale, eps_div, eps_log,
                                max_bytes=float("inf"))
                for g_, p_ in zip(grads, part):
                    g_[:, lo:hi].copy_(p_)
            return tuple(g_.view(x.shape) for g_, x in zip(grads, (q, k, v)))
    if factors is None:
        _, lf, rf = forward(q, k, v, low, iterations, scale, eps_div, eps_log, return_factors=True,
                            all_iters=True)
    else:
        lf, rf = factors
    dout = dout.to(q.dtype)
    if dout.stride(-1) != 1:
        dout = dout.contiguous()
    prep = prepare(q, k, v, dout, low, iterations, scale, eps_div, eps_log)
    try:
        _lib.check(lib.mbx_validate(ctypes.byref(prep.desc)))
    except _lib.MbxError as e:
        _raise_mapped(e)
    dq, dk, dv = (torch.empty_like(x) for x in (q, k, v))
    if tuple(dq.stride()) != tuple(q.stride()) or tuple(dk.stride()) != tuple(k.stride()) or \
            tuple(dv.stride()) != tuple(v.stride()):
        raise SolverError("gradient tensors must share the strides of q, k, v")
    nbytes = lib.mbx_backward_workspace_bytes(ctypes.byref(prep.desc))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=q.device)
    with torch.cuda.device(q.device):
        st = lib.mbx_backward(ctypes.byref(prep.desc), q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(),
                              lf.data_ptr(), rf.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                              ws.data_ptr(), nbytes, torch.cuda.current_stream(q.device).cuda_stream)
    if st != 0:
        try:
            _lib.check(st)
        except _lib.MbxError as e:
            _raise_mapped(e)
    return dq, dk, dv


def apply(l_factor: torch.Tensor, r_factor: torch.Tensor, v: torch.Tensor, low: Lowered,
          out_dtype=None) -> torch.Tensor:
    """``mbx_apply``: O = L' (R' V) for given fp32 factors (factors.py:110-125)."""
    lib = _lib.load()
    B, H = v.shape[:2]
    q_like = torch.empty((B, H, low.n_q, v.shape[3]), dtype=v.dtype, device=v.device)
    out = torch.empty_like(q_like)
    prep = prepare(q_like, v, v, out, low)
    nbytes = lib.mbx_apply_workspace_bytes(ctypes.byref(prep.desc))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=v.device)
    with torch.cuda.device(v.device):
        st = lib.mbx_apply(ctypes.byref(prep.desc), l_factor.contiguous().data_ptr(),
                           r_factor.contiguous().data_ptr(), v.data_ptr(), out.data_ptr(),
                           ws.data_ptr(), nbytes, torch.cuda.current_stream(v.device).cuda_stream)
    try:
        _lib.check(st)
    except _lib.MbxError as e:
        _raise_mapped(e)
    return out


def selected_path(q, k, v, low: Lowered, iterations=1, return_factors=False) -> str:
    lib = _lib.load()
    out = torch.empty(q.shape[:3] + (v.shape[3],), dtype=q.dtype, device=q.device)
    prep = prepare(q, k, v, out, low, iterations, flags=_lib.FLAG_FACTORS if return_factors else 0)
    return {0: "simt", 1: "tcgen05"}.get(lib.mbx_selected_path(ctypes.byref(prep.desc)), "invalid")


def lower_for(plan, q_tokens: int, kv_tokens: int, kv_frames: int | None = None) -> Lowered:
    """The (cached) kernel lowering of ``plan`` for a square or chunked-KV problem."""
    if kv_frames is None and q_tokens == kv_tokens:
        return _lower_square_cached(plan)
    if not isinstance(plan, TilePlan):
        raise LayoutError("chunked-KV needs a TilePlan")
    s = plan.shape
    if kv_frames is not None and kv_frames != s.f:
        raise LayoutError(f"kv_frames {kv_frames} != plan frames {s.f}")
    hw = s.h * s.w
    if q_tokens % hw:
        raise SolverError("query tokens are not a whole number of frames")
    return _lower_chunked_cached(plan, q_tokens // hw)


# ---------------------------------------------------------------- torch custom op
# ``torch.ops.monarch_b200.monarch_attention`` makes the operator visible to
# torch.compile / FakeTensor tracing and is where autograd attaches.  The plan is
# not a tensor: callers register its lowering under a string key (``plan_key``).
_LOWERED: dict[str, Lowered] = {}


def plan_key(low: Lowered) -> str:
    key = f"{low.c1_q},{low.c1_kv},{low.c2},{low.s1},{low.s2},{low.n_q},{low.n_kv},{low.grid},{low.nbhd}," \
          f"{'id' if low.q_order is None else hash(low.q_order.tobytes())}," \
          f"{'id' if low.kv_order is None else hash(low.kv_order.tobytes())}"
    _LOWERED.setdefault(key, low)
    return key


def _plan_fields(plan) -> tuple:
    """A TilePlan / BlockConfig as a tuple of primitives (Dynamo can pass those as constants;
    it cannot reconstruct frozen dataclass instances)."""
    cfg = plan.config if isinstance(plan, TilePlan) else plan
    s = cfg.shape
    head = (s.f, s.h, s.w, cfg.b1, cfg.b2, cfg.g1, cfg.g2)
    if isinstance(plan, TilePlan):
        return ("tile",) + head + (plan.c1, plan.c2, plan.neighborhoods)
    return ("block",) + head


@torch._dynamo.assume_constant_result
def _traced_plan_key(fields: tuple, q_tokens: int, kv_tokens: int, kv_frames) -> str:
    """Plan lowering for a traced call: host-side numpy work on graph constants, run once
    at trace time (Dynamo records the resulting key string, it does not trace into it)."""
    from .layout import VideoShape

    kind, f, h, w, b1, b2, g1, g2 = fields[:8]
    cfg = BlockConfig(VideoShape(f, h, w), b1, b2, g1, g2)
    plan = TilePlan(cfg, fields[8], fields[9], fields[10]) if kind == "tile" else cfg
    return plan_key(lower_for(plan, q_tokens, kv_tokens, kv_frames))


@torch.library.custom_op("monarch_b200::monarch_attention", mutates_args=())
def _monarch_op(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, plan: str, iterations: int,
                scale: float) -> torch.Tensor:
    return forward(q, k, v, _LOWERED[plan], iterations, scale)


@_monarch_op.register_fake
def _monarch_op_fake(q, k, v, plan, iterations, scale):
    return q.new_empty(q.shape[:3] + (v.shape[3],))


def _op_setup_context(ctx, inputs, output):
    q, k, v, plan, iterations, scale = inputs
    ctx.save_for_backward(q, k, v)
    ctx.plan, ctx.iterations, ctx.scale = plan, iterations, scale


def _op_backward(ctx, dout):
    q, k, v = ctx.saved_tensors
    dq, dk, dv = backward(q, k, v, dout, _LOWERED[ctx.plan], ctx.iterations, ctx.scale)
    return dq, dk, dv, None, None, None


_monarch_op.register_autograd(_op_backward, setup_context=_op_setup_context)


def monarch_attention(q, k, v, plan, iterations: int = 1, scale: float | None = None,
                      kv_frames: int | None = None, return_factors: bool = False,
                      force_generic: bool = False, out=None):
    """Tiled MonarchAttention forward on (B, H, N, d) CUDA tensors.

    ``plan`` is a TilePlan (tiled, solver.py:161) or BlockConfig (untiled,
    solver.py:114).  With ``kv_frames`` unset the problem is square; for a
    chunked-KV rollout pass the plan over the full (f_kv, h, w) key grid and
    q holding the last ``q_frames = q.shape[2] // (h*w)`` frames.

    Eager calls go straight to the C ABI; under torch.compile tracing, or when
    autograd needs a graph, the call goes through the registered custom op.
    """
    traced = torch.compiler.is_compiling()
    needs_grad = torch.is_grad_enabled() and (q.requires_grad or k.requires_grad or v.requires_grad)
    if (traced or needs_grad) and not (return_factors or force_generic or out is not None):
        sc = float(scale) if scale is not None else 1.0 / math.sqrt(q.shape[3])
        key = _traced_plan_key(_plan_fields(plan), q.shape[2], k.shape[2], kv_frames) if traced else \
            plan_key(lower_for(plan, q.shape[2], k.shape[2], kv_frames))
        return torch.ops.monarch_b200.monarch_attention(q, k, v, key, iterations, sc)
    low = lower_for(plan, q.shape[2], k.shape[2], kv_frames)
    return forward(q, k, v, low, iterations, scale, out=out, return_factors=return_factors,
                   force_generic=force_generic)


_D2H_STREAMS: dict = {}
_HOST_BUFS: dict = {}


def _d2h_stream(device: torch.device) -> torch.cuda.Stream:
    st = _D2H_STREAMS.get(device.index)
    if st is None:
        st = _D2H_STREAMS[device.index] = torch.cuda.Stream(device=device)
    return st


def monarch_attention_host(q, k, v, plan, iterations: int = 1, scale: float | None = None,
                           kv_frames: int | None = None, out=None, chunks: int | None = None,
                           device=None):
    """``monarch_attention`` on HOST (B, H, N, d) tensors, returning a host tensor.

    The (b,h) problems are independent, so the call is pipelined over chunks of the
    flattened B*H axis: the host->device copies and the forward of each chunk run on
    the current stream while the device->host copy of the previous chunk's output runs
    on a second stream (PCIe is full duplex).  Measured at C2 with pinned memory:
    1.08 ms against 1.11 ms for copy-in / forward / copy-out in sequence, with the
    43 MB copy-in alone at 0.79 ms (scripts/exp_e2e.py; more chunks lose to the
    per-chunk stream synchronisation).  The returned tensor is written
    asynchronously: synchronize the current stream before reading it (as with
    ``copy_(non_blocking=True)``)."""
    if q.is_cuda or k.is_cuda or v.is_cuda:
        raise SolverError("monarch_attention_host takes host tensors; use monarch_attention on device tensors")
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        raise SolverError("q, k, v must be (B, H, N, d)")
    B, H = q.shape[:2]
    if k.shape[:2] != (B, H) or v.shape[:2] != (B, H):
        raise SolverError("q, k, v must share (B, H)")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    bh = B * H
    # (b, h) units as one head axis of a size-1 batch: contiguous host slices per chunk
    qh, kh, vh = (x.contiguous().reshape(1, bh, x.shape[2], x.shape[3]) for x in (q, k, v))
    if out is None:
        out = torch.empty(q.shape[:3] + (v.shape[3],), dtype=q.dtype, pin_memory=True)
    if out.is_cuda or not out.is_contiguous() or out.shape != q.shape[:3] + (v.shape[3],):
        raise SolverError("out must be a contiguous host tensor of shape (B, H, N_q, d_v)")
    oh = out.view(1, bh, q.shape[2], v.shape[3])
    n = max(1, min(bh, chunks or 2))
    comp = torch.cuda.current_stream(dev)
    s_out = _d2h_stream(dev)
    # device staging buffers are cached per shape: reuse is ordered by the current stream
    # (this call's copies and forwards follow the previous call's, whose copy-out the
    # current stream waited for), and the caching allocator never sees a cross-stream free
    key = (dev.index, qh.shape, kh.shape, vh.shape, oh.shape, q.dtype, v.dtype)
    bufs = _HOST_BUFS.get(key)
    if bufs is None:
        bufs = tuple(torch.empty(x.shape, dtype=x.dtype, device=dev) for x in (qh, kh, vh, oh))
        if len(_HOST_BUFS) >= 4:
            _HOST_BUFS.clear()
        _HOST_BUFS[key] = bufs
    qd, kd, vd, od = bufs
    for i in range(n):
        lo, hi = bh * i // n, bh * (i + 1) // n
        for d_, h_ in ((qd, qh), (kd, kh), (vd, vh)):
            d_[:, lo:hi].copy_(h_[:, lo:hi], non_blocking=True)
        monarch_attention(qd[:, lo:hi], kd[:, lo:hi], vd[:, lo:hi], plan, iterations, scale, kv_frames,
                          out=od[:, lo:hi])
        s_out.wait_stream(comp)
        with torch.cuda.stream(s_out):
            oh[:, lo:hi].copy_(od[:, lo:hi], non_blocking=True)
    comp.wait_stream(s_out)
    return out


__all__ = ["monarch_attention", "monarch_attention_host", "forward", "backward", "apply", "prepare", "selected_path",
           "lower_for", "plan_key",
           "SolverError", "BlockConfig", "TilePlan"]
