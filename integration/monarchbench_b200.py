"""Reference-side binding: route ``monarchbench``'s hot path through the B200 C ABI.

This is the file a maintainer of the reference package would add:
it keeps every caller of ``monarchbench`` unchanged and swaps the arithmetic of

    solve(problem, config, solver)          solver.py:114-158
    solve_tiled(problem, plan, solver)      solver.py:161-204
    attention_output(factors, v)            solver.py:207-217

for ``mbx_forward`` / ``mbx_apply`` (include/monarch_b200.h) over ctypes, with
torch supplying device memory and the stream.  Inputs and outputs keep the
reference's types and layouts (``MonarchFactors`` / ``TiledMonarchFactors``,
float64 numpy, phi-order output).  fp32 arithmetic on the device: results match
the float64 reference to the north-star fp32 tolerance (1e-4 relative L2), not
to float64 round-off.  Per-refinement traces (``trace_objective`` /
``trace_mse``) are delegated to the package's device verification path.

    import monarchbench as mb
    from integration import monarchbench_b200
    monarchbench_b200.install(mb)      # mb.solve / mb.solve_tiled / mb.attention_output now run on the GPU
    monarchbench_b200.uninstall(mb)
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from paper_2602_12271_b200 import _lib

_SAVED: dict = {}


def _errors(mb):
    """(SolverError, LayoutError, ShapeError) of the reference (solver.py:25, layout.py:21, tensorops.py:18)."""
    import importlib

    sub = lambda name: importlib.import_module(f"{mb.__name__}.{name}")   # noqa: E731
    return sub("solver").SolverError, sub("layout").LayoutError, sub("tensorops").ShapeError


def _desc(mb, n_q, d, dv, c1, c2, s1, s2, iterations, scale, eps_div, eps_log, order_dev, flags):
    desc = _lib.MbxDesc()
    desc.abi_version = _lib.ABI_VERSION
    desc.dtype = _lib.F32
    desc.batch, desc.heads, desc.head_dim, desc.v_dim = 1, 1, d, dv
    desc.c1_q, desc.c1_kv, desc.c2, desc.s1, desc.s2 = c1, c1, c2, s1, s2
    desc.iterations = iterations
    desc.flags = flags
    desc.scale = scale
    desc.eps_div, desc.eps_log = eps_div, eps_log
    for name, width in (("q_stride", d), ("k_stride", d), ("v_stride", dv), ("o_stride", dv)):
        getattr(desc, name)[:] = (n_q * width, n_q * width, width)
    ptr = order_dev.data_ptr() if order_dev is not None else None
    desc.q_order = desc.kv_order = ptr
    return desc


def _raise(mb, lib, status):
    msg = lib.mbx_last_error().decode()
    solver_error, layout_error, _ = _errors(mb)
    if status == _lib.BAD_PLAN:
        raise layout_error(msg)
    if status in (_lib.BAD_SHAPE, _lib.BAD_ITERS, _lib.BAD_EPS, _lib.BAD_DTYPE, _lib.UNSUPPORTED):
        raise solver_error(msg)
    raise RuntimeError(f"mbx status {status}: {msg}")


def _factors(mb, problem, plan_like, c1, c2, s1, s2, solver):
    """mbx_forward with MBX_FLAG_NO_OUTPUT: the factors only (solve / solve_tiled)."""
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    order = plan_like.ordering().to_phi()
    n, d = problem.q.shape
    dv = problem.v.shape[1]
    q, k, v = (torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32), device=dev) for x in
               (problem.q, problem.k, problem.v))
    identity = np.array_equal(order, np.arange(n))
    order_dev = None if identity else torch.as_tensor(order.astype(np.int32), device=dev)
    L = torch.empty((c1, c2, c1, c2, s2, s1, s1), dtype=torch.float32, device=dev)
    R = torch.empty((c1, c2, c1, c2, s1, s2, s2), dtype=torch.float32, device=dev)
    desc = _desc(mb, n, d, dv, c1, c2, s1, s2, solver.iterations, float(problem.logit_scale),
                 solver.eps_div, solver.eps_log, order_dev, _lib.FLAG_NO_OUTPUT | _lib.FLAG_FACTORS)
    st = lib.mbx_validate(ctypes.byref(desc))
    if st:
        _raise(mb, lib, st)
    nbytes = lib.mbx_workspace_bytes(ctypes.byref(desc))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    st = lib.mbx_forward(ctypes.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(), None, L.data_ptr(),
                         R.data_ptr(), ws.data_ptr(), nbytes, torch.cuda.current_stream(dev).cuda_stream)
    if st:
        _raise(mb, lib, st)
    return L.double().cpu().numpy(), R.double().cpu().numpy(), order


def _pk_types(mb, problem, solver):
    import paper_2602_12271_b200 as pk

    s = problem.shape
    shape = pk.VideoShape(s.f, s.h, s.w)
    prob = pk.AttentionProblem(problem.q, problem.k, problem.v, shape, problem.scale)
    sc = pk.SolverConfig(iterations=solver.iterations, eps_div=solver.eps_div, eps_log=solver.eps_log,
                         trace_objective=solver.trace_objective, trace_mse=solver.trace_mse)
    return pk, shape, prob, sc


def _trace(mb, solver, problem, config_or_plan, tiled):
    """trace_objective / trace_mse: per-refinement values from the package's device path."""
    pk, shape, prob, sc = _pk_types(mb, problem, solver)
    cfg = config_or_plan.config if tiled else config_or_plan
    base = pk.BlockConfig(shape, cfg.b1, cfg.b2, cfg.g1, cfg.g2)
    if tiled:
        plan = pk.TilePlan(base, config_or_plan.c1, config_or_plan.c2, config_or_plan.neighborhoods)
        _, tr = pk.solve_tiled(prob, plan, sc)
    else:
        _, tr = pk.solve(prob, base, sc)
    return mb.SolverTrace(objectives=list(tr.objectives), mses=list(tr.mses))


def solve_b200(mb, problem, config, solver=None):
    solver = solver or mb.SolverConfig()
    if config.shape != problem.shape:
        raise _errors(mb)[0](f"config shape {config.shape} != problem shape {problem.shape}")
    if solver.keep_workspace:
        raise _errors(mb)[0]("keep_workspace: the fused kernels never materialise the solver's intermediates")
    L, R, order = _factors(mb, problem, config, 1, 1, config.b1, config.b2, solver)
    trace = _trace(mb, solver, problem, config, False) if (solver.trace_objective or solver.trace_mse) \
        else mb.SolverTrace()
    return mb.MonarchFactors(config.b1, config.b2, L[0, 0, 0, 0], R[0, 0, 0, 0], order=order), trace


def solve_tiled_b200(mb, problem, plan, solver=None):
    solver = solver or mb.SolverConfig()
    if plan.shape != problem.shape:
        raise _errors(mb)[0](f"plan shape {plan.shape} != problem shape {problem.shape}")
    if solver.keep_workspace:
        raise _errors(mb)[0]("keep_workspace: the fused kernels never materialise the solver's intermediates")
    L, R, order = _factors(mb, problem, plan, plan.c1, plan.c2, plan.tile_b1, plan.tile_b2, solver)
    trace = _trace(mb, solver, problem, plan, True) if (solver.trace_objective or solver.trace_mse) \
        else mb.SolverTrace()
    return mb.TiledMonarchFactors(plan, L, R, order=order), trace


def attention_output_b200(mb, factors, v):
    """mbx_apply: O = L' (R' V) in phi order (factors.py:110-125 via solver.py:207-217)."""
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    if isinstance(factors, mb.MonarchFactors):
        b1, b2, c1, c2 = factors.b1, factors.b2, 1, 1
        lf, rf = factors.l_blocks[None, None, None, None], factors.r_blocks[None, None, None, None]
    else:
        p = factors.plan
        b1, b2, c1, c2 = p.config.b1, p.config.b2, p.c1, p.c2
        lf, rf = factors.l_blocks, factors.r_blocks
    v = np.asarray(v)
    if v.ndim != 2 or v.shape[0] != b1 * b2:
        raise _errors(mb)[2](f"v must have {b1 * b2} rows, got {v.shape}")
    n, dv = v.shape
    order = factors.order
    order_dev = None if order is None or np.array_equal(order, np.arange(n)) else \
        torch.as_tensor(np.asarray(order, dtype=np.int32), device=dev)
    vt = torch.as_tensor(np.ascontiguousarray(v, dtype=np.float32), device=dev)
    out = torch.empty_like(vt)
    lt = torch.as_tensor(np.ascontiguousarray(lf, dtype=np.float32), device=dev)
    rt = torch.as_tensor(np.ascontiguousarray(rf, dtype=np.float32), device=dev)
    desc = _desc(mb, n, dv, dv, c1, c2, b1 // c1, b2 // c2, 1, 1.0, 1e-30, 1e-300, order_dev, 0)
    nbytes = lib.mbx_apply_workspace_bytes(ctypes.byref(desc))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    st = lib.mbx_apply(ctypes.byref(desc), lt.data_ptr(), rt.data_ptr(), vt.data_ptr(), out.data_ptr(),
                       ws.data_ptr(), nbytes, torch.cuda.current_stream(dev).cuda_stream)
    if st:
        _raise(mb, lib, st)
    return out.double().cpu().numpy()


def install(mb) -> None:
    """Patch ``mb`` (the monarchbench package) and ``mb.solver`` in place."""
    import importlib

    solver_mod = importlib.import_module(mb.__name__ + ".solver")
    if id(mb) in _SAVED:
        return
    _SAVED[id(mb)] = {(m, name): getattr(m, name) for m in (mb, solver_mod)
                      for name in ("solve", "solve_tiled", "attention_output")}
    for m in (mb, solver_mod):
        m.solve = lambda problem, config, solver=None: solve_b200(mb, problem, config, solver)
        m.solve_tiled = lambda problem, plan, solver=None: solve_tiled_b200(mb, problem, plan, solver)
        m.attention_output = lambda factors, v: attention_output_b200(mb, factors, v)


def uninstall(mb) -> None:
    for (m, name), fn in _SAVED.pop(id(mb), {}).items():
        setattr(m, name, fn)


__all__ = ["install", "uninstall", "solve_b200", "solve_tiled_b200", "attention_output_b200"]
