"""Reference-compatible operator API (drop-in for monarchbench.solver).

Same names, argument meaning, return layout and error classes as
/root/reference/pkg/src/monarchbench/solver.py and factors.py:

* ``AttentionProblem`` (solver.py:29-60) — validates (N, d) q, k, v over a
  VideoShape, scale defaults to 1/sqrt(d);
* ``SolverConfig`` (solver.py:63-77) — iterations >= 1, eps in (0, 1e-6];
* ``solve(problem, config, solver)`` (solver.py:114-158) and
  ``solve_tiled(problem, plan, solver)`` (solver.py:161-204) return
  ``(MonarchFactors | TiledMonarchFactors, SolverTrace)`` with the factors in
  the reference layout (factors.py:33-83) and ``order`` set;
* ``attention_output(factors, v)`` (solver.py:207-217) applies factors to a
  row-major V and returns a row-major output.

The arithmetic runs on the GPU through the C ABI (fp32 for numpy inputs,
bf16 for bfloat16 torch inputs); results come back as float64 numpy arrays
like the reference's.  trace_objective / trace_mse (N <= 4096 verification
paths) are recorded on the GPU by verify.solve_traced; keep_workspace (the
solver's intermediate tensors) raises SolverError.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .layout import BlockConfig, TilePlan, VideoShape, lower_square
from .ops import SolverError


class FactorError(ValueError):
    """Malformed factor container (factors.py:29-30)."""


class ShapeError(ValueError):
    """Operand shapes inconsistent with the operation (tensorops.py:18-19)."""


def _as_array(m):
    if isinstance(m, torch.Tensor):
        return m
    return np.asarray(m)


def _finite(m) -> bool:
    if isinstance(m, torch.Tensor):
        return bool(torch.isfinite(m).all())
    return bool(np.isfinite(m).all())


@dataclass(frozen=True)
class AttentionProblem:
    """Q, K, V of shape (N, d) over a video grid; scale defaults to 1/sqrt(d)."""

    q: object
    k: object
    v: object
    shape: VideoShape
    scale: float | None = None

    def __post_init__(self) -> None:
        n = self.shape.n
        for name in ("q", "k", "v"):
            object.__setattr__(self, name, _as_array(getattr(self, name)))
        d = self.q.shape[1] if self.q.ndim == 2 else -1
        for name, m in (("q", self.q), ("k", self.k), ("v", self.v)):
            if m.ndim != 2 or m.shape[0] != n:
                raise SolverError(f"{name} must be ({n}, d), got {tuple(m.shape)}")
            if not _finite(m):
                raise SolverError(f"{name} has non-finite entries")
        if self.k.shape[1] != d:
            raise SolverError("q and k must share the head dimension")

    @property
    def n(self) -> int:
        return self.shape.n

    @property
    def head_dim(self) -> int:
        return int(self.q.shape[1])

    @property
    def logit_scale(self) -> float:
        return float(self.scale) if self.scale is not None else 1.0 / float(np.sqrt(self.head_dim))


@dataclass(frozen=True)
class SolverConfig:
    iterations: int = 1
    eps_div: float = 1e-30
    eps_log: float = 1e-300
    trace_objective: bool = False
    trace_mse: bool = False
    keep_workspace: bool = False

    def __post_init__(self) -> None:
        if self.iterations < 1:
            raise SolverError("iterations must be >= 1")
        for name in ("eps_div", "eps_log"):
            eps = getattr(self, name)
            if not 0.0 < eps <= 1e-6:
                raise SolverError(f"{name} must lie in (0, 1e-6], got {eps}")


@dataclass
class SolverTrace:
    """Per-iteration traces (always empty here: tracing densifies N x N)."""

    objectives: list[float] = field(default_factory=list)
    mses: list[float] = field(default_factory=list)
    workspace: object | None = None


@dataclass(frozen=True)
class MonarchFactors:
    """Untiled factors L (b2, b1, b1) [j,l,k], R (b1, b2, b2) [k,j,i] (factors.py:33-54)."""

    b1: int
    b2: int
    l_blocks: np.ndarray
    r_blocks: np.ndarray
    order: np.ndarray | None = None

    def __post_init__(self) -> None:
        if tuple(self.l_blocks.shape) != (self.b2, self.b1, self.b1):
            raise FactorError(f"L shape {self.l_blocks.shape} != {(self.b2, self.b1, self.b1)}")
        if tuple(self.r_blocks.shape) != (self.b1, self.b2, self.b2):
            raise FactorError(f"R shape {self.r_blocks.shape} != {(self.b1, self.b2, self.b2)}")
        if not (np.isfinite(self.l_blocks).all() and np.isfinite(self.r_blocks).all()):
            raise FactorError("factor entries must be finite")

    @property
    def n(self) -> int:
        return self.b1 * self.b2


@dataclass(frozen=True)
class TiledMonarchFactors:
    """Per-tile factors (factors.py:57-83): L' (c1,c2,c1,c2,s2,s1,s1)
    [l1,j1,k1,i1,j2,l2,k2], R' (c1,c2,c1,c2,s1,s2,s2) [l1,j1,k1,i1,k2,j2,i2]."""

    plan: TilePlan
    l_blocks: np.ndarray
    r_blocks: np.ndarray
    order: np.ndarray | None = None

    def __post_init__(self) -> None:
        c1, c2, s1, s2 = self.plan.c1, self.plan.c2, self.plan.tile_b1, self.plan.tile_b2
        if tuple(self.l_blocks.shape) != (c1, c2, c1, c2, s2, s1, s1):
            raise FactorError(f"L' shape {self.l_blocks.shape} != {(c1, c2, c1, c2, s2, s1, s1)}")
        if tuple(self.r_blocks.shape) != (c1, c2, c1, c2, s1, s2, s2):
            raise FactorError(f"R' shape {self.r_blocks.shape} != {(c1, c2, c1, c2, s1, s2, s2)}")
        if not (np.isfinite(self.l_blocks).all() and np.isfinite(self.r_blocks).all()):
            raise FactorError("factor entries must be finite")

    @property
    def n(self) -> int:
        return self.plan.config.b1 * self.plan.config.b2


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise SolverError("the B200 operator needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_device(m, dtype=None) -> torch.Tensor:
    dev = _device()
    if isinstance(m, torch.Tensor):
        t = m.to(dev)
        if dtype is not None:
            t = t.to(dtype)
        elif t.dtype not in (torch.float32, torch.bfloat16):
            t = t.float()
        return t.contiguous()
    return torch.from_numpy(np.ascontiguousarray(m, dtype=np.float32)).to(dev)


def _check_unsupported(solver: SolverConfig) -> None:
    if solver.keep_workspace:
        raise SolverError("keep_workspace exports the solver's intermediate tensors (alpha/beta/z of both "
                          "stages); the fused kernels never materialise them")


def _run(problem: AttentionProblem, low, solver: SolverConfig, want_output: bool):
    q = _to_device(problem.q)
    k = _to_device(problem.k, q.dtype)
    v = _to_device(problem.v, q.dtype)
    out, lf, rf = ops.forward(q[None, None], k[None, None], v[None, None], low, solver.iterations,
                              problem.logit_scale, solver.eps_div, solver.eps_log,
                              return_factors=True)
    return out[0, 0], lf[0, 0], rf[0, 0]


def _host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def solve(problem: AttentionProblem, config: BlockConfig,
          solver: SolverConfig = SolverConfig()) -> tuple[MonarchFactors, SolverTrace]:
    """Untiled factors under ``config`` (solver.py:114-158).  trace_objective /
    trace_mse record per-refinement values on the GPU (verify.solve_traced)."""
    if config.shape != problem.shape:
        raise SolverError(f"config shape {config.shape} != problem shape {problem.shape}")
    _check_unsupported(solver)
    if solver.trace_objective or solver.trace_mse:
        from .verify import solve_traced
        return solve_traced(problem, config, solver)
    return _solve_untraced(problem, config, solver)


def _solve_untraced(problem: AttentionProblem, config: BlockConfig, solver: SolverConfig):
    low = lower_square(config)
    _, lf, rf = _run(problem, low, solver, False)
    order = config.ordering().to_phi()
    fac = MonarchFactors(config.b1, config.b2, _host(lf)[0, 0, 0, 0], _host(rf)[0, 0, 0, 0], order=order)
    return fac, SolverTrace()


def solve_tiled(problem: AttentionProblem, plan: TilePlan,
                solver: SolverConfig = SolverConfig()) -> tuple[TiledMonarchFactors, SolverTrace]:
    """Tiled factors for ``plan`` (solver.py:161-204); traces as in ``solve``."""
    if plan.shape != problem.shape:
        raise SolverError(f"plan shape {plan.shape} != problem shape {problem.shape}")
    _check_unsupported(solver)
    if solver.trace_objective or solver.trace_mse:
        from .verify import solve_traced
        return solve_traced(problem, plan, solver)
    return _solve_tiled_untraced(problem, plan, solver)


def _solve_tiled_untraced(problem: AttentionProblem, plan: TilePlan, solver: SolverConfig):
    low = lower_square(plan)
    _, lf, rf = _run(problem, low, solver, False)
    order = plan.ordering().to_phi()
    return TiledMonarchFactors(plan, _host(lf), _host(rf), order=order), SolverTrace()


def attention_output(factors, v) -> np.ndarray:
    """Apply factors to a row-major V; row-major output (solver.py:207-217)."""
    if isinstance(factors, MonarchFactors):
        b1, b2, c1, c2 = factors.b1, factors.b2, 1, 1
        lf = factors.l_blocks[None, None, None, None]
        rf = factors.r_blocks[None, None, None, None]
    else:
        p = factors.plan
        b1, b2, c1, c2 = p.config.b1, p.config.b2, p.c1, p.c2
        lf, rf = factors.l_blocks, factors.r_blocks
    v_arr = _as_array(v)
    if v_arr.ndim != 2 or v_arr.shape[0] != b1 * b2:
        raise ShapeError(f"v must have {b1 * b2} rows, got {tuple(v_arr.shape)}")
    from .layout import Lowered
    order = factors.order
    order32 = None if order is None else np.ascontiguousarray(order, dtype=np.int32)
    low = Lowered(c1, c1, c2, b1 // c1, b2 // c2, b1 * b2, b1 * b2, order32, order32)
    vt = _to_device(v_arr, torch.float32)
    dev = vt.device
    lt = torch.from_numpy(np.ascontiguousarray(lf, dtype=np.float32)).to(dev)
    rt = torch.from_numpy(np.ascontiguousarray(rf, dtype=np.float32)).to(dev)
    out = ops.apply(lt, rt, vt[None, None], low)
    return _host(out[0, 0])
