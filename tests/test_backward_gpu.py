"""GPU backward pass (mbx_backward) against float64 torch autograd of the oracle.

Oracle: oracle/monarch_torch.py, whose forward equals the golden-pinned numpy
oracle (tests/test_backward_oracle.py).  Tolerances (BASELINE.json north star):
fp32 within 1e-4 relative L2, bf16 within 2e-2 relative L2 of the fp64 gradients.
"""

import zlib

import numpy as np
import pytest
import torch

import paper_2602_12271_b200 as pk
from paper_2602_12271_b200 import ops
from oracle import monarch_oracle as orc
from oracle import monarch_torch as ort

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4
BF16_TOL = 2e-2


def _orders(low):
    oq = np.arange(low.n_q) if low.q_order is None else low.q_order
    ok = np.arange(low.n_kv) if low.kv_order is None else low.kv_order
    return oq, ok


def _oracle_grads(q, k, v, dout, low, T, b=0, h=0):
    oq, ok = _orders(low)
    to64 = lambda x: x[b, h].double().cpu()   # noqa: E731
    return ort.grads(to64(q), to64(k), to64(v), to64(dout), oq, ok, low.c1_q, low.c1_kv, low.c2, low.s1, low.s2, T)


def _plan(shape, kind):
    if kind[0] == "nb":
        return pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), kind[1])
    if kind[0] == "aligned":
        base = pk.aligned_config(shape, kind[1])
        return pk.TilePlan(base, *kind[2]) if len(kind) > 2 else base
    if kind[0] == "raw":
        return pk.config_from_sizes(shape, kind[1], kind[2])
    raise ValueError(kind)


CASES = [
    ("nb_tiled", (3, 4, 6), ("nb", (1, 4, 6)), None, 1),
    ("nb_tiled_T2", (3, 4, 6), ("nb", (1, 4, 6)), None, 2),
    ("nb_tiled_T3", (3, 4, 6), ("nb", (1, 2, 3)), None, 3),
    ("nb_c2", (2, 4, 6), ("nb", (1, 2, 3)), None, 2),
    ("untiled_fh_w", (2, 3, 5), ("aligned", ("f", "h")), None, 1),
    ("permuted_w_fh", (2, 3, 4), ("aligned", ("w",)), None, 2),
    ("permuted_tiled", (2, 4, 4), ("aligned", ("h",), (2, 2)), None, 1),
    ("raw", (2, 3, 4), ("raw", 8, 3), None, 2),
    ("chunked_kv", (4, 3, 4), ("nb", (1, 3, 4)), 2, 1),
    ("chunked_kv_T2", (4, 3, 4), ("nb", (2, 3, 4)), 2, 2),
]


@pytest.mark.parametrize("name,fhw,kind,q_frames,T", CASES, ids=[c[0] for c in CASES])
def test_backward_fp32_matches_autograd_oracle(cuda, name, fhw, kind, q_frames, T):
    shape = pk.VideoShape(*fhw)
    plan = _plan(shape, kind)
    low = pk.lower_chunked(plan, q_frames) if q_frames else pk.lower_square(plan)
    g = torch.Generator(device="cpu").manual_seed(zlib.crc32(name.encode()) % 997)
    B, H, d = 2, 2, 16
    q = torch.randn(B, H, low.n_q, d, generator=g).to(cuda)
    k, v = (torch.randn(B, H, low.n_kv, d, generator=g).to(cuda) for _ in range(2))
    dout = torch.randn(B, H, low.n_q, d, generator=g).to(cuda)
    dq, dk, dv = ops.backward(q, k, v, dout, low, T)
    for b in range(B):
        for h in range(H):
            rq, rk, rv = _oracle_grads(q, k, v, dout, low, T, b, h)
            assert orc.rel_l2(dq[b, h].cpu().numpy(), rq.numpy()) < FP32_TOL, (name, "dq", b, h)
            assert orc.rel_l2(dk[b, h].cpu().numpy(), rk.numpy()) < FP32_TOL, (name, "dk", b, h)
            assert orc.rel_l2(dv[b, h].cpu().numpy(), rv.numpy()) < FP32_TOL, (name, "dv", b, h)


@pytest.mark.parametrize("T", [1, 2])
def test_backward_bf16_self_forcing_shape(cuda, T):
    """The north-star done criterion: bf16 gradients at the C2 shape within 2e-2 of fp64."""
    s = pk.VideoShape(3, 30, 52)
    plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, 30, 52))
    low = pk.lower_square(plan)
    g = torch.Generator(device="cpu").manual_seed(40 + T)
    q, k, v, dout = (torch.randn(1, 2, 4680, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(4))
    dq, dk, dv = ops.backward(q, k, v, dout, low, T)
    assert dq.dtype == torch.bfloat16
    rq, rk, rv = _oracle_grads(q, k, v, dout, low, T, 0, 1)
    for got, ref, nm in ((dq, rq, "dq"), (dk, rk, "dk"), (dv, rv, "dv")):
        err = orc.rel_l2(got[0, 1].float().cpu().numpy(), ref.numpy())
        assert err < BF16_TOL, (nm, err)


def test_autograd_through_public_api(cuda):
    """monarch_attention on tensors that require grad goes through the custom op and its
    registered backward; the gradients equal ops.backward's."""
    s = pk.VideoShape(3, 30, 52)
    plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, 30, 52))
    g = torch.Generator(device="cpu").manual_seed(3)
    q0, k0, v0 = (torch.randn(1, 2, 4680, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    dout = torch.randn(1, 2, 4680, 128, generator=g).to(cuda, torch.bfloat16)
    q, k, v = (x.clone().requires_grad_(True) for x in (q0, k0, v0))
    out = pk.monarch_attention(q, k, v, plan)
    assert out.requires_grad
    out.backward(dout)
    dq, dk, dv = ops.backward(q0, k0, v0, dout, pk.lower_square(plan), 1)
    torch.cuda.synchronize()
    assert torch.equal(q.grad, dq) and torch.equal(k.grad, dk) and torch.equal(v.grad, dv)
    eager = pk.monarch_attention(q0, k0, v0, plan)
    assert torch.equal(out.detach(), eager)


@pytest.mark.parametrize("dtype,T", [(torch.bfloat16, 2), (torch.bfloat16, 3), (torch.float32, 3)])
def test_all_iteration_factor_export(cuda, dtype, T):
    """MBX_FLAG_ALL_ITERS: slice t holds refinement t's factors; the last slice equals the
    ordinary export, and slice t equals the final factors of a T = t + 1 run."""
    s = pk.VideoShape(3, 30, 52)
    plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, 30, 52))
    low = pk.lower_square(plan)
    g = torch.Generator(device="cpu").manual_seed(9)
    q, k, v = (torch.randn(1, 2, 4680, 128, generator=g).to(cuda, dtype) for _ in range(3))
    _, lf, rf = ops.forward(q, k, v, low, T, return_factors=True, all_iters=True)
    assert lf.shape[0] == T and rf.shape[0] == T
    for t in range(T):
        _, l1, r1 = ops.forward(q, k, v, low, t + 1, return_factors=True)
        torch.cuda.synchronize()
        assert torch.equal(lf[t], l1), t
        assert torch.equal(rf[t], r1), t


def test_backward_head_chunks_equal_one_call(cuda):
    """Mini-sequence chunking of the backward (recompute + gradients per chunk of (b,h)
    heads under a memory cap) gives the one-call gradients (to TF32 round-off: cuBLAS
    may pick another batched kernel for another batch count)."""
    s = pk.VideoShape(3, 30, 52)
    plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, 30, 52))
    low = pk.lower_square(plan)
    g = torch.Generator(device="cpu").manual_seed(9)
    q, k, v, dout = (torch.randn(2, 3, 4680, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(4))
    full = ops.backward(q, k, v, dout, low, 1, max_bytes=float("inf"))
    per = ops._backward_bytes_per_head(q, k, v, low, 1)
    chunked = ops.backward(q, k, v, dout, low, 1, max_bytes=2 * per + 1)   # chunks of 2 heads
    torch.cuda.synchronize()
    for a, b in zip(full, chunked):
        err = ((a.float() - b.float()).norm() / a.float().norm()).item()
        assert err < 2e-3, err


@pytest.mark.parametrize("name,fhw,kind,q_frames,T", CASES, ids=[c[0] for c in CASES])
def test_backward_bf16_matches_autograd_oracle(cuda, name, fhw, kind, q_frames, T):
    """bf16 I/O runs the contractions on the tensor cores (TF32 mma.sync batched GEMM):
    every plan geometry (folded and two-level reduction indices, broadcast operands)
    within the bf16 tolerance of the fp64 gradients of the bf16-rounded inputs."""
    shape = pk.VideoShape(*fhw)
    plan = _plan(shape, kind)
    low = pk.lower_chunked(plan, q_frames) if q_frames else pk.lower_square(plan)
    g = torch.Generator(device="cpu").manual_seed(zlib.crc32(name.encode()) % 991)
    B, H, d = 1, 2, 128
    q = torch.randn(B, H, low.n_q, d, generator=g).to(cuda, torch.bfloat16)
    k, v = (torch.randn(B, H, low.n_kv, d, generator=g).to(cuda, torch.bfloat16) for _ in range(2))
    dout = torch.randn(B, H, low.n_q, d, generator=g).to(cuda, torch.bfloat16)
    dq, dk, dv = ops.backward(q, k, v, dout, low, T)
    for h in range(H):
        rq, rk, rv = _oracle_grads(q, k, v, dout, low, T, 0, h)
        for got, ref, nm in ((dq, rq, "dq"), (dk, rk, "dk"), (dv, rv, "dv")):
            err = orc.rel_l2(got[0, h].float().cpu().numpy(), ref.numpy())
            assert err < BF16_TOL, (name, nm, h, err)
