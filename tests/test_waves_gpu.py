"""(b,h) waves of the tensor-core path (mbx_tc.cu tc_forward_waves): the workspace cap
(MBX_WS_CAP_MB, the paper's mini-sequence chunking) and the automatic
one-head waves of long odd-G_q problems.  Waves only regroup independent (b,h)
problems, so with the row-stage variant pinned (MBX_PAIR) a wave-scheduled forward is
bitwise equal to the single-wave one; the automatic choice is checked against the
fp64 oracle at full N=32760 size."""

import numpy as np
import pytest
import torch

import paper_2602_12271_b200 as pk
from paper_2602_12271_b200 import _lib, ops
from oracle import monarch_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture
def opts():
    saved = []

    def set_(name, val):
        saved.append((name, _lib.set_option(name, int(val))))

    yield set_
    for name, prev in reversed(saved):
        _lib.set_option(name, prev)


def _problem(frames, nb, B, H, seed, dev, q_frames=None):
    shape = pk.VideoShape(frames, 30, 52)
    plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), nb)
    low = pk.lower_square(plan) if q_frames is None else pk.lower_chunked(plan, q_frames)
    g = torch.Generator(device="cpu").manual_seed(seed)
    nq = low.n_q
    q = torch.randn(B, H, nq, 128, generator=g).to(dev, torch.bfloat16)
    k = torch.randn(B, H, shape.n, 128, generator=g).to(dev, torch.bfloat16)
    v = torch.randn(B, H, shape.n, 128, generator=g).to(dev, torch.bfloat16)
    return low, q, k, v


def _ws_bytes(q, k, v, low, T):
    out = torch.empty(q.shape[:3] + (v.shape[3],), dtype=q.dtype, device=q.device)
    prep = ops.prepare(q, k, v, out, low, T)
    return _lib.load().mbx_workspace_bytes(__import__("ctypes").byref(prep.desc))


@pytest.mark.parametrize("pair", [0, 1])
@pytest.mark.parametrize("T", [1, 2])
def test_workspace_cap_waves_bitwise(cuda, opts, pair, T):
    """B=2, H=3 Self-Forcing chunks: waves of one (b,h) slice under a 1 MiB cap, of
    batches, and of head groups all give the single-wave bytes."""
    low, q, k, v = _problem(3, (1, 30, 52), 2, 3, 7 + T, cuda)
    opts("MBX_PAIR", pair)
    opts("MBX_SPLIT", 0)
    opts("MBX_WAVE", 0)
    full = _ws_bytes(q, k, v, low, T)
    ref = ops.forward(q, k, v, low, T).clone()
    for wave in (1, 2, 3, 4):
        opts("MBX_WAVE", wave)
        out = ops.forward(q, k, v, low, T)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), f"MBX_WAVE={wave}"
    opts("MBX_WAVE", -1)
    opts("MBX_WS_CAP_MB", 1)
    capped = _ws_bytes(q, k, v, low, T)
    assert capped * 3 < full, (capped, full)
    out = ops.forward(q, k, v, low, T)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_chunked_kv_waves_bitwise(cuda, opts):
    """Chunked-KV (3 query frames against 9 KV frames), waves of two heads."""
    low, q, k, v = _problem(9, (1, 30, 52), 1, 5, 3, cuda, q_frames=3)
    opts("MBX_PAIR", 1)
    opts("MBX_WAVE", 0)
    ref = ops.forward(q, k, v, low, 1).clone()
    opts("MBX_WAVE", 2)
    out = ops.forward(q, k, v, low, 1)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_auto_one_head_waves_n32k(cuda, opts):
    """N=32760 (h,w) with 3 heads: the automatic plan runs one-head waves on the
    half-packed row stage; bitwise equal to one wave with that stage forced, and the
    last head within the bf16 tolerance of the oracle."""
    low, q, k, v = _problem(21, (1, 30, 52), 1, 3, 11, cuda)
    out = ops.forward(q, k, v, low, 1).clone()
    torch.cuda.synchronize()
    opts("MBX_PAIR", 1)
    opts("MBX_WAVE", 0)
    ref = ops.forward(q, k, v, low, 1)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    qn, kn, vn = (x[0, 2].float().cpu().numpy().astype(np.float64) for x in (q, k, v))
    idx = np.arange(low.n_q)
    _, _, o = orc.forward_phi(qn, kn, vn, idx, idx, low.c1_q, low.c1_kv, low.c2, low.s1, low.s2, 1)
    err = orc.rel_l2(out[0, 2].float().cpu().numpy(), o)
    assert err < 2e-2, err
