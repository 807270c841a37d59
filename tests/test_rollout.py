"""QKV1 real-activation I/O pinned to bytes written by the reference (qkv_io.py),
and the KV-cache rollout driver (GPU)."""
import os

import numpy as np
import pytest
import torch

import paper_2602_12271_b200 as pk
from oracle import monarch_oracle as orc
from paper_2602_12271_b200 import ops, rollout

GOLD = os.path.join(os.path.dirname(__file__), "golden", "qkv1_small.bin")
BF16_TOL = 2e-2


def _oracle(q, k, v, low, T):
    """fp64 oracle per head of (H, N, d) tensors."""
    oq = np.arange(low.n_q) if low.q_order is None else low.q_order
    ok = np.arange(low.n_kv) if low.kv_order is None else low.kv_order
    return np.stack([orc.forward_phi(*(x[i].double().cpu().numpy() for x in (q, k, v)), oq, ok, low.c1_q,
                                     low.c1_kv, low.c2, low.s1, low.s2, T)[2] for i in range(q.shape[0])])


def _golden_arrays():
    rng = np.random.default_rng(7)
    return [rng.standard_normal((24, 5)) for _ in range(3)]   # make_qkv1.py: VideoShape(2, 3, 4), d = 5


def test_qkv1_reads_reference_bytes():
    p = rollout.load_problem(GOLD)
    assert (p.shape.f, p.shape.h, p.shape.w, p.head_dim) == (2, 3, 4, 5)
    for got, want in zip((p.q, p.k, p.v), _golden_arrays()):
        np.testing.assert_array_equal(got, want)


def test_qkv1_writer_reproduces_reference_bytes(tmp_path):
    p = rollout.load_problem(GOLD, scale=0.25)
    assert p.logit_scale == 0.25
    out = tmp_path / "rt.bin"
    rollout.save_problem(p, out)
    assert out.read_bytes() == open(GOLD, "rb").read()


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"QKV2" + b[4:], "bad magic"),
    (lambda b: b[:10], "truncated header"),
    (lambda b: b[:4] + (0).to_bytes(4, "little") + b[8:], "invalid header"),
    (lambda b: b[:-8], "8 missing"),
    (lambda b: b + b"\0" * 16, "16 trailing"),
])
def test_qkv1_malformed_containers(tmp_path, mutate, msg):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(mutate(open(GOLD, "rb").read()))
    with pytest.raises(rollout.TensorFileError, match=msg):
        rollout.load_problem(bad)


def test_qkv1_rejects_nonfinite(tmp_path):
    q, k, v = _golden_arrays()
    q[3, 1] = np.nan
    path = tmp_path / "nan.bin"
    with open(GOLD, "rb") as fh:
        head = fh.read(20)
    path.write_bytes(head + q.astype("<f8").tobytes() + k.astype("<f8").tobytes() + v.astype("<f8").tobytes())
    with pytest.raises(pk.SolverError):
        rollout.load_problem(path)


@pytest.mark.gpu
@pytest.mark.parametrize("tile,T", [((1, 30, 52), 1), ((3, 30, 52), 1), ((1, 30, 52), 2)])
def test_rollout_matches_independent_chunked_calls(cuda, tile, T):
    """Three 3-frame chunks through the frame cache: each step equals the chunked-KV
    operator on a contiguous copy of the cached prefix (bitwise), the first step
    equals the square problem, and every step matches the oracle (2 heads)."""
    h, w, cf, nch = 30, 52, 3, 3
    g = torch.Generator(device="cpu").manual_seed(21 + T)
    q, k, v = (torch.randn(1, 2, nch * cf * h * w, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    out = rollout.rollout_chunks(q, k, v, h, w, cf, tile=tile, iterations=T)
    hw = h * w
    for c in range(nch):
        f_kv = (c + 1) * cf
        shape = pk.VideoShape(f_kv, h, w)
        plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), tile)
        qs = q[:, :, c * cf * hw:(c + 1) * cf * hw].contiguous()
        kp, vp = k[:, :, :f_kv * hw].contiguous(), v[:, :, :f_kv * hw].contiguous()
        low = pk.lower_chunked(plan, cf)
        assert ops.selected_path(qs, kp, vp, low, T) == "tcgen05"
        ref = ops.forward(qs, kp, vp, low, T)
        got = out[:, :, c * cf * hw:(c + 1) * cf * hw]
        assert torch.equal(got, ref)
        if c == 0:
            assert torch.equal(got, pk.monarch_attention(qs, kp, vp, plan, iterations=T))
        assert orc.rel_l2(got[0].float().cpu().numpy(), _oracle(qs[0], kp[0], vp[0], low, T)) < BF16_TOL


@pytest.mark.gpu
def test_load_qkv_runs_on_device(cuda, tmp_path):
    """A QKV1 file's activations go straight to the operator (fp32 SIMT path here:
    d = 5) and match the reference-compatible solver on the same problem."""
    q, k, v, shape = rollout.load_qkv(GOLD, cuda, torch.float32)
    assert q.shape == (1, 1, 24, 5) and q.device.type == "cuda"
    plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), (1, 3, 4))
    out = pk.monarch_attention(q, k, v, plan)
    p = rollout.load_problem(GOLD)
    factors, _ = pk.solve_tiled(p, plan)
    ref = pk.attention_output(factors, p.v)
    assert orc.rel_l2(out[0, 0].double().cpu().numpy(), ref) < 1e-4


@pytest.mark.gpu
def test_rollout_is_cuda_graph_capturable(cuda):
    """The whole rollout (cache appends + chunked-KV forwards) captures into one CUDA
    graph; replays reproduce the eager outputs bitwise."""
    h, w, cf, nch = 30, 52, 3, 2
    g = torch.Generator(device="cpu").manual_seed(5)
    q, k, v = (torch.randn(1, 2, nch * cf * h * w, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    hw = h * w
    cache = rollout.FrameKVCache(1, 2, nch * cf, h, w, 128, device=cuda)
    ro = rollout.Rollout(h, w, cache)
    outs = [None] * nch

    def run():
        cache.reset()
        for c in range(nch):
            sl = slice(c * cf * hw, (c + 1) * cf * hw)
            outs[c] = ro.step(q[:, :, sl], k[:, :, sl], v[:, :, sl])

    run()
    eager = [o.clone() for o in outs]
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        run()
    for o in outs:
        o.zero_()
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(outs, eager):
        assert torch.equal(a, b)
