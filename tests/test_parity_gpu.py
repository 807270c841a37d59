"""GPU parity of the CUDA path against the reference goldens and the oracle.

Tolerances (BASELINE.json north_star): fp32 kernels within 1e-4 relative L2,
bf16 kernels within 2e-2 relative L2 of the fp64/fp32 reference output and
factors.  Every call goes through the C ABI (libmonarch_b200.so).
"""

import numpy as np
import pytest
import torch

import paper_2602_12271_b200 as pk
from paper_2602_12271_b200 import ops
from cases import case_inputs, oracle_lowering, package_lowering, package_plan
from oracle import monarch_oracle as orc

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4
BF16_TOL = 2e-2


@pytest.fixture
def mbx_option():
    """Set process-wide library options (mbx_set_option) for one test, restoring them after."""
    from paper_2602_12271_b200 import _lib

    saved = []

    def set_(name, val):
        saved.append((name, _lib.set_option(name, int(val))))

    yield set_
    for name, prev in reversed(saved):
        _lib.set_option(name, prev)


def _t(x, dev, dtype=torch.float32):
    return torch.as_tensor(np.asarray(x), dtype=dtype, device=dev)


def test_library_is_the_cuda_path(cuda):
    from paper_2602_12271_b200 import _lib

    lib = _lib.load()
    assert lib.mbx_version() == _lib.ABI_VERSION


def test_goldens_fp32_through_abi(goldens, cuda):
    manifest, data = goldens
    for meta in manifest:
        q, k, v = case_inputs(meta, data)
        low = package_lowering(meta)
        out, lf, rf = ops.forward(_t(q, cuda)[None, None], _t(k, cuda)[None, None],
                                  _t(v, cuda)[None, None], low, meta["T"], return_factors=True)
        name = meta["name"]
        ref = data[f"{name}/out"]
        assert orc.rel_l2(out[0, 0].cpu().numpy(), ref) < FP32_TOL, name
        if f"{name}/L" in data:
            assert orc.rel_l2(lf[0, 0].cpu().numpy(), data[f"{name}/L"]) < FP32_TOL, name
            assert orc.rel_l2(rf[0, 0].cpu().numpy(), data[f"{name}/R"]) < FP32_TOL, name


def test_reference_api_drop_in(goldens, cuda):
    """solve / solve_tiled + attention_output with the reference's call shapes."""
    manifest, data = goldens
    for meta in manifest:
        if meta["kind"] == "chunk":
            continue
        q, k, v = case_inputs(meta, data)
        shape = pk.VideoShape(*meta["shape"])
        plan = package_plan(meta)
        problem = pk.AttentionProblem(q, k, v, shape)
        cfg = pk.SolverConfig(iterations=meta["T"])
        if meta["kind"] == "solve":
            fac, trace = pk.solve(problem, plan, cfg)
            assert isinstance(fac, pk.MonarchFactors)
        else:
            fac, trace = pk.solve_tiled(problem, plan, cfg)
            assert isinstance(fac, pk.TiledMonarchFactors)
        assert trace.objectives == [] and fac.order is not None
        out = pk.attention_output(fac, v)
        assert out.dtype == np.float64 and out.shape == (shape.n, v.shape[1])
        name = meta["name"]
        assert orc.rel_l2(out, data[f"{name}/out"]) < FP32_TOL, name
        if f"{name}/L" in data:
            L = data[f"{name}/L"]
            R = data[f"{name}/R"]
            if meta["kind"] == "solve":
                L, R = L[0, 0, 0, 0], R[0, 0, 0, 0]
            assert orc.rel_l2(fac.l_blocks, L) < FP32_TOL, name
            assert orc.rel_l2(fac.r_blocks, R) < FP32_TOL, name


def test_solver_errors_match_reference(cuda):
    s = pk.VideoShape(2, 3, 3)
    rng = np.random.default_rng(0)
    q = rng.standard_normal((18, 4))
    with pytest.raises(pk.SolverError):
        pk.SolverConfig(iterations=0)
    with pytest.raises(pk.SolverError):
        bad = q.copy()
        bad[0, 0] = np.nan
        pk.AttentionProblem(bad, q, q, s)
    problem = pk.AttentionProblem(q, q, q, s)
    with pytest.raises(pk.SolverError):
        pk.solve(problem, pk.aligned_config(pk.VideoShape(1, 3, 6), ("f", "h")))
    with pytest.raises(pk.SolverError):
        pk.solve(problem, pk.aligned_config(s, ("f", "h")), pk.SolverConfig(keep_workspace=True))
    _, trace = pk.solve(problem, pk.aligned_config(s, ("f", "h")), pk.SolverConfig(iterations=2, trace_mse=True))
    assert len(trace.mses) == 2 and not trace.objectives
    with pytest.raises(pk.ShapeError):
        fac, _ = pk.solve(problem, pk.aligned_config(s, ("f", "h")))
        pk.attention_output(fac, q[:5])


def _sf_plan(f=3, h=30, w=52, nb=None):
    s = pk.VideoShape(f, h, w)
    return pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), nb or (1, h, w))


def _oracle_heads(q, k, v, low, T, scale=None):
    """fp64 oracle per (b, h) of (B, H, N, d) tensors."""
    qn, kn, vn = (x.float().cpu().numpy().astype(np.float64) for x in (q, k, v))
    oq = np.arange(low.n_q) if low.q_order is None else low.q_order
    ok = np.arange(low.n_kv) if low.kv_order is None else low.kv_order
    out = np.empty(q.shape[:3] + (v.shape[3],))
    for b in range(q.shape[0]):
        for h in range(q.shape[1]):
            _, _, out[b, h] = orc.forward_phi(qn[b, h], kn[b, h], vn[b, h], oq, ok, low.c1_q,
                                              low.c1_kv, low.c2, low.s1, low.s2, T, scale)
    return out


@pytest.mark.parametrize("dtype,tol", [(torch.float32, FP32_TOL), (torch.bfloat16, BF16_TOL)])
@pytest.mark.parametrize("T", [1, 2, 3])
def test_self_forcing_chunk_shape(cuda, dtype, tol, T):
    """C2 shape (3 frames x 30x52, d=128, (h,w) tiles) on 2 heads vs the oracle."""
    g = torch.Generator(device="cpu").manual_seed(T)
    q, k, v = (torch.randn(1, 2, 4680, 128, generator=g).to(cuda, dtype) for _ in range(3))
    plan = _sf_plan()
    out = pk.monarch_attention(q, k, v, plan, iterations=T)
    ref = _oracle_heads(q, k, v, pk.lower_square(plan), T)
    assert orc.rel_l2(out.float().cpu().numpy(), ref) < tol


@pytest.mark.parametrize("T", [1, 2])
def test_chunked_kv_rollout(cuda, T):
    """3 query frames vs 7 KV frames, (h,w) tiles — rectangular tile grid."""
    g = torch.Generator(device="cpu").manual_seed(11)
    fkv, fq, h, w = 7, 3, 30, 52
    q = torch.randn(1, 1, fq * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    k = torch.randn(1, 1, fkv * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    v = torch.randn(1, 1, fkv * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    plan = _sf_plan(fkv, h, w)
    out = pk.monarch_attention(q, k, v, plan, iterations=T, kv_frames=fkv)
    ref = _oracle_heads(q, k, v, pk.lower_chunked(plan, fq), T)
    assert orc.rel_l2(out.float().cpu().numpy(), ref) < BF16_TOL


def test_strided_batch_heads_and_permuted_plan(cuda):
    """(B, N, H, d) storage viewed as (B, H, N, d); neighborhood plan with c2 > 1."""
    g = torch.Generator(device="cpu").manual_seed(3)
    B, H, f, h, w, d = 2, 3, 4, 6, 8, 32
    n = f * h * w
    base = [torch.randn(B, n, H, d, generator=g).to(cuda) for _ in range(3)]
    q, k, v = (x.permute(0, 2, 1, 3) for x in base)
    plan = _sf_plan(f, h, w, (2, 3, 4))
    out = pk.monarch_attention(q, k, v, plan, iterations=2)
    ref = _oracle_heads(q, k, v, pk.lower_square(plan), 2)
    assert orc.rel_l2(out.cpu().numpy(), ref) < FP32_TOL


def test_deterministic_bitwise(cuda):
    """Back-to-back launches (no host sync, fresh workspaces from the caching
    allocator) must agree bitwise: catches races between pipeline stages."""
    g = torch.Generator(device="cpu").manual_seed(4)
    q, k, v = (torch.randn(1, 12, 4680, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    plan = _sf_plan()
    outs = [pk.monarch_attention(q, k, v, plan) for _ in range(16)]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_factors_row_stochastic_on_device(cuda):
    g = torch.Generator(device="cpu").manual_seed(5)
    q, k, v = (torch.randn(1, 1, 4 * 6 * 8, 16, generator=g).to(cuda) for _ in range(3))
    plan = _sf_plan(4, 6, 8, (2, 3, 4))
    _, lf, rf = pk.monarch_attention(q, k, v, plan, iterations=3, return_factors=True)
    assert (rf.sum(-1) - 1).abs().max().item() < 1e-5
    assert (lf.sum(dim=(4, 5, 8)) - 1).abs().max().item() < 1e-5


@pytest.mark.parametrize("frames,q_frames,B,H,T", [(3, 3, 1, 12, 1), (5, 3, 2, 2, 1), (21, 3, 1, 1, 1),
                                                   (3, 3, 1, 4, 2), (3, 3, 1, 2, 3), (7, 3, 1, 2, 2),
                                                   (21, 3, 1, 1, 3)])
def test_tensor_core_path(cuda, frames, q_frames, B, H, T):
    """The tcgen05 path is the one selected for the hot shapes -- for every
    refinement count (T >= 2 adds the statistics / alpha_R hand-off kernels) --
    and matches both the oracle (2e-2) and the SIMT path run on the same inputs."""
    g = torch.Generator(device="cpu").manual_seed(frames * 10 + T)
    h, w = 30, 52
    q = torch.randn(B, H, q_frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    k = torch.randn(B, H, frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    v = torch.randn(B, H, frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    plan = _sf_plan(frames, h, w)
    low = pk.lower_chunked(plan, q_frames) if q_frames != frames else pk.lower_square(plan)
    assert ops.selected_path(q, k, v, low, T) == "tcgen05"
    out = ops.forward(q, k, v, low, T)
    ref_simt = ops.forward(q, k, v, low, T, force_generic=True)
    assert orc.rel_l2(out.float().cpu().numpy(), ref_simt.float().cpu().numpy()) < 1e-2
    nh = min(H, 2)
    ref = _oracle_heads(q[:1, :nh], k[:1, :nh], v[:1, :nh], low, T)
    assert orc.rel_l2(out[:1, :nh].float().cpu().numpy(), ref) < BF16_TOL


def test_rejects_cpu_tensors():
    q = torch.zeros(1, 1, 4680, 128)
    with pytest.raises(pk.SolverError):
        pk.monarch_attention(q, q, q, _sf_plan())


@pytest.mark.parametrize("frames,q_frames,nb,H,T", [(3, 3, (3, 30, 52), 2, 1), (6, 3, (3, 30, 52), 2, 1),
                                                    (2, 2, None, 2, 1), (5, 5, (5, 30, 52), 1, 1),
                                                    (7, 7, None, 1, 1), (5, 5, "raw", 1, 1),
                                                    (3, 3, (3, 30, 52), 2, 2), (6, 3, (3, 30, 52), 1, 3),
                                                    (4, 4, (4, 30, 52), 1, 2)])
def test_wide_column_path(cuda, frames, q_frames, nb, H, T):
    """Plans with more than 32 rows per tile -- the paper's (3h, w) tiles (s1 = 90),
    untiled (fh, w) configs (s1 = 60, 210), s1 = 150 (two M tiles), a raw
    misaligned (b1, b2) = (300, 26) blocking, and T = 2, 3 (alpha_R hand-off with
    up to 128 query rows) -- run on tensor cores and match the oracle."""
    g = torch.Generator(device="cpu").manual_seed(frames * 7 + q_frames + 100 * T)
    h, w = 30, 52
    q = torch.randn(1, H, q_frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    k = torch.randn(1, H, frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    v = torch.randn(1, H, frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    shape = pk.VideoShape(frames, h, w)
    if nb is None:
        plan = pk.aligned_config(shape, ("f", "h"))
        low = pk.lower_square(plan)
    elif nb == "raw":
        plan = pk.config_from_sizes(shape, 300, 26)
        low = pk.lower_square(plan)
    else:
        plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), nb)
        low = pk.lower_chunked(plan, q_frames) if q_frames != frames else pk.lower_square(plan)
    assert low.s1 > 32
    assert ops.selected_path(q, k, v, low, T) == "tcgen05"
    out = ops.forward(q, k, v, low, T)
    ref = _oracle_heads(q, k, v, low, T)
    assert orc.rel_l2(out.float().cpu().numpy(), ref) < BF16_TOL


@pytest.mark.parametrize("frames,q_frames,nb,T", [(3, 3, (3, 30, 52), 1), (6, 3, (3, 30, 52), 2), (7, 7, None, 1),
                                                  (5, 5, "raw", 1), (3, 3, None, 1)])
def test_wide_column_ping_pong_vs_single_stream(cuda, mbx_option, frames, q_frames, nb, T):
    """The output pass of the wide column stage, two item streams per CTA (tc_column_wide2,
    the default) against the single-stream kernel (MBX_WIDE2=0): same softmax arithmetic,
    per-chunk O accumulation order identical, so equal up to the MMA's bf16 rounding of P;
    odd and even item counts per CTA, one and several key chunks per column."""
    g = torch.Generator(device="cpu").manual_seed(frames * 11 + q_frames + 7 * T)
    h, w = 30, 52
    q = torch.randn(1, 3, q_frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    k = torch.randn(1, 3, frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    v = torch.randn(1, 3, frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    shape = pk.VideoShape(frames, h, w)
    if nb is None:
        low = pk.lower_square(pk.aligned_config(shape, ("f", "h")))
    elif nb == "raw":
        low = pk.lower_square(pk.config_from_sizes(shape, 300, 26))
    else:
        plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), nb)
        low = pk.lower_chunked(plan, q_frames) if q_frames != frames else pk.lower_square(plan)
    assert low.s1 > 32
    two = ops.forward(q, k, v, low, T).clone()
    mbx_option("MBX_WIDE2", 0)
    one = ops.forward(q, k, v, low, T)
    torch.cuda.synchronize()
    assert orc.rel_l2(two.float().cpu().numpy(), one.float().cpu().numpy()) < 2e-3


@pytest.mark.parametrize("row_stage", ["0", "1"])
@pytest.mark.parametrize("frames,q_frames,h,nb,T", [(3, 3, 30, None, 1), (5, 3, 30, None, 2), (2, 2, 30, None, 1),
                                                    (4, 4, 30, None, 1), (3, 3, 30, (3, 30, 52), 1),
                                                    (3, 3, 30, "raw", 2), (7, 3, 30, None, 3), (3, 3, 15, None, 2)])
def test_row_stage_variants(cuda, mbx_option, row_stage, frames, q_frames, h, nb, T):
    """Both row-stage kernels -- the classic one (whole query tiles per M=128 task)
    and the half-packed one (two M=64 (query tile, row) halves per task, halves with
    the same row sharing one K/V stage) -- on G_q = 1, 2, 3, 4, a raw (117, 40) blocking
    (odd s1: a lone last half) and G_q s1 = 3 x 15 odd, against the oracle.  MBX_PAIR
    forces the variant."""
    mbx_option("MBX_PAIR", row_stage)
    g = torch.Generator(device="cpu").manual_seed(frames * 13 + q_frames + 7 * T + h)
    w = 52
    shape = pk.VideoShape(frames, h, w)
    if nb is None:
        plan = _sf_plan(frames, h, w)
    elif nb == "raw":
        plan = pk.config_from_sizes(shape, 117, 40)
    else:
        plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), nb)
    low = pk.lower_chunked(plan, q_frames) if q_frames != frames else pk.lower_square(plan)
    q = torch.randn(1, 2, q_frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    k = torch.randn(1, 2, frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    v = torch.randn(1, 2, frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    assert ops.selected_path(q, k, v, low, T) == "tcgen05"
    out = ops.forward(q, k, v, low, T)
    ref = _oracle_heads(q, k, v, low, T)
    assert orc.rel_l2(out.float().cpu().numpy(), ref) < BF16_TOL


def test_head_slices_of_single_batch_stay_on_tensor_cores(cuda):
    """Head slices of a B = 1 tensor keep the parent's batch stride (PyTorch calls them
    contiguous); a size-1 batch has nothing to fold, so they must still run on the
    tcgen05 path -- and give the same rows as the full-head call."""
    g = torch.Generator(device="cpu").manual_seed(11)
    q, k, v = (torch.randn(1, 4, 4680, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    low = pk.lower_square(_sf_plan())
    full = ops.forward(q, k, v, low, 1)
    qs, ks, vs = (x[:, 1:3].contiguous() for x in (q, k, v))
    assert qs.stride(0) == q.stride(0)
    assert ops.selected_path(qs, ks, vs, low, 1) == "tcgen05"
    part = ops.forward(qs, ks, vs, low, 1)
    assert torch.equal(part, full[:, 1:3])


@pytest.mark.parametrize("B,H,chunks,q_frames", [(1, 12, None, 3), (2, 3, 4, 3), (1, 2, 2, 1)])
def test_host_api_pipelined_matches_device(cuda, B, H, chunks, q_frames):
    """monarch_attention_host (pinned host tensors, H2D / forward / D2H pipelined over
    (b,h) chunks on three streams) returns exactly the device call's output, for
    square and chunked-KV problems."""
    g = torch.Generator(device="cpu").manual_seed(B * 10 + H)
    frames = 3
    q = torch.randn(B, H, q_frames * 4680 // 3, 128, generator=g).to(torch.bfloat16).pin_memory()
    k, v = (torch.randn(B, H, frames * 1560, 128, generator=g).to(torch.bfloat16).pin_memory() for _ in range(2))
    plan = _sf_plan(frames)
    kvf = frames if q_frames != frames else None
    out = pk.monarch_attention_host(q, k, v, plan, kv_frames=kvf, chunks=chunks)
    torch.cuda.synchronize()
    ref = pk.monarch_attention(q.to(cuda), k.to(cuda), v.to(cuda), plan, kv_frames=kvf)
    assert out.device.type == "cpu"
    assert torch.equal(out, ref.cpu())
    with pytest.raises(pk.SolverError):
        pk.monarch_attention_host(q.to(cuda), k, v, plan)


@pytest.mark.parametrize("env", [{"MBX_PDL": "0"}, {"MBX_L2HINT": "0"}, {"MBX_WIDE": "1"}])
def test_diagnostic_switches_keep_results(cuda, mbx_option, env):
    """The diagnostic switches (no programmatic dependent launch, no L2 residency
    hints, the FlashAttention-style column stage forced on s1 <= 32) change
    scheduling only: results stay within the bf16 budget of the oracle and, for
    the first two, bitwise equal to the default launch sequence."""
    g = torch.Generator(device="cpu").manual_seed(17)
    q, k, v = (torch.randn(1, 2, 4680, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    low = pk.lower_square(_sf_plan())
    ref = ops.forward(q, k, v, low, 2)
    for key, val in env.items():
        mbx_option(key, val)
    out = ops.forward(q, k, v, low, 2)
    if "MBX_WIDE" in env:
        assert orc.rel_l2(out.float().cpu().numpy(), _oracle_heads(q, k, v, low, 2)) < BF16_TOL
    else:
        assert torch.equal(out, ref)


@pytest.mark.parametrize("q_frames,T", [(3, 1), (3, 2), (1, 1)])
def test_head_split_concurrent_halves_bitwise(cuda, q_frames, T):
    """split=True runs the two halves of the heads concurrently on the caller's stream
    and a side stream (the default for long problems); the result is bitwise the
    single-sequence one, square and chunked-KV."""
    g = torch.Generator(device="cpu").manual_seed(23 + T + q_frames)
    frames, h, w = 7, 30, 52
    q = torch.randn(1, 4, q_frames * h * w, 128, generator=g).to(cuda, torch.bfloat16)
    k, v = (torch.randn(1, 4, frames * h * w, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(2))
    plan = _sf_plan(frames, h, w)
    low = pk.lower_chunked(plan, q_frames)
    ref = ops.forward(q, k, v, low, T, split=False)
    out = ops.forward(q, k, v, low, T, split=True)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_batch_split_concurrent_halves_bitwise(cuda):
    """With B even the concurrent halves are halves of the batch (odd head count here)."""
    g = torch.Generator(device="cpu").manual_seed(29)
    q, k, v = (torch.randn(2, 3, 4680, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    low = pk.lower_square(_sf_plan())
    ref = ops.forward(q, k, v, low, 1, split=False)
    out = ops.forward(q, k, v, low, 1, split=True)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_head_split_is_graph_capturable(cuda):
    """The side-stream fork / join of the concurrent halves records into a CUDA graph
    (the capture stream's side stream is created by an eager call on that stream first;
    the library never creates streams inside a capture)."""
    g = torch.Generator(device="cpu").manual_seed(31)
    q, k, v = (torch.randn(1, 4, 4680, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    low = pk.lower_square(_sf_plan())
    out = torch.empty_like(q)
    ref = ops.forward(q, k, v, low, 1, split=False)
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        ops.forward(q, k, v, low, 1, out=out, split=True)   # creates cap's side stream
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=cap):
        ops.forward(q, k, v, low, 1, out=out, split=True)
    out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_split_side_streams_are_per_caller_stream(cuda):
    """Two caller streams each get their own side stream: interleaved split forwards on
    both streams give each stream's own result (no shared fork/join events)."""
    g = torch.Generator(device="cpu").manual_seed(37)
    qa, ka, va, qb, kb, vb = (torch.randn(1, 4, 4680, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(6))
    low = pk.lower_square(_sf_plan())
    ra = ops.forward(qa, ka, va, low, 1, split=False)
    rb = ops.forward(qb, kb, vb, low, 1, split=False)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    oa, ob = torch.empty_like(qa), torch.empty_like(qb)
    for s_ in (sa, sb):
        s_.wait_stream(torch.cuda.current_stream())
    for _ in range(4):
        with torch.cuda.stream(sa):
            ops.forward(qa, ka, va, low, 1, out=oa, split=True)
        with torch.cuda.stream(sb):
            ops.forward(qb, kb, vb, low, 1, out=ob, split=True)
    torch.cuda.synchronize()
    assert torch.equal(oa, ra) and torch.equal(ob, rb)


@pytest.mark.parametrize("T", [1, 2])
def test_permuted_aligned_configs_gathered(cuda, T):
    """Every aligned (b1, b2) configuration of a 3 x 30 x 52 grid (enumerate_aligned_configs,
    layout.py:252-276) -- including the permuted ones whose tile rows are not contiguous token
    runs ((w, fh), (hw, f), (fw, h), (h, fw)): those run gathered into slot order on the
    tensor cores -- against the oracle, at T = 1 and 2 (the alpha_R hand-off steps over
    rows l in chunks of 128 where s1 > 128)."""
    shape = pk.VideoShape(3, 30, 52)
    g = torch.Generator(device="cpu").manual_seed(21 + T)
    q, k, v = (torch.randn(1, 1, shape.n, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    seen = 0
    for cfg in pk.enumerate_aligned_configs(shape):
        low = pk.lower_square(cfg)
        assert ops.selected_path(q, k, v, low, T) == "tcgen05", (cfg.g1, cfg.g2)
        out = ops.forward(q, k, v, low, T)
        ref = _oracle_heads(q, k, v, low, T)
        err = orc.rel_l2(out.float().cpu().numpy(), ref)
        assert err < BF16_TOL, (cfg.g1, cfg.g2, err)
        seen += 1
    assert seen == 6


@pytest.mark.parametrize("T", [2, 3])
def test_factor_export_rows_beyond_128(cuda, T):
    """Untiled (fh, w) plan with s1 = 150 > 128 rows per tile: the refinement hand-off and
    the L' export step over rows l in chunks of 128 on the tensor cores; output and both
    factors against the oracle."""
    shape = pk.VideoShape(5, 30, 52)
    low = pk.lower_square(pk.aligned_config(shape, ("f", "h")))
    assert low.s1 == 150
    g = torch.Generator(device="cpu").manual_seed(61 + T)
    q, k, v = (torch.randn(1, 1, shape.n, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))
    assert ops.selected_path(q, k, v, low, T, return_factors=True) == "tcgen05"
    out, lf, rf = ops.forward(q, k, v, low, T, return_factors=True)
    qn, kn, vn = (x[0, 0].float().cpu().numpy().astype(np.float64) for x in (q, k, v))
    idx = np.arange(low.n_q)
    L, R, o = orc.forward_phi(qn, kn, vn, idx, idx, low.c1_q, low.c1_kv, low.c2, low.s1, low.s2, T)
    assert orc.rel_l2(out[0, 0].float().cpu().numpy(), o) < BF16_TOL
    assert orc.rel_l2(lf[0, 0].cpu().numpy(), L) < BF16_TOL
    assert orc.rel_l2(rf[0, 0].cpu().numpy(), R) < BF16_TOL
