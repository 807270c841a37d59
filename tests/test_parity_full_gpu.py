"""Full-size parity of every configuration bench.py reports, and bf16 factor export.

Each bench configuration (BASELINE.json C2-C4, bench.py CONFIGS) runs at its full
token count on one or two heads through the C ABI and is compared with the fp64
oracle (oracle/monarch_oracle.py, pinned to the reference goldens) at the
north-star bf16 tolerance: 2e-2 relative L2 on the output and, where exported,
on both factors L' and R' (factors.py:57-79 layout).  The oracle takes 1-11 s
per N=32760 head on one host core.
"""

import zlib

import numpy as np
import pytest
import torch

import paper_2602_12271_b200 as pk
from paper_2602_12271_b200 import ops
from oracle import monarch_oracle as orc

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _plan(frames, nb, h=30, w=52):
    shape = pk.VideoShape(frames, h, w)
    if nb is None:
        return pk.aligned_config(shape, ("f", "h"))
    if nb == "mis":
        return pk.config_from_sizes(shape, 1260, 26)
    return pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), nb)


def _lower(plan, frames, q_frames):
    if q_frames != frames:
        return pk.lower_chunked(plan, q_frames)
    return pk.lower_square(plan)


def _inputs(seed, heads, nq, nk, dev):
    g = torch.Generator(device="cpu").manual_seed(seed)
    q = torch.randn(1, heads, nq, 128, generator=g).to(dev, torch.bfloat16)
    k = torch.randn(1, heads, nk, 128, generator=g).to(dev, torch.bfloat16)
    v = torch.randn(1, heads, nk, 128, generator=g).to(dev, torch.bfloat16)
    return q, k, v


def _oracle(q, k, v, low, T, b=0, h=0):
    qn, kn, vn = (x[b, h].float().cpu().numpy().astype(np.float64) for x in (q, k, v))
    oq = np.arange(low.n_q) if low.q_order is None else low.q_order
    ok = np.arange(low.n_kv) if low.kv_order is None else low.kv_order
    return orc.forward_phi(qn, kn, vn, oq, ok, low.c1_q, low.c1_kv, low.c2, low.s1, low.s2, T)


# (bench config, frames_kv, frames_q, plan, T): every line bench.py can print, at full size
FULL = [
    ("n32k", 21, 21, (1, 30, 52), 1),
    ("n32k_3hw", 21, 21, (3, 30, 52), 1),
    ("n32k_fhw", 21, 21, None, 1),
    ("n32k_mis", 21, 21, "mis", 1),
    ("kv21", 21, 3, (1, 30, 52), 1),
    ("kv21_T2", 21, 3, (1, 30, 52), 2),
    ("kv21_T3", 21, 3, (1, 30, 52), 3),
    ("kv21_3hw", 21, 3, (3, 30, 52), 1),
    ("kv21_3hw_T2", 21, 3, (3, 30, 52), 2),
    ("kv21_3hw_T3", 21, 3, (3, 30, 52), 3),
    ("sf_T3", 3, 3, (1, 30, 52), 3),
    ("sf3hw_T3", 3, 3, (3, 30, 52), 3),
]


@pytest.mark.parametrize("name,frames,q_frames,nb,T", FULL, ids=[c[0] for c in FULL])
def test_bench_config_full_size(cuda, name, frames, q_frames, nb, T):
    """One head of the configuration on the tcgen05 path vs the oracle."""
    plan = _plan(frames, nb)
    low = _lower(plan, frames, q_frames)
    q, k, v = _inputs(zlib.crc32(name.encode()) % 1000, 1, low.n_q, low.n_kv, cuda)
    assert ops.selected_path(q, k, v, low, T) == "tcgen05", name
    out = ops.forward(q, k, v, low, T)
    _, _, ref = _oracle(q, k, v, low, T)
    err = orc.rel_l2(out[0, 0].float().cpu().numpy(), ref)
    assert err < BF16_TOL, (name, err)


SPLIT = [("n32k", 21, 21, (1, 30, 52), 1), ("kv21_T2", 21, 3, (1, 30, 52), 2),
         ("n32k_3hw", 21, 21, (3, 30, 52), 1)]


@pytest.mark.parametrize("name,frames,q_frames,nb,T", SPLIT, ids=[c[0] for c in SPLIT])
def test_concurrent_halves_full_size(cuda, name, frames, q_frames, nb, T):
    """The concurrent head halves (the default for these sizes) at full size: both
    halves match the oracle, and the split result equals the unsplit one bitwise."""
    plan = _plan(frames, nb)
    low = _lower(plan, frames, q_frames)
    q, k, v = _inputs(7 + T, 2, low.n_q, low.n_kv, cuda)
    out = ops.forward(q, k, v, low, T, split=True)
    ref1 = ops.forward(q, k, v, low, T, split=False)
    torch.cuda.synchronize()
    assert torch.equal(out, ref1)
    for h in range(2):
        _, _, ref = _oracle(q, k, v, low, T, 0, h)
        assert orc.rel_l2(out[0, h].float().cpu().numpy(), ref) < BF16_TOL, (name, h)


FACT = [("sf", 3, 3, (1, 30, 52), 1, 2), ("sf_T2", 3, 3, (1, 30, 52), 2, 2), ("sf_T3", 3, 3, (1, 30, 52), 3, 1),
        ("sf3hw", 3, 3, (3, 30, 52), 1, 1), ("sf3hw_T2", 3, 3, (3, 30, 52), 2, 1),
        ("kv7_T2", 7, 3, (1, 30, 52), 2, 1), ("kv6_3hw", 6, 3, (3, 30, 52), 1, 1),
        ("fh_s1_60", 2, 2, None, 1, 1)]


@pytest.mark.parametrize("name,frames,q_frames,nb,T,H", FACT, ids=[c[0] for c in FACT])
def test_bf16_factor_export_tensor_cores(cuda, name, frames, q_frames, nb, T, H):
    """bf16 forward with factor export stays on the tcgen05 path: R' comes from the
    last row stage's softmax, L' from the statistics pass + the alpha kernel in
    export mode; output, L' and R' all within 2e-2 of the fp64 oracle."""
    plan = _plan(frames, nb)
    low = _lower(plan, frames, q_frames)
    q, k, v = _inputs(101 + T, H, low.n_q, low.n_kv, cuda)
    assert ops.selected_path(q, k, v, low, T, return_factors=True) == "tcgen05"
    out, lf, rf = ops.forward(q, k, v, low, T, return_factors=True)
    plain = ops.forward(q, k, v, low, T)
    for h in range(H):
        L, R, ref = _oracle(q, k, v, low, T, 0, h)
        assert orc.rel_l2(out[0, h].float().cpu().numpy(), ref) < BF16_TOL, name
        assert orc.rel_l2(lf[0, h].cpu().numpy(), L) < BF16_TOL, name
        assert orc.rel_l2(rf[0, h].cpu().numpy(), R) < BF16_TOL, name
    # factor export does not change the output path's arithmetic beyond the extra passes
    assert orc.rel_l2(out.float().cpu().numpy(), plain.float().cpu().numpy()) < 1e-2
    # both factors are row-stochastic (solver.py:189, 195)
    assert (rf.sum(-1) - 1).abs().max().item() < 1e-4
    assert (lf.sum(dim=(4, 5, 8)) - 1).abs().max().item() < 1e-3


def test_solve_tiled_bf16_reaches_tensor_cores(cuda):
    """The reference API with bfloat16 torch inputs (solve_tiled + attention_output)
    runs on tcgen05 and returns reference-layout factors within 2e-2 of the oracle."""
    shape = pk.VideoShape(3, 30, 52)
    plan = _plan(3, (1, 30, 52))
    g = torch.Generator(device="cpu").manual_seed(5)
    q, k, v = (torch.randn(shape.n, 128, generator=g).to(torch.bfloat16) for _ in range(3))
    low = pk.lower_square(plan)
    assert ops.selected_path(q[None, None].to(cuda), k[None, None].to(cuda), v[None, None].to(cuda), low, 2,
                             return_factors=True) == "tcgen05"
    fac, _ = pk.solve_tiled(pk.AttentionProblem(q, k, v, shape), plan, pk.SolverConfig(iterations=2))
    L, R, ref = _oracle(q[None, None], k[None, None], v[None, None], low, 2)
    assert orc.rel_l2(fac.l_blocks, L) < BF16_TOL
    assert orc.rel_l2(fac.r_blocks, R) < BF16_TOL
    out = pk.attention_output(fac, v.float().numpy())
    assert orc.rel_l2(out, ref) < BF16_TOL


# Long tile rows (s2 > 64) -> the online-softmax row stage (tc_row_flash): the paper's 720p
# latent grid (h, w) = (45, 80) and the aligned (f, hw) configuration.
FLASH = [
    ("sf720_hw", (3, 45, 80), ("nb", (1, 45, 80)), None, 1, 2),
    ("sf720_hw_T2", (3, 45, 80), ("nb", (1, 45, 80)), None, 2, 1),
    ("sf720_3hw", (3, 45, 80), ("nb", (3, 45, 80)), None, 1, 1),
    ("kv9_720_hw", (9, 45, 80), ("nb", (1, 45, 80)), 3, 1, 1),
    ("n32k_f", (21, 30, 52), ("aligned", ("f",)), None, 1, 1),
    ("n32k_f_T2", (21, 30, 52), ("aligned", ("f",)), None, 2, 1),
    ("raw_b2_200", (4, 10, 60), ("raw", 12, 200), None, 1, 2),
    ("raw_b2_100_T3", (2, 10, 30), ("raw", 6, 100), None, 3, 1),
]


def _plan_kind(fhw, kind):
    shape = pk.VideoShape(*fhw)
    if kind[0] == "nb":
        return pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), kind[1])
    if kind[0] == "aligned":
        return pk.aligned_config(shape, kind[1])
    return pk.config_from_sizes(shape, kind[1], kind[2])


@pytest.mark.parametrize("name,fhw,kind,q_frames,T,H", FLASH, ids=[c[0] for c in FLASH])
def test_long_tile_rows_flash_row_stage(cuda, name, fhw, kind, q_frames, T, H):
    plan = _plan_kind(fhw, kind)
    low = pk.lower_chunked(plan, q_frames) if q_frames else pk.lower_square(plan)
    assert low.s2 > 64
    q, k, v = _inputs(zlib.crc32(name.encode()) % 1000, H, low.n_q, low.n_kv, cuda)
    assert ops.selected_path(q, k, v, low, T) == "tcgen05", name
    out = ops.forward(q, k, v, low, T)
    for h in range(H):
        _, _, ref = _oracle(q, k, v, low, T, 0, h)
        err = orc.rel_l2(out[0, h].float().cpu().numpy(), ref)
        assert err < BF16_TOL, (name, h, err)


@pytest.mark.parametrize("g1", [("f", "h"), ("w",), ("f",), ("h", "w"), ("f", "w"), ("h",)])
def test_all_aligned_configs_n32k_tensor_cores(cuda, g1):
    """All six aligned (b1, b2) configurations of the N=32760 (21, 30, 52) grid
    (enumerate_aligned_configs, layout.py:252-276; BASELINE.json config 4's aligned
    sweep) select the tensor-core path -- the permuted ones gathered into slot order --
    and match the oracle on one head at T = 1."""
    shape = pk.VideoShape(21, 30, 52)
    low = pk.lower_square(pk.aligned_config(shape, g1))
    q, k, v = _inputs(zlib.crc32(repr(g1).encode()) & 0xFFFF, 1, shape.n, shape.n, cuda)
    assert ops.selected_path(q, k, v, low, 1) == "tcgen05", g1
    out = ops.forward(q, k, v, low, 1)
    _, _, ref = _oracle(q, k, v, low, 1)
    err = orc.rel_l2(out[0, 0].float().cpu().numpy(), ref)
    assert err < BF16_TOL, (g1, err)


@pytest.mark.parametrize("name,g1,T", [("n32k_fhw", ("f", "h"), 2), ("n32k_hw", ("h", "w"), 2),
                                       ("n32k_fw", ("f", "w"), 3)])
def test_iterations_rows_beyond_128_n32k(cuda, name, g1, T):
    """T >= 2 for untiled N=32760 plans with s1 = 630, 1560, 1092 rows per tile (the alpha_R
    hand-off over rows l in steps of 128) on the tensor cores, against the oracle."""
    shape = pk.VideoShape(21, 30, 52)
    low = pk.lower_square(pk.aligned_config(shape, g1))
    assert low.s1 > 128
    q, k, v = _inputs(zlib.crc32(name.encode()) & 0xFFFF, 1, shape.n, shape.n, cuda)
    assert ops.selected_path(q, k, v, low, T) == "tcgen05", name
    out = ops.forward(q, k, v, low, T)
    _, _, ref = _oracle(q, k, v, low, T)
    err = orc.rel_l2(out[0, 0].float().cpu().numpy(), ref)
    assert err < BF16_TOL, (name, err)
