"""Pin the CPU oracle against golden vectors from the unmodified reference.

tests/golden/goldens.npz was produced by tests/golden/make_goldens.py, which
runs monarchbench.solve / solve_tiled + attention_output (solver.py:114-217).
"""

import numpy as np
import pytest

from cases import case_inputs, oracle_lowering
from oracle import monarch_oracle as orc


def _names(goldens):
    return [m["name"] for m in goldens[0]]


def test_manifest_covers_hot_path_variants(goldens):
    manifest, _ = goldens
    kinds = {m["kind"] for m in manifest}
    assert kinds == {"solve", "tiled", "chunk"}
    assert any(m.get("T", 1) >= 3 for m in manifest)
    assert any(m["config"][0] == "raw" for m in manifest)
    assert any(m["name"].startswith("c1_") for m in manifest)


def test_oracle_matches_reference_goldens(goldens):
    manifest, data = goldens
    worst = 0.0
    for meta in manifest:
        q, k, v = case_inputs(meta, data)
        oq, ok, c1q, c1k, c2, s1, s2 = oracle_lowering(meta)
        L, R, out = orc.forward_phi(q, k, v, oq, ok, c1q, c1k, c2, s1, s2, meta["T"])
        ref_out = data[f"{meta['name']}/out"]
        tol = 1e-6 if meta.get("input_dtype") == "float32" else 1e-10
        diff = np.abs(out - ref_out).max()
        assert diff < tol, (meta["name"], diff)
        if f"{meta['name']}/L" in data:
            assert np.abs(L - data[f"{meta['name']}/L"]).max() < 1e-10, meta["name"]
            assert np.abs(R - data[f"{meta['name']}/R"]).max() < 1e-10, meta["name"]
        worst = max(worst, diff)
    assert worst < 1e-6


def test_dense_degenerate_is_exact_attention(goldens):
    # (N, 1) configs and (1,1,1) neighborhoods reduce to softmax(QK^T/sqrt d) V
    manifest, data = goldens
    for name in ("dense_N1", "nbhd_2x2x4_n111_T1"):
        meta = next(m for m in manifest if m["name"] == name)
        q, k, v = case_inputs(meta, data)
        oq, ok, c1q, c1k, c2, s1, s2 = oracle_lowering(meta)
        _, _, out = orc.forward_phi(q, k, v, oq, ok, c1q, c1k, c2, s1, s2, 1)
        assert np.abs(out - orc.dense_attention(q, k, v)).max() < 1e-8


def test_chunked_kv_rect_matches_square_embedding():
    # query tiles are independent (solver.py:184-195): rows of the query frames of
    # the square problem equal the rectangular result for any padding rows.
    rng = np.random.default_rng(5)
    f, fq, h, w, d = 4, 2, 3, 4, 6
    shape = (f, h, w)
    order = orc.order_neighborhood(shape, (1, h, w))
    k = rng.standard_normal((f * h * w, d))
    v = rng.standard_normal((f * h * w, d))
    q = rng.standard_normal((fq * h * w, d))
    outs = []
    for _ in range(2):
        pad = rng.standard_normal(((f - fq) * h * w, d))
        _, _, o = orc.forward_phi(np.vstack([pad, q]), k, v, order, order, f, f, 1, h, w, 2)
        outs.append(o[(f - fq) * h * w:])
    _, _, rect = orc.forward_phi(q, k, v, order[(f - fq) * h * w:] - (f - fq) * h * w, order,
                                 fq, f, 1, h, w, 2)
    assert np.abs(outs[0] - outs[1]).max() < 1e-12
    assert np.abs(rect - outs[0]).max() < 1e-12


@pytest.mark.parametrize("t", [1, 2, 3])
def test_factors_row_stochastic(t):
    rng = np.random.default_rng(t)
    c1, c2, s1, s2, d = 2, 2, 3, 4, 5
    n = c1 * c2 * s1 * s2
    q, k, v = (rng.standard_normal((n, d)) for _ in range(3))
    idx = np.arange(n)
    L, R, _ = orc.forward_phi(q, k, v, idx, idx, c1, c1, c2, s1, s2, t)
    assert np.abs(R.sum(-1) - 1).max() < 1e-12
    assert np.abs(L.sum(axis=(2, 3, 6)) - 1).max() < 1e-12
