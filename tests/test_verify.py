"""Verification path: MNR1 containers pinned to reference bytes (CPU), densify /
objective / per-iteration traces against reference fixtures (GPU).
Fixtures: tests/golden/make_verify_goldens.py (unmodified reference)."""
import io
import os

import numpy as np
import pytest

import paper_2602_12271_b200 as pk
from paper_2602_12271_b200 import verify

G = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def vg():
    return np.load(os.path.join(G, "verify_goldens.npz"))


@pytest.mark.parametrize("name", ["mnr1_untiled.bin", "mnr1_tiled.bin"])
def test_mnr1_round_trip_reproduces_reference_bytes(name):
    raw = open(os.path.join(G, name), "rb").read()
    fac = verify.load_factors(os.path.join(G, name))
    buf = io.BytesIO()
    verify.save_factors(fac, buf)
    assert buf.getvalue() == raw
    assert fac.n == 48
    if name == "mnr1_tiled.bin":
        assert isinstance(fac, pk.TiledMonarchFactors) and (fac.plan.c1, fac.plan.c2) == (4, 1)


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"MNR2" + b[4:], "bad magic"),
    (lambda b: b[:12], "truncated header"),
    (lambda b: b[:4] + (7).to_bytes(4, "little") + b[8:], "unknown kind"),
    (lambda b: b[:-8], "expected"),
])
def test_mnr1_malformed(mutate, msg):
    raw = open(os.path.join(G, "mnr1_tiled.bin"), "rb").read()
    with pytest.raises(pk.FactorError, match=msg):
        verify.load_factors(io.BytesIO(mutate(raw)))


def test_keep_workspace_still_refused():
    shape = pk.VideoShape(1, 2, 3)
    prob = pk.AttentionProblem(np.ones((6, 4)), np.ones((6, 4)), np.ones((6, 4)), shape)
    with pytest.raises(pk.SolverError, match="keep_workspace"):
        pk.solve(prob, pk.aligned_config(shape, ("f", "h")), pk.SolverConfig(keep_workspace=True))


@pytest.mark.gpu
def test_densify_reference_factors(cuda, vg):
    fu = verify.load_factors(os.path.join(G, "mnr1_untiled.bin"))
    ft = verify.load_factors(os.path.join(G, "mnr1_tiled.bin"))
    np.testing.assert_allclose(verify.densify(fu), vg["untiled_dense"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(verify.densify_tiled(ft), vg["tiled_dense"], rtol=0, atol=1e-12)
    eye = verify.densify(verify.identity_factors(6, 8))
    np.testing.assert_array_equal(eye, np.eye(48))
    with pytest.raises(pk.FactorError, match="verification path"):
        verify.densify(verify.identity_factors(65, 64))


@pytest.mark.gpu
def test_traces_objective_and_approx_match_reference(cuda, vg):
    shape = pk.VideoShape(2, 4, 6)
    prob = pk.AttentionProblem(vg["q"], vg["k"], vg["v"], shape)
    cfg = pk.aligned_config(shape, ("f", "h"))
    plan = pk.make_tile_plan(shape, cfg, (1, 2, 6))
    traced = pk.SolverConfig(iterations=3, trace_objective=True, trace_mse=True)
    fu, tu = pk.solve(prob, cfg, traced)
    ft, tt = pk.solve_tiled(prob, plan, traced)
    np.testing.assert_allclose(tu.objectives, vg["untiled_objectives"], rtol=1e-5)
    np.testing.assert_allclose(tt.objectives, vg["tiled_objectives"], rtol=1e-5)
    np.testing.assert_allclose(tu.mses, vg["untiled_mses"], rtol=1e-3, atol=1e-12)
    np.testing.assert_allclose(tt.mses, vg["tiled_mses"], rtol=1e-3, atol=1e-12)
    np.testing.assert_allclose(verify.objective(ft, vg["q"], vg["k"]), float(vg["tiled_objective"]), rtol=1e-5)
    np.testing.assert_allclose(verify.approx_attention_matrix(ft), vg["tiled_approx_token_order"], atol=1e-5)
