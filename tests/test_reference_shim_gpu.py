"""The reference package itself, with its hot path routed through the B200 C ABI.

``integration/monarchbench_b200.install`` patches ``solve`` / ``solve_tiled`` /
``attention_output`` of the unmodified reference installed under
``baseline/_ref`` (never /root/reference: it does not exist on the GPU box).
The assertions are the reference's own hot-path properties
(pkg/tests/test_solver.py:41-163), with the reference's float64 helpers
(``reference_solve``, ``reference_solve_tiled``, ``dense_attention``,
``densify``, ``approx_attention_matrix``) as the expected values.  The device
computes in fp32, so closeness is asserted at fp32 round-off (absolute 2e-5 on
entries of magnitude <= ~3, the north-star 1e-4 relative L2 on outputs) instead
of the reference's float64 1e-10..1e-13; the structural properties (bitwise
trivial tiling, row-stochastic factors) are asserted as in the reference.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu

ATOL = 2e-5


@pytest.fixture(scope="module")
def mb(cuda):
    if not os.path.isdir(os.path.join(REF, "monarchbench")):
        pytest.skip("baseline/_ref (the installed reference) is absent")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import monarchbench

    from integration import monarchbench_b200

    monarchbench_b200.install(monarchbench)
    yield monarchbench
    monarchbench_b200.uninstall(monarchbench)


def _line(mb, b1, b2):
    return mb.BlockConfig(mb.VideoShape(1, b1, b2), b1, b2, ("f", "h"), ("w",))


def _problem(mb, rng, shape, d=4):
    n = shape.n
    return mb.AttentionProblem(rng.standard_normal((n, d)), rng.standard_normal((n, d)),
                               rng.standard_normal((n, d)), shape)


def _rel(x, ref):
    return float(np.linalg.norm(np.asarray(x) - ref) / np.linalg.norm(ref))


def test_patched_solver_is_the_b200_path(mb):
    from integration import monarchbench_b200

    assert mb.solve.__code__.co_filename == monarchbench_b200.__file__
    assert mb.solver.solve_tiled.__code__.co_filename == monarchbench_b200.__file__


def test_first_iteration_r_is_blockwise_softmax(mb):
    """test_solver.py:41-51: with identity L the R update is softmax_i(Q[k,j].K[k,i])."""
    rng = np.random.default_rng(0)
    b1, b2, d = 3, 4, 5
    problem = _problem(mb, rng, mb.VideoShape(1, b1, b2), d)
    factors, _ = mb.solve(problem, _line(mb, b1, b2), mb.SolverConfig(iterations=1))
    qb = (problem.q * problem.logit_scale).reshape(b1, b2, d)
    kb = problem.k.reshape(b1, b2, d)
    expected = mb.softmax_rows(np.einsum("kjv,kiv->kji", qb, kb))
    assert np.abs(factors.r_blocks - expected).max() < ATOL


def test_single_block_degenerate_is_exact_attention(mb):
    """test_solver.py:66-74: config (N, 1) reproduces dense attention."""
    rng = np.random.default_rng(1)
    shape = mb.VideoShape(1, 9, 1)
    problem = _problem(mb, rng, shape)
    factors, _ = mb.solve(problem, mb.aligned_config(shape, ("f", "h")), mb.SolverConfig(iterations=1))
    a, out = mb.dense_attention(problem)
    assert np.abs(mb.densify(factors) - a).max() < ATOL
    assert np.abs(mb.attention_output(factors, problem.v) - out).max() < ATOL


@pytest.mark.parametrize("t_steps", [1, 5, 10])
def test_untiled_matches_reference_loops(mb, t_steps):
    """test_solver.py:76-87: factors and output vs the reference's explicit loops."""
    from monarchbench.reference import reference_output, reference_solve

    rng = np.random.default_rng(2 + t_steps)
    b1, b2, d = 6, 3, 4
    problem = _problem(mb, rng, mb.VideoShape(1, b1, b2), d)
    factors, _ = mb.solve(problem, _line(mb, b1, b2), mb.SolverConfig(iterations=t_steps))
    ref_l, ref_r = reference_solve(problem.q * problem.logit_scale, problem.k, b1, b2, t_steps)
    assert np.abs(factors.l_blocks - ref_l).max() < ATOL
    assert np.abs(factors.r_blocks - ref_r).max() < ATOL
    out = mb.attention_output(factors, problem.v)
    assert _rel(out, reference_output(ref_l, ref_r, problem.v, b1, b2)) < 1e-4


def test_deterministic_bitwise(mb):
    rng = np.random.default_rng(3)
    problem = _problem(mb, rng, mb.VideoShape(2, 2, 3))
    cfg = mb.aligned_config(mb.VideoShape(2, 2, 3), ("f", "h"))
    f1, _ = mb.solve(problem, cfg, mb.SolverConfig(iterations=3))
    f2, _ = mb.solve(problem, cfg, mb.SolverConfig(iterations=3))
    assert np.array_equal(f1.l_blocks, f2.l_blocks) and np.array_equal(f1.r_blocks, f2.r_blocks)


def test_row_stochastic_densified(mb):
    """test_solver.py:98-104 for the permuted aligned configs."""
    rng = np.random.default_rng(4)
    shape = mb.VideoShape(2, 3, 3)
    problem = _problem(mb, rng, shape)
    for g1 in (("f", "h"), ("w",), ("f",)):
        factors, _ = mb.solve(problem, mb.aligned_config(shape, g1), mb.SolverConfig(iterations=2))
        assert np.abs(mb.densify(factors).sum(axis=1) - 1.0).max() <= 1e-5


def test_errors_are_the_reference_classes(mb):
    rng = np.random.default_rng(5)
    problem = _problem(mb, rng, mb.VideoShape(2, 3, 3))
    with pytest.raises(mb.solver.SolverError):
        mb.solve(problem, _line(mb, 3, 6), mb.SolverConfig())
    with pytest.raises(mb.solver.SolverError):
        mb.solve(problem, mb.aligned_config(mb.VideoShape(2, 3, 3), ("f", "h")),
                 mb.SolverConfig(keep_workspace=True))


def test_trivial_tiling_bitwise_equal_to_untiled(mb):
    """test_solver.py:124-133: TilePlan(cfg, 1, 1) gives the untiled factors bitwise,
    and the same per-refinement objectives."""
    rng = np.random.default_rng(6)
    b1, b2 = 4, 3
    problem = _problem(mb, rng, mb.VideoShape(1, b1, b2))
    cfg = _line(mb, b1, b2)
    fu, tu = mb.solve(problem, cfg, mb.SolverConfig(iterations=3, trace_objective=True))
    ft, tt = mb.solve_tiled(problem, mb.TilePlan(cfg, 1, 1), mb.SolverConfig(iterations=3, trace_objective=True))
    assert np.array_equal(ft.l_blocks[0, 0, 0, 0], fu.l_blocks)
    assert np.array_equal(ft.r_blocks[0, 0, 0, 0], fu.r_blocks)
    assert len(tu.objectives) == 3 and tt.objectives == tu.objectives


def test_unit_neighborhoods_reproduce_dense_attention(mb):
    """test_solver.py:135-143."""
    rng = np.random.default_rng(7)
    shape = mb.VideoShape(2, 2, 4)
    problem = _problem(mb, rng, shape)
    plan = mb.make_tile_plan(shape, mb.aligned_config(shape, ("f", "h")), (1, 1, 1))
    factors, _ = mb.solve_tiled(problem, plan, mb.SolverConfig(iterations=1))
    a, out = mb.dense_attention(problem)
    assert np.abs(mb.approx_attention_matrix(factors) - a).max() < ATOL
    assert np.abs(mb.attention_output(factors, problem.v) - out).max() < ATOL


@pytest.mark.parametrize("t_steps", [1, 3])
def test_tiled_matches_reference_loops(mb, t_steps):
    """test_solver.py:145-163: permuted neighborhood plan vs reference_solve_tiled."""
    from monarchbench.reference import reference_output_tiled, reference_solve_tiled

    rng = np.random.default_rng(8 + t_steps)
    shape = mb.VideoShape(2, 4, 4)
    problem = _problem(mb, rng, shape)
    plan = mb.make_tile_plan(shape, mb.aligned_config(shape, ("f", "h")), (1, 4, 4))
    assert (plan.c1, plan.c2) == (2, 1)
    factors, _ = mb.solve_tiled(problem, plan, mb.SolverConfig(iterations=t_steps))
    order = plan.ordering().to_phi()
    ref_l, ref_r = reference_solve_tiled((problem.q * problem.logit_scale)[order], problem.k[order], 8, 4, 2, 1,
                                         t_steps)
    assert np.abs(factors.l_blocks - ref_l).max() < ATOL
    assert np.abs(factors.r_blocks - ref_r).max() < ATOL
    out = mb.attention_output(factors, problem.v)
    ref_out = reference_output_tiled(ref_l, ref_r, problem.v[order], 8, 4, 2, 1)
    unperm = np.empty_like(ref_out)
    unperm[order] = ref_out
    assert _rel(out, unperm) < 1e-4


def test_tiled_row_stochastic(mb):
    rng = np.random.default_rng(10)
    shape = mb.VideoShape(2, 4, 4)
    problem = _problem(mb, rng, shape)
    plan = mb.make_tile_plan(shape, mb.aligned_config(shape, ("f", "h")), (2, 2, 2))
    factors, _ = mb.solve_tiled(problem, plan, mb.SolverConfig(iterations=2))
    assert np.abs(mb.densify_tiled(factors).sum(axis=1) - 1.0).max() <= 1e-5
