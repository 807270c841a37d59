"""Fixtures for the verification path (MNR1 containers, densify, per-iteration traces)
from the UNMODIFIED reference (factors.py:86-298, solver.py:114-254):

    python tests/golden/make_verify_goldens.py      # in the build container

Writes verify_goldens.npz and mnr1_{untiled,tiled}.bin next to this file.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from monarchbench import factors as rf  # noqa: E402
from monarchbench import solver as rs  # noqa: E402
from monarchbench.layout import VideoShape, aligned_config, make_tile_plan  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(11)
out = {}
shape = VideoShape(2, 4, 6)
q, k, v = (rng.standard_normal((shape.n, 8)) for _ in range(3))
prob = rs.AttentionProblem(q, k, v, shape)
out["q"], out["k"], out["v"] = q, k, v
cfg = aligned_config(shape, ("f", "h"))
plan = make_tile_plan(shape, cfg, (1, 2, 6))
traced = rs.SolverConfig(iterations=3, trace_objective=True, trace_mse=True)
fu, tu = rs.solve(prob, cfg, traced)
ft, tt = rs.solve_tiled(prob, plan, traced)
out["untiled_objectives"], out["untiled_mses"] = np.array(tu.objectives), np.array(tu.mses)
out["tiled_objectives"], out["tiled_mses"] = np.array(tt.objectives), np.array(tt.mses)
out["untiled_dense"] = rf.densify(fu)
out["tiled_dense"] = rf.densify_tiled(ft)
out["tiled_approx_token_order"] = rs.approx_attention_matrix(ft)
out["tiled_objective"] = np.array(rs.objective(ft, q, k))
rf.save_factors(fu, os.path.join(HERE, "mnr1_untiled.bin"))
rf.save_factors(ft, os.path.join(HERE, "mnr1_tiled.bin"))
np.savez_compressed(os.path.join(HERE, "verify_goldens.npz"), **out)
print({k_: np.asarray(v_).shape for k_, v_ in out.items()})
