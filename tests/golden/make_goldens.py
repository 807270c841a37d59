"""Generate golden vectors for the hot path from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_goldens.py

It imports ``monarchbench`` from /root/reference/pkg/src (never copied), runs
``solve`` / ``solve_tiled`` + ``attention_output`` (solver.py:114-217) on
seeded inputs, and writes ``goldens.npz`` + ``manifest.json`` next to this
file.  The chunked-KV cases use the square embedding: the
reference solves the full f_kv-frame problem with arbitrary query rows in the
non-query frames, and the rows/factors of the last f_q frames are the
rectangular result.  The GPU box never reads /root/reference; only the
committed fixtures travel.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import monarchbench as mb  # noqa: E402

    return mb


def main() -> None:
    mb = _ref()
    arrays: dict[str, np.ndarray] = {}
    manifest: list[dict] = []

    def add(name, meta, q, k, v, L, R, out, store_inputs=True):
        meta = dict(meta, name=name)
        if store_inputs:
            arrays[f"{name}/q"] = q
            arrays[f"{name}/k"] = k
            arrays[f"{name}/v"] = v
        else:
            meta["input_sums"] = [float(np.sum(q)), float(np.sum(k)), float(np.sum(v))]
        if L is not None:
            arrays[f"{name}/L"] = L
            arrays[f"{name}/R"] = R
        arrays[f"{name}/out"] = out
        manifest.append(meta)

    def rnd(rng, n, d):
        return rng.standard_normal((n, d))

    # --- A: untiled line configs + tiled line plans (verify.py:163-219 size tables)
    sizes = ((4, 3), (3, 4), (6, 3), (2, 8), (8, 4), (6, 4), (4, 6), (5, 4))
    tiled = ((4, 4, 2, 2), (6, 2, 3, 1), (4, 3, 2, 3), (8, 4, 2, 2), (6, 4, 2, 2),
             (9, 2, 3, 2), (4, 8, 2, 2), (8, 2, 4, 2))
    rng = np.random.default_rng(777)
    for idx, (b1, b2) in enumerate(sizes):
        t, d = int(rng.integers(1, 6)), int(rng.integers(2, 9))
        shape = mb.VideoShape(1, b1, b2)
        q, k, v = rnd(rng, b1 * b2, d), rnd(rng, b1 * b2, d), rnd(rng, b1 * b2, d)
        cfg = mb.BlockConfig(shape, b1, b2, ("f", "h"), ("w",))
        fac, _ = mb.solve(mb.AttentionProblem(q, k, v, shape), cfg, mb.SolverConfig(iterations=t))
        out = mb.attention_output(fac, v)
        add(f"line_untiled_{idx}", dict(kind="solve", shape=[1, b1, b2], config=["fh"], T=t),
            q, k, v, fac.l_blocks[None, None, None, None], fac.r_blocks[None, None, None, None], out)
    for idx, (b1, b2, c1, c2) in enumerate(tiled):
        t, d = int(rng.integers(1, 6)), int(rng.integers(2, 9))
        shape = mb.VideoShape(1, b1, b2)
        q, k, v = rnd(rng, b1 * b2, d), rnd(rng, b1 * b2, d), rnd(rng, b1 * b2, d)
        cfg = mb.BlockConfig(shape, b1, b2, ("f", "h"), ("w",))
        plan = mb.TilePlan(cfg, c1, c2)
        fac, _ = mb.solve_tiled(mb.AttentionProblem(q, k, v, shape), plan, mb.SolverConfig(iterations=t))
        out = mb.attention_output(fac, v)
        add(f"line_tiled_{idx}", dict(kind="tiled", shape=[1, b1, b2], config=["fh"], c=[c1, c2], T=t),
            q, k, v, fac.l_blocks, fac.r_blocks, out)

    # --- B: aligned configs with permuted slot orders (layout.py:218-221), dv != d
    rng = np.random.default_rng(4242)
    shape = mb.VideoShape(2, 3, 4)
    for g1 in (("f", "h"), ("w",), ("f",), ("h", "w"), ("f", "w"), ("h",)):
        q, k, v = rnd(rng, 24, 5), rnd(rng, 24, 5), rnd(rng, 24, 3)
        cfg = mb.aligned_config(shape, g1)
        fac, _ = mb.solve(mb.AttentionProblem(q, k, v, shape), cfg, mb.SolverConfig(iterations=2))
        out = mb.attention_output(fac, v)
        add(f"aligned_{''.join(g1)}", dict(kind="solve", shape=[2, 3, 4], config=list(g1), T=2),
            q, k, v, fac.l_blocks[None, None, None, None], fac.r_blocks[None, None, None, None], out)
        plan = mb.TilePlan(cfg, 1 if cfg.b1 % 2 else 2, 2 if cfg.b2 % 2 == 0 else 1)
        fac, _ = mb.solve_tiled(mb.AttentionProblem(q, k, v, shape), plan, mb.SolverConfig(iterations=2))
        out = mb.attention_output(fac, v)
        add(f"aligned_tiled_{''.join(g1)}",
            dict(kind="tiled", shape=[2, 3, 4], config=list(g1), c=[plan.c1, plan.c2], T=2),
            q, k, v, fac.l_blocks, fac.r_blocks, out)

    # --- C: raw (misaligned) configs (layout.py:224-239) incl. tiled
    rng = np.random.default_rng(99)
    shape = mb.VideoShape(2, 3, 4)
    for (b1, b2, c1, c2) in ((8, 3, 2, 3), (4, 6, 2, 2), (8, 3, 1, 1)):
        cfg = mb.config_from_sizes(shape, b1, b2)
        assert not cfg.aligned
        q, k, v = rnd(rng, 24, 4), rnd(rng, 24, 4), rnd(rng, 24, 4)
        plan = mb.TilePlan(cfg, c1, c2)
        fac, _ = mb.solve_tiled(mb.AttentionProblem(q, k, v, shape), plan, mb.SolverConfig(iterations=3))
        out = mb.attention_output(fac, v)
        add(f"raw_{b1}x{b2}_c{c1}{c2}", dict(kind="tiled", shape=[2, 3, 4], config=["raw", b1, b2],
                                               c=[c1, c2], T=3), q, k, v, fac.l_blocks, fac.r_blocks, out)

    # --- D: neighborhood plans (layout.py:342-351), test_solver.py:135-172 recipes
    rng = np.random.default_rng(8)
    for shp, nb, t, d in (((2, 4, 4), (1, 4, 4), 1, 4), ((2, 4, 4), (1, 4, 4), 3, 4),
                          ((2, 4, 4), (2, 2, 2), 2, 4), ((3, 4, 6), (1, 2, 3), 2, 6),
                          ((2, 2, 4), (1, 1, 1), 1, 4), ((3, 6, 8), (1, 6, 8), 1, 16),
                          ((3, 6, 8), (1, 6, 8), 3, 16), ((4, 6, 8), (2, 3, 4), 2, 8)):
        shape = mb.VideoShape(*shp)
        n = shape.n
        q, k, v = rnd(rng, n, d), rnd(rng, n, d), rnd(rng, n, d)
        plan = mb.make_tile_plan(shape, mb.aligned_config(shape, ("f", "h")), nb)
        fac, _ = mb.solve_tiled(mb.AttentionProblem(q, k, v, shape), plan, mb.SolverConfig(iterations=t))
        out = mb.attention_output(fac, v)
        add(f"nbhd_{'x'.join(map(str, shp))}_n{''.join(map(str, nb))}_T{t}",
            dict(kind="tiled", shape=list(shp), config=["fh"], nbhd=list(nb), T=t),
            q, k, v, fac.l_blocks, fac.r_blocks, out)

    # --- E: dense degenerate (N, 1) (test_solver.py:66-74)
    shape = mb.VideoShape(1, 9, 1)
    q, k, v = rnd(rng, 9, 4), rnd(rng, 9, 4), rnd(rng, 9, 4)
    fac, _ = mb.solve(mb.AttentionProblem(q, k, v, shape), mb.aligned_config(shape, ("f", "h")),
                      mb.SolverConfig())
    add("dense_N1", dict(kind="solve", shape=[1, 9, 1], config=["fh"], T=1), q, k, v,
        fac.l_blocks[None, None, None, None], fac.r_blocks[None, None, None, None],
        mb.attention_output(fac, v))

    # --- F: chunked-KV via the square embedding
    rng = np.random.default_rng(2602)
    for (fkv, fq, h, w, nb, t, d) in ((5, 2, 3, 4, (1, 3, 4), 1, 8), (5, 2, 3, 4, (1, 3, 4), 3, 8),
                                      (6, 2, 4, 4, (2, 2, 2), 2, 6), (4, 1, 3, 5, (1, 3, 5), 2, 8)):
        shape = mb.VideoShape(fkv, h, w)
        nq, nk = fq * h * w, fkv * h * w
        qq, k, v = rnd(rng, nq, d), rnd(rng, nk, d), rnd(rng, nk, d)
        pad = rnd(rng, nk - nq, d)
        plan = mb.make_tile_plan(shape, mb.aligned_config(shape, ("f", "h")), nb)
        fac, _ = mb.solve_tiled(mb.AttentionProblem(np.vstack([pad, qq]), k, v, shape), plan,
                                mb.SolverConfig(iterations=t))
        out = mb.attention_output(fac, v)[nk - nq:]
        c1q = (fq // nb[0]) * (h // nb[1])
        L = fac.l_blocks[-c1q:]
        R = fac.r_blocks[-c1q:]
        add(f"chunk_kv{fkv}_q{fq}_{h}x{w}_n{''.join(map(str, nb))}_T{t}",
            dict(kind="chunk", shape=[fkv, h, w], f_q=fq, config=["fh"], nbhd=list(nb), T=t),
            qq, k, v, L, R, out)

    # --- G: BASELINE config 1 (C1): B=1 H=2 N=1024 (1,32,32) untiled, d=64, fp32 inputs
    rng = np.random.default_rng(0)
    shape = mb.VideoShape(1, 32, 32)
    for head in range(2):
        q = rng.standard_normal((1024, 64)).astype(np.float32)
        k = rng.standard_normal((1024, 64)).astype(np.float32)
        v = rng.standard_normal((1024, 64)).astype(np.float32)
        fac, _ = mb.solve(mb.AttentionProblem(q, k, v, shape), mb.aligned_config(shape, ("f", "h")),
                          mb.SolverConfig(iterations=1))
        out = mb.attention_output(fac, v).astype(np.float32)
        add(f"c1_head{head}", dict(kind="solve", shape=[1, 32, 32], config=["fh"], T=1, seed=0,
                                   head=head, input_dtype="float32"),
            q, k, v, None, None, out, store_inputs=False)

    np.savez_compressed(os.path.join(HERE, "goldens.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print(f"wrote {len(manifest)} cases, {sum(a.nbytes for a in arrays.values()) / 1e6:.2f} MB raw")


if __name__ == "__main__":
    main()
