"""Lower golden-case metadata to kernel coordinates — twice, independently:
with the oracle's own ordering restatement (the checker) and with the
package's layout mirror (the product).  Tests assert both agree."""

from __future__ import annotations

import numpy as np

from oracle import monarch_oracle as orc


def oracle_lowering(meta):
    """(order_q, order_k, c1q, c1k, c2, s1, s2) via oracle/monarch_oracle.py."""
    f, h, w = meta["shape"]
    n = f * h * w
    cfg = meta["config"]
    nb = meta.get("nbhd")
    if nb is not None:
        order = orc.order_neighborhood((f, h, w), nb)
        b1, b2 = f * h, w
        c1 = (f // nb[0]) * (h // nb[1])
        c2 = w // nb[2]
    elif cfg[0] == "raw":
        b1, b2 = cfg[1], cfg[2]
        order = orc.order_phi((f, h, w))
        c1, c2 = meta.get("c", [1, 1])
    else:
        g1 = "".join(cfg) if cfg != ["fh"] else "fh"
        order = orc.order_aligned((f, h, w), tuple(g1))
        sizes = {"f": f, "h": h, "w": w}
        b1 = int(np.prod([sizes[a] for a in g1])) if g1 else 1
        b2 = n // b1
        c1, c2 = meta.get("c", [1, 1])
    s1, s2 = b1 // c1, b2 // c2
    if meta["kind"] == "chunk":
        fq = meta["f_q"]
        c1q = (fq // nb[0]) * (h // nb[1])
        q_order = order[(c1 - c1q) * s1 * b2:] - (f - fq) * h * w
        return q_order, order, c1q, c1, c2, s1, s2
    return order, order, c1, c1, c2, s1, s2


def package_plan(meta):
    """Build the package's BlockConfig / TilePlan for a golden case."""
    import paper_2602_12271_b200 as pk

    shape = pk.VideoShape(*meta["shape"])
    cfg = meta["config"]
    if meta.get("nbhd") is not None:
        return pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), tuple(meta["nbhd"]))
    if cfg[0] == "raw":
        base = pk.config_from_sizes(shape, cfg[1], cfg[2])
    else:
        base = pk.aligned_config(shape, tuple(cfg) if cfg != ["fh"] else ("f", "h"))
    if meta["kind"] == "solve":
        return base
    return pk.TilePlan(base, *meta["c"])


def package_lowering(meta):
    import paper_2602_12271_b200 as pk

    plan = package_plan(meta)
    if meta["kind"] == "chunk":
        return pk.lower_chunked(plan, meta["f_q"])
    return pk.lower_square(plan)


def c1_inputs(meta):
    """Regenerate the seeded C1 inputs (make_goldens.py section G)."""
    rng = np.random.default_rng(meta["seed"])
    for _ in range(meta["head"] + 1):
        q = rng.standard_normal((1024, 64)).astype(np.float32)
        k = rng.standard_normal((1024, 64)).astype(np.float32)
        v = rng.standard_normal((1024, 64)).astype(np.float32)
    return q, k, v


def case_inputs(meta, data):
    name = meta["name"]
    if "input_sums" in meta:
        q, k, v = c1_inputs(meta)
        sums = [float(np.sum(x)) for x in (q, k, v)]
        assert np.allclose(sums, meta["input_sums"], rtol=0, atol=1e-3), "seeded inputs drifted"
        return q, k, v
    return data[f"{name}/q"], data[f"{name}/k"], data[f"{name}/v"]
