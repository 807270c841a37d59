"""Host-side layout mirror: orderings, plans, lowering (layout.py:25-351)."""

import os
import sys

import numpy as np
import pytest

import paper_2602_12271_b200 as pk
from cases import oracle_lowering, package_lowering
from oracle import monarch_oracle as orc

REF = "/root/reference/pkg/src"


def test_lowering_agrees_with_oracle_on_every_golden_case(goldens):
    manifest, _ = goldens
    for meta in manifest:
        oq, ok, c1q, c1k, c2, s1, s2 = oracle_lowering(meta)
        low = package_lowering(meta)
        assert (low.c1_q, low.c1_kv, low.c2, low.s1, low.s2) == (c1q, c1k, c2, s1, s2), meta["name"]
        pq = np.arange(low.n_q) if low.q_order is None else low.q_order
        pkv = np.arange(low.n_kv) if low.kv_order is None else low.kv_order
        assert np.array_equal(pq, oq), meta["name"]
        assert np.array_equal(pkv, ok), meta["name"]


@pytest.mark.parametrize("shape", [(2, 3, 4), (4, 6, 10), (1, 5, 7), (3, 1, 2)])
def test_aligned_orderings_are_reshape_transposes(shape):
    s = pk.VideoShape(*shape)
    for cfg in pk.enumerate_aligned_configs(s) + [pk.aligned_config(s, ("f", "h"))]:
        assert np.array_equal(cfg.ordering().to_phi(), orc.order_aligned(shape, cfg.g1))


def test_neighborhood_ordering_and_identity_cases():
    s = pk.VideoShape(3, 30, 52)
    plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, 30, 52))
    assert (plan.c1, plan.c2, plan.tile_b1, plan.tile_b2) == (3, 1, 30, 52)
    assert pk.lower_square(plan).q_order is None         # (h,w) tiles: identity
    plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (3, 30, 52))
    assert (plan.c1, plan.c2) == (1, 1) and pk.lower_square(plan).q_order is None
    s = pk.VideoShape(4, 6, 10)
    plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (2, 3, 5))
    assert np.array_equal(plan.ordering().to_phi(), orc.order_neighborhood((4, 6, 10), (2, 3, 5)))


def test_positions_by_phi_is_inverse():
    s = pk.VideoShape(2, 3, 4)
    o = pk.rho_ordering(s)
    p = o.to_phi()
    assert np.array_equal(o.positions_by_phi()[p], np.arange(s.n))
    for pos in [(0, 0, 0), (1, 2, 3), (1, 0, 2)]:
        assert p[pk.flatten_index(o, pos)] == (pos[0] * 3 + pos[1]) * 4 + pos[2]


def test_layout_errors():
    s = pk.VideoShape(2, 3, 4)
    with pytest.raises(pk.LayoutError):
        pk.VideoShape(0, 1, 1)
    with pytest.raises(pk.LayoutError):
        pk.BlockConfig(s, 5, 5)
    with pytest.raises(pk.LayoutError):
        pk.TilePlan(pk.aligned_config(s, ("f", "h")), 4, 1)
    with pytest.raises(pk.LayoutError):
        pk.make_tile_plan(s, pk.aligned_config(s, ("w",)), (1, 1, 1))
    with pytest.raises(pk.LayoutError):
        pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, 2, 4))
    plan = pk.make_tile_plan(pk.VideoShape(6, 4, 4), pk.aligned_config(pk.VideoShape(6, 4, 4), ("f", "h")),
                             (2, 2, 2))
    with pytest.raises(pk.LayoutError):
        pk.lower_chunked(plan, 3)                         # n_f = 2 does not divide 3
    low = pk.lower_chunked(plan, 2)
    assert (low.c1_q, low.c1_kv, low.n_q, low.n_kv) == (2, 6, 32, 96)


def test_config_from_sizes_detects_alignment():
    s = pk.VideoShape(2, 3, 4)
    assert pk.config_from_sizes(s, 6, 4).g1 == ("f", "h")
    assert pk.config_from_sizes(s, 2, 12).g1 == ("f",)
    assert not pk.config_from_sizes(s, 8, 3).aligned


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present (GPU box)")
def test_matches_reference_layout_module():
    sys.path.insert(0, REF)
    import monarchbench as mb

    for shape in [(2, 3, 4), (4, 6, 10), (3, 30, 52)]:
        s_ref, s_pk = mb.VideoShape(*shape), pk.VideoShape(*shape)
        for g1 in [("f", "h"), ("w",), ("f",), ("h", "w"), ("f", "w"), ("h",)]:
            a = mb.aligned_config(s_ref, g1).ordering().to_phi()
            b = pk.aligned_config(s_pk, g1).ordering().to_phi()
            assert np.array_equal(a, b)
        assert [c.descriptor() for c in mb.enumerate_aligned_configs(s_ref)] == \
               [c.descriptor() for c in pk.enumerate_aligned_configs(s_pk)]
        for nb in [(1, shape[1], shape[2]), (shape[0], 1, 1), (1, 1, 1)]:
            pr = mb.make_tile_plan(s_ref, mb.aligned_config(s_ref, ("f", "h")), nb)
            pp = pk.make_tile_plan(s_pk, pk.aligned_config(s_pk, ("f", "h")), nb)
            assert np.array_equal(pr.ordering().to_phi(), pp.ordering().to_phi())
            assert pr.descriptor() == pp.descriptor()
        assert np.array_equal(mb.rho_ordering(s_ref).to_phi(), pk.rho_ordering(s_pk).to_phi())
