"""The C-ABI library loads, exports every symbol include/monarch_b200.h
declares, and validates descriptors with the reference's error conditions —
all host-side, no kernel launches (runs without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2602_12271_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_12271_b200 import build

    build.build()
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    header = open(os.path.join(ROOT, "include", "monarch_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(mbx_\w+)\s*\(", header, re.M))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name)
    assert lib.mbx_version() == _lib.ABI_VERSION


def _desc(**kw):
    d = _lib.MbxDesc()
    d.abi_version = _lib.ABI_VERSION
    d.dtype = _lib.BF16
    d.batch, d.heads, d.head_dim, d.v_dim = 1, 12, 128, 128
    d.c1_q, d.c1_kv, d.c2, d.s1, d.s2 = 3, 3, 1, 30, 52
    d.iterations, d.flags, d.scale = 1, 0, 128 ** -0.5
    d.eps_div, d.eps_log = 1e-30, 1e-300
    n = 4680
    for name in ("q_stride", "k_stride", "v_stride", "o_stride"):
        getattr(d, name)[:] = (12 * n * 128, n * 128, 128)
    for key, val in kw.items():
        setattr(d, key, val)
    return d


def test_validate_ok_and_workspace(lib):
    d = _desc()
    assert lib.mbx_validate(ctypes.byref(d)) == _lib.OK
    assert lib.mbx_workspace_bytes(ctypes.byref(d)) > 0
    assert lib.mbx_selected_path(ctypes.byref(d)) in (0, 1)
    d.flags = _lib.FLAG_FORCE_GENERIC
    assert lib.mbx_selected_path(ctypes.byref(d)) == 0


@pytest.mark.parametrize("field,value,status", [
    ("iterations", 0, _lib.BAD_ITERS),
    ("eps_div", 0.0, _lib.BAD_EPS),
    ("eps_div", 1e-3, _lib.BAD_EPS),
    ("eps_log", 2e-6, _lib.BAD_EPS),
    ("dtype", 7, _lib.BAD_DTYPE),
    ("s1", 0, _lib.BAD_PLAN),
    ("c1_q", 4, _lib.BAD_PLAN),
    ("head_dim", 512, _lib.UNSUPPORTED),
    ("abi_version", 99, _lib.BAD_SHAPE),
])
def test_validate_rejects(lib, field, value, status):
    d = _desc(**{field: value})
    assert lib.mbx_validate(ctypes.byref(d)) == status
    assert lib.mbx_last_error().decode()
    assert lib.mbx_workspace_bytes(ctypes.byref(d)) == 0


def test_forward_rejects_null_and_small_workspace(lib):
    d = _desc()
    st = lib.mbx_forward(ctypes.byref(d), None, None, None, None, None, None, None, 0, None)
    assert st == _lib.NULL
    fake = ctypes.c_void_p(16)   # never dereferenced: validation fails first
    st = lib.mbx_forward(ctypes.byref(d), fake, fake, fake, fake, None, None, fake, 1, None)
    assert st == _lib.WORKSPACE


def test_closed_form_addressing_matches_orders(lib, goldens):
    """mbx_token_index (the tensor-core path's row addressing) reproduces the
    plan permutation for every neighborhood / identity golden case."""
    import numpy as np

    from cases import package_lowering

    manifest, _ = goldens
    checked = 0
    for meta in manifest:
        low = package_lowering(meta)
        if low.nbhd is None and (low.q_order is not None or low.kv_order is not None):
            continue
        d = _desc(c1_q=low.c1_q, c1_kv=low.c1_kv, c2=low.c2, s1=low.s1, s2=low.s2, head_dim=8, v_dim=8)
        if low.nbhd is not None:
            d.grid[:] = low.grid
            d.nbhd[:] = low.nbhd
        assert lib.mbx_validate(ctypes.byref(d)) == _lib.OK, lib.mbx_last_error()
        for is_q, order, n in ((1, low.q_order, low.n_q), (0, low.kv_order, low.n_kv)):
            ref = np.arange(n) if order is None else order
            got = np.array([lib.mbx_token_index(ctypes.byref(d), is_q, p) for p in range(n)])
            assert np.array_equal(got, ref), meta["name"]
        checked += 1
    assert checked >= 10


def test_closed_form_rejects_inconsistent_neighborhood(lib):
    d = _desc()
    d.grid[:] = (3, 30, 52)
    d.nbhd[:] = (1, 30, 26)          # would need c2 = 2, s2 = 26
    assert lib.mbx_validate(ctypes.byref(d)) == _lib.BAD_PLAN
