"""The backward pass's oracle (oracle/monarch_torch.py) on CPU: its forward is the
pinned numpy oracle's, and its gradients pass finite-difference gradcheck."""

import numpy as np
import pytest
import torch

from cases import case_inputs, oracle_lowering
from oracle import monarch_oracle as orc
from oracle import monarch_torch as ort


def test_torch_forward_matches_numpy_oracle_on_goldens(goldens):
    manifest, data = goldens
    checked = 0
    for meta in manifest:
        if meta["T"] > 3 or meta.get("kind") == "chunk":
            continue
        q, k, v = case_inputs(meta, data)
        oq, ok, c1q, c1k, c2, s1, s2 = oracle_lowering(meta)
        out_t = ort.forward_phi_torch(torch.as_tensor(q, dtype=torch.float64), torch.as_tensor(k, dtype=torch.float64),
                                      torch.as_tensor(v, dtype=torch.float64), oq, ok, c1q, c1k, c2, s1, s2, meta["T"])
        _, _, ref = orc.forward_phi(q, k, v, oq, ok, c1q, c1k, c2, s1, s2, meta["T"])
        assert np.abs(out_t.numpy() - ref).max() < 1e-12, meta["name"]
        checked += 1
    assert checked >= 10


@pytest.mark.parametrize("T", [1, 2, 3])
def test_gradcheck_small_tiled(T):
    torch.manual_seed(T)
    f, h, w, d = 2, 2, 3, 4
    order = orc.order_neighborhood((f, h, w), (1, 2, 3))
    n = f * h * w
    q, k, v = (torch.randn(n, d, dtype=torch.float64, requires_grad=True) for _ in range(3))

    def fn(q, k, v):
        return ort.forward_phi_torch(q, k, v, order, order, f, f, 1, h, w, T)

    assert torch.autograd.gradcheck(fn, (q, k, v), eps=1e-6, atol=1e-6)


def test_gradcheck_chunked_kv():
    """Rectangular (chunked-KV) grid: 1 query frame against 3 key frames."""
    torch.manual_seed(7)
    f, fq, h, w, d = 3, 1, 2, 3, 4
    order = orc.order_neighborhood((f, h, w), (1, 2, 3))
    q_order = order[(f - fq) * h * w:] - (f - fq) * h * w
    q = torch.randn(fq * h * w, d, dtype=torch.float64, requires_grad=True)
    k, v = (torch.randn(f * h * w, d, dtype=torch.float64, requires_grad=True) for _ in range(2))

    def fn(q, k, v):
        return ort.forward_phi_torch(q, k, v, q_order, order, fq, f, 1, h, w, 2)

    assert torch.autograd.gradcheck(fn, (q, k, v), eps=1e-6, atol=1e-6)
