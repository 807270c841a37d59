"""The torch.library custom op (``torch.ops.monarch_b200.monarch_attention``): schema,
fake-tensor kernel and autograd registration (torch.library.opcheck), and a
torch.compile(fullgraph=True) graph around the public ``monarch_attention`` that
gives the eager bytes -- the operator is not opaque to tracing (SURVEY.md §8b:
"torch custom op wrapper")."""

import pytest
import torch

import paper_2602_12271_b200 as pk
from paper_2602_12271_b200 import ops

pytestmark = pytest.mark.gpu


def _case(dev, dtype, d, frames=2, h=4, w=8, heads=2, seed=0):
    s = pk.VideoShape(frames, h, w)
    plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, h, w))
    g = torch.Generator(device="cpu").manual_seed(seed)
    q, k, v = (torch.randn(1, heads, s.n, d, generator=g).to(dev, dtype) for _ in range(3))
    return plan, q, k, v


@pytest.mark.parametrize("dtype,d", [(torch.float32, 32), (torch.bfloat16, 128)])
def test_opcheck(cuda, dtype, d):
    plan, q, k, v = _case(cuda, dtype, d)
    key = ops.plan_key(ops.lower_for(plan, q.shape[2], k.shape[2], None))
    q, k, v = (x.requires_grad_(True) for x in (q, k, v))
    torch.library.opcheck(torch.ops.monarch_b200.monarch_attention.default, (q, k, v, key, 1, d ** -0.5),
                          test_utils=("test_schema", "test_autograd_registration", "test_faketensor"))


def test_compile_fullgraph_matches_eager(cuda):
    s = pk.VideoShape(3, 30, 52)
    plan = pk.make_tile_plan(s, pk.aligned_config(s, ("f", "h")), (1, 30, 52))
    g = torch.Generator(device="cpu").manual_seed(5)
    q, k, v = (torch.randn(1, 2, s.n, 128, generator=g).to(cuda, torch.bfloat16) for _ in range(3))

    def block(q, k, v):
        o = pk.monarch_attention(q, k, v, plan)
        return o * 2.0 + 1.0

    eager = block(q, k, v)
    compiled = torch.compile(block, fullgraph=True)(q, k, v)
    torch.cuda.synchronize()
    assert torch.equal(compiled, eager)
