"""World-size-2 gloo test of the head-sharded launcher logic on CPU: each rank
computes its (b, h) shard (with the CPU oracle standing in for the CUDA
operator, which these CPU tests cannot launch) and the all-gather reassembles
the full layer exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_12271_b200.shard import all_gather_heads, head_shard, local_slice


def test_head_shard_partition():
    for units_b, units_h, world in [(1, 12, 8), (2, 12, 8), (8, 12, 8), (1, 3, 2), (1, 2, 4)]:
        spans = [head_shard(units_b, units_h, world, r) for r in range(world)]
        covered = [u for s, e in spans for u in range(s, e)]
        assert covered == list(range(units_b * units_h))
        sizes = [e - s for s, e in spans]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        head_shard(1, 2, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import monarch_oracle as orc   # CPU stand-in for the CUDA operator

    g = torch.Generator().manual_seed(0)
    B, H, f, h, w, d = 1, 3, 2, 3, 4, 8
    n = f * h * w
    q, k, v = (torch.randn(B, H, n, d, generator=g, dtype=torch.float64) for _ in range(3))
    order = orc.order_neighborhood((f, h, w), (1, h, w))
    ql, kl, vl = (local_slice(x, world, rank) for x in (q, k, v))
    out = torch.stack([torch.from_numpy(orc.forward_phi(ql[0, u].numpy(), kl[0, u].numpy(), vl[0, u].numpy(),
                                                        order, order, f, f, 1, h, w, 2)[2])
                       for u in range(ql.shape[1])]).unsqueeze(0)
    full = all_gather_heads(out, B, H)
    ref = torch.stack([torch.from_numpy(orc.forward_phi(q[0, u].numpy(), k[0, u].numpy(), v[0, u].numpy(),
                                                        order, order, f, f, 1, h, w, 2)[2])
                       for u in range(H)]).unsqueeze(0)
    result[rank] = float((full - ref).abs().max())
    dist.destroy_process_group()


def test_gloo_world2_sharded_layer():
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    result = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, result)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(result.keys()) == [0, 1]
    assert max(result.values()) == 0.0
