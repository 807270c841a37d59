"""Head-sharded multi-GPU launcher helpers (one process per GPU).

(b, h) problems of a MonarchAttention layer are independent (the solver keeps
no cross-head state, solver.py:161-204), so a layer is partitioned by
batch×head with no communication in the operator.  ``all_gather_heads`` is the
optional output all-gather of a sequence-parallel DiT block (NCCL over
NVLink/NVSwitch when the process group uses the nccl backend).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def head_shard(batch: int, heads: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [start, stop) of the flattened (b*H + h) unit list owned
    by ``rank``; sizes differ by at most one."""
    units = batch * heads
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(units, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def local_slice(x: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """The (b, h) units of ``x`` (B, H, N, d) owned by ``rank`` as (1, units, N, d)."""
    B, H = x.shape[:2]
    start, stop = head_shard(B, H, world, rank)
    return x.reshape(B * H, *x.shape[2:])[start:stop].unsqueeze(0)


def all_gather_heads(local_out: torch.Tensor, batch: int, heads: int, group=None) -> torch.Tensor:
    """Reassemble (B, H, N, d) from every rank's (1, units, N, d) output shard."""
    world = dist.get_world_size(group)
    shards = [head_shard(batch, heads, world, r) for r in range(world)]
    width = max(stop - start for start, stop in shards)
    pad = torch.zeros((1, width) + tuple(local_out.shape[2:]), dtype=local_out.dtype, device=local_out.device)
    pad[:, : local_out.shape[1]] = local_out
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    parts = [buf[0, : stop - start] for buf, (start, stop) in zip(bufs, shards)]
    return torch.cat(parts, dim=0).reshape(batch, heads, *local_out.shape[2:])
