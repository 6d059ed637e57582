"""Host-side sharding of batched workloads across the GPUs of one box.

Batched configs (BASELINE.json configs[3] batch, configs[4]) are independent
instances: each rank takes a contiguous, equal share (the counts divide
evenly for 1/2/4/8 GPUs), computes it with no data-path collective, and the
outputs are gathered to rank 0 with one all-gather over NCCL/NVLink (the only
collective, as the north star allows: "NCCL ... used only to gather or sum
shards").  Single-instance configs do not shard: every rank runs a replica.
"""
from __future__ import annotations

from typing import Tuple


def shard_range(count: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [start, stop) share of `count` instances for `rank`.

    Shares differ by at most one instance; with count % world == 0 they are
    equal, which the all-gather below requires."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(count, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_rows(local, dist, world: int):
    """All-gather equal row blocks (torch tensors on the device) into one
    [world * rows, ...] tensor on every rank (NCCL: over NVLink)."""
    import torch

    if world == 1 or dist is None:
        return local
    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous())
    return out
