"""Host-side sharding of batched workloads across the GPUs of one box.

Batched configs (BASELINE.json configs[3] batch, configs[4]) are independent
instances: each rank takes a contiguous, equal share (the counts divide
evenly for 1/2/4/8 GPUs), computes it with no data-path collective, and the
outputs are gathered to rank 0 with one all-gather over NCCL/NVLink (the only
collective, as the north star allows: "NCCL ... used only to gather or sum
shards").  The large single product (cfg1) shards by output range, balanced
by work; the GCD and division chains do not shard: every rank
runs a replica.
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


def product_work(na: int, nb: int, k: int) -> int:
    """Terms summed into output k of an na x nb product: min(k+1, na, nb, na+nb-1-k)."""
    return max(0, min(k + 1, na, nb, na + nb - 1 - k))


def _prefix_work(na: int, nb: int, k: int) -> int:
    """Work of outputs [0, k), closed form over ramp, plateau and descent."""
    nf = na + nb - 1
    lo, hi = min(na, nb), max(na, nb)
    k = max(0, min(k, nf))
    a = min(k, lo)  # ramp: 1..lo
    w = a * (a + 1) // 2
    if k > lo:  # plateau of height lo
        w += (min(k, hi) - lo) * lo
    if k > hi:  # descending ramp lo-1..1
        c = k - hi
        w += c * lo - c * (c + 1) // 2
    return w


def range_work(na: int, nb: int, k0: int, k1: int) -> int:
    """Terms summed into outputs [k0, k1) (modular MACs of that slice)."""
    return _prefix_work(na, nb, k1) - _prefix_work(na, nb, k0)


def balanced_output_ranges(na: int, nb: int, world: int, align: int = 1):
    """Split the product's outputs [0, na+nb-1) into `world` contiguous ranges
    of (near) equal work -- the triangular/trapezoid profile product_work --
    not equal counts.  Boundaries are rounded to `align`.
    Returns [(k0, k1)] covering the outputs exactly."""
    if world < 1 or na < 1 or nb < 1:
        raise ValueError("balanced_output_ranges: need world, na, nb >= 1")
    nf = na + nb - 1
    total = na * nb

    def prefix(k):
        return _prefix_work(na, nb, k)

    bounds = [0]
    for r in range(1, world):
        target = total * r // world
        a, b = bounds[-1], nf  # smallest k with prefix(k) >= target
        while a < b:
            mid = (a + b) // 2
            if prefix(mid) < target:
                a = mid + 1
            else:
                b = mid
        k = min(nf, max(bounds[-1], (a + align // 2) // align * align))
        bounds.append(k)
    bounds.append(nf)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


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
