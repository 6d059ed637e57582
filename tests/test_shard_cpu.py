"""CPU: the multi-rank host logic of the batched configs (sharding, gather,
max-over-ranks timing), run with world_size 2 over gloo on 127.0.0.1."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1402_0264_b200.shard import gather_rows, shard_range


def test_shard_range_partitions():
    for count in (1, 7, 256, 4096):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(count, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        count, width = 8, 5
        start, stop = shard_range(count, world, rank)
        # each rank "computes" its instances: row i = i * 10 + column
        local = torch.stack([torch.arange(width) + 10 * i for i in range(start, stop)])
        full = torch.empty((count, width), dtype=local.dtype)
        dist.all_gather_into_tensor(full, local) if hasattr(dist, "all_gather_into_tensor") \
            and dist.get_backend() == "nccl" else dist.all_gather(list(full.chunk(world)), local)
        ok = torch.equal(full, torch.stack([torch.arange(width) + 10 * i for i in range(count)]))
        # max over ranks of a per-rank time, as bench.py reports it
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, bool(ok), float(t.item())))
    finally:
        dist.destroy_process_group()


def test_gather_and_max_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [True, True]
    assert [r[2] for r in res] == [2.0, 2.0]


def test_gather_rows_single_rank_is_identity():
    x = torch.arange(6).reshape(3, 2)
    assert gather_rows(x, None, 1) is x
