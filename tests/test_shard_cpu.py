"""CPU: the multi-rank host logic of the batched configs (sharding, gather,
max-over-ranks timing), run with world_size 2 over gloo on 127.0.0.1."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1402_0264_b200.shard import (balanced_output_ranges, gather_rows, product_work,
                                         range_work, shard_range)


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


def test_balanced_output_ranges_cover_and_balance():
    for na, nb in [(1, 1), (1, 9), (9, 1), (5, 5), (100, 7), (7, 100), (1 << 14, 1 << 14)]:
        nf = na + nb - 1
        for world in (1, 2, 3, 4, 8):
            for align in (1, 4, 1024):
                rs = balanced_output_ranges(na, nb, world, align=align)
                assert len(rs) == world and rs[0][0] == 0 and rs[-1][1] == nf
                assert all(a[1] == b[0] and a[0] <= a[1] for a, b in zip(rs, rs[1:]))
                works = [range_work(na, nb, k0, k1) for k0, k1 in rs]
                assert sum(works) == na * nb
                if na * nb <= 10000:
                    assert works == [sum(product_work(na, nb, k) for k in range(k0, k1))
                                     for k0, k1 in rs]
    rs = balanced_output_ranges(1 << 14, 1 << 14, 8, align=32)  # as bench.py shards cfg1
    works = [range_work(1 << 14, 1 << 14, k0, k1) for k0, k1 in rs]
    assert max(works) / min(works) < 1.02  # cfg1: equal work (to 32 outputs), not equal counts
    assert rs[0][1] - rs[0][0] > 2 * (rs[3][1] - rs[3][0])


def _range_worker(rank, world, port, q):
    """Each rank produces its balanced output slice of a product (here the
    oracle's coefficients stand in for the GPU kernel: host logic only), pads it
    to the longest slice and all-gathers; every rank reassembles the product."""
    import numpy as np
    from oracle import pyoracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, na, nb = 469762049, 700, 300
        rng = np.random.default_rng(5)
        a, b = rng.integers(0, p, na), rng.integers(1, p, nb)
        full = np.asarray(pyoracle.best().mul(a, b, p), dtype=np.int64)
        ranges = balanced_output_ranges(na, nb, world, align=64)
        k0, k1 = ranges[rank]
        L = max(y - x for x, y in ranges)
        local = torch.zeros(L, dtype=torch.int64)
        local[: k1 - k0] = torch.from_numpy(full[k0:k1])
        parts = [torch.empty(L, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, local)
        got = torch.cat([parts[r][: y - x] for r, (x, y) in enumerate(ranges)]).numpy()
        q.put((rank, bool(np.array_equal(got, full))))
    finally:
        dist.destroy_process_group()


def test_output_range_gather_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_range_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, True), (1, True)]


def _ntt_exchange_worker(rank, world, port, q):
    """The sharded NTT's two block exchanges and final reduction over gloo:
    column slices -> row slices -> column slices, against the whole matrix."""
    from paper_1402_0264_b200.shard import NttShards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n1, n2 = 16, 32
        sh = NttShards(n1, n2, world)
        full = torch.arange(n1 * n2, dtype=torch.int64).view(n1, n2)
        w = torch.full((n1 * n2,), -1, dtype=torch.int64)
        c0, cn = sh.cols(rank)
        w.view(n1, n2)[:, c0:c0 + cn] = full[:, c0:c0 + cn]  # "phase 0": my columns
        send = sh.pack_to_rows(w, rank)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send)
        sh.unpack_rows(recv, w, rank)
        r0, rn = sh.rows(rank)
        ok1 = torch.equal(w.view(n1, n2)[r0:r0 + rn], full[r0:r0 + rn])
        w.view(n1, n2)[r0:r0 + rn] *= -3  # "phase 1": my rows
        send = sh.pack_to_cols(w, rank)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send)
        sh.unpack_cols(recv, w, rank)
        ok2 = torch.equal(w.view(n1, n2)[:, c0:c0 + cn], -3 * full[:, c0:c0 + cn])
        out = torch.zeros(n1, n2, dtype=torch.int64)  # "phase 2": disjoint columns
        out[:, c0:c0 + cn] = w.view(n1, n2)[:, c0:c0 + cn]
        dist.all_reduce(out)
        ok3 = torch.equal(out, -3 * full)
        q.put((rank, bool(ok1), bool(ok2), bool(ok3)))
    finally:
        dist.destroy_process_group()


def test_ntt_block_exchange_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ntt_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, True, True, True), (1, True, True, True)]


def test_ntt_shards_validation():
    from paper_1402_0264_b200.shard import NttShards
    with pytest.raises(ValueError):
        NttShards(16, 32, 3)
    sh = NttShards(1024, 2048, 8)
    assert sh.cols(7) == (7 * 256, 256) and sh.rows(7) == (7 * 128, 128)


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
