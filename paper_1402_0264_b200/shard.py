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


class PeerOutputs:
    """Full-size output regions on every rank in one symmetric-memory
    allocation (torch symmetric memory: each rank's buffer is mapped into every
    peer's address space; stores travel over NVLink/NVSwitch).  A fan-out kernel
    (mmm_cu_*_fanout_dev) given `ptrs(i, off)` stores its rows or range into
    region i of *every* rank's buffer, so the all-gather of a sharded batch
    happens in the producing kernel's epilogue; `barrier()` (device-side, on the
    current stream) orders the ranks before anyone reads.  Raises if symmetric
    memory is unavailable: callers fall back to gather_rows (NCCL)."""

    def __init__(self, sizes, dist):
        import itertools

        import torch
        import torch.distributed._symmetric_memory as symm_mem

        self.sizes = [int(n) for n in sizes]
        self.offs = list(itertools.accumulate([0] + self.sizes[:-1]))
        self.t = symm_mem.empty(sum(self.sizes), dtype=torch.int32, device="cuda")
        self.h = symm_mem.rendezvous(self.t, dist.group.WORLD)
        off = int(getattr(self.h, "offset", 0) or 0)
        self.bases = [int(p) + off for p in self.h.buffer_ptrs]
        if self.bases[dist.get_rank()] != self.t.data_ptr():
            raise RuntimeError("symmetric buffer pointers do not match the local tensor")

    def view(self, i, shape):
        return self.t[self.offs[i]: self.offs[i] + self.sizes[i]].view(shape)

    def ptrs(self, i, off_words=0):
        return [b + 4 * (self.offs[i] + off_words) for b in self.bases]

    def barrier(self):
        self.h.barrier()


# --------------------------------------------------- sharded four-step NTT --
class NttShards:
    """Layout of the four-step NTT product over `world` ranks.

    The N = n1 x n2 workspace w[n2*k1 + col] is a n1 x n2 matrix.  Rank r
    owns the columns [r*n2/W, (r+1)*n2/W) in the column phases (0: forward
    columns of both operands, 2: inverse columns into the output) and the rows
    [r*n1/W, (r+1)*n1/W) in the row phase (1: forward rows, pointwise product,
    inverse rows).  Between them the workspace blocks move with one
    all-to-all each way: block (rows of q) x (cols of r) goes from r to q."""

    def __init__(self, n1: int, n2: int, world: int):
        if world < 1 or n1 % world or n2 % (4 * world):
            raise ValueError(f"sharded NTT: {n1} x {n2} does not split over {world} ranks")
        self.n1, self.n2, self.W = n1, n2, world
        self.R, self.Cw = n1 // world, n2 // world

    def cols(self, r: int):
        return r * self.Cw, self.Cw

    def rows(self, r: int):
        return r * self.R, self.R

    def _blocks(self, work):  # [W (row group), R, W (col group), Cw] view
        return work.view(self.W, self.R, self.W, self.Cw)

    def pack_to_rows(self, work, r: int):
        """After phase 0 on rank r: chunk q = (rows of q) x (cols of r)."""
        return self._blocks(work)[:, :, r, :].contiguous()

    def unpack_rows(self, recv, work, r: int):
        """recv[q] = (rows of r) x (cols of q), from rank q."""
        self._blocks(work)[r] = recv.permute(1, 0, 2)

    def pack_to_cols(self, work, r: int):
        """After phase 1 on rank r: chunk q = (rows of r) x (cols of q)."""
        return self._blocks(work)[r].permute(1, 0, 2).contiguous()

    def unpack_cols(self, recv, work, r: int):
        """recv[q] = (rows of q) x (cols of r), from rank q."""
        self._blocks(work)[:, :, r, :] = recv


def ntt_mul_sharded(mmm, p, d_a, na, d_b, nb, d_f, dist, world: int, rank: int, stream: int):
    """f = a * b (nf = na+nb-1 words in d_f, int32 tensor on this rank's GPU)
    with the NTT split over the ranks: three phase kernels, two all-to-alls of
    workspace blocks and one all-reduce of the disjoint column outputs, all on
    NCCL over NVLink.  d_a, d_b: replicated int32 device tensors."""
    import torch

    # every step -- phase kernels, block packing, collectives -- on the caller's
    # stream, in order (torch ops and NCCL calls follow the current stream)
    ext = torch.cuda.ExternalStream(stream, device=d_a.device) if stream else \
        torch.cuda.current_stream(d_a.device)
    with torch.cuda.stream(ext):
        return _ntt_mul_sharded(mmm, p, d_a, na, d_b, nb, d_f, dist, world, rank, ext.cuda_stream)


def _ntt_mul_sharded(mmm, p, d_a, na, d_b, nb, d_f, dist, world, rank, stream):
    import torch

    nf = na + nb - 1
    n1, n2 = mmm.ntt_shape(p, nf)
    sh = NttShards(n1, n2, world)
    wa = torch.empty(n1 * n2, dtype=torch.int32, device=d_a.device)
    wb = torch.empty_like(wa)
    c0, cn = sh.cols(rank)
    mmm.ntt_phase_dev(p, 0, d_a.data_ptr(), na, d_b.data_ptr(), nb, c0, cn, wa.data_ptr(),
                      wb.data_ptr(), 0, stream)
    if world > 1:
        for w in (wa, wb):
            send = sh.pack_to_rows(w, rank)
            recv = torch.empty_like(send)
            dist.all_to_all_single(recv, send)
            sh.unpack_rows(recv, w, rank)
    r0, rn = sh.rows(rank)
    mmm.ntt_phase_dev(p, 1, d_a.data_ptr(), na, d_b.data_ptr(), nb, r0, rn, wa.data_ptr(),
                      wb.data_ptr(), 0, stream)
    if world > 1:
        send = sh.pack_to_cols(wa, rank)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send)
        sh.unpack_cols(recv, wa, rank)
    d_f.zero_()
    mmm.ntt_phase_dev(p, 2, d_a.data_ptr(), na, d_b.data_ptr(), nb, c0, cn, wa.data_ptr(),
                      wb.data_ptr(), d_f.data_ptr(), stream)
    if world > 1:
        dist.all_reduce(d_f)  # every word was written by exactly one rank (< p < 2^31)
    return d_f


def ntt_mul_virtual(mmm, p, d_a, na, d_b, nb, world: int, stream: int):
    """The sharded product with `world` virtual ranks on one GPU (the
    all-to-alls become local block copies): exercises the phase kernels'
    slices and the block layout exactly as ntt_mul_sharded runs them."""
    import torch

    nf = na + nb - 1
    n1, n2 = mmm.ntt_shape(p, nf)
    sh = NttShards(n1, n2, world)
    wa = [torch.empty(n1 * n2, dtype=torch.int32, device=d_a.device) for _ in range(world)]
    wb = [torch.empty_like(wa[0]) for _ in range(world)]
    for r in range(world):
        c0, cn = sh.cols(r)
        mmm.ntt_phase_dev(p, 0, d_a.data_ptr(), na, d_b.data_ptr(), nb, c0, cn, wa[r].data_ptr(),
                          wb[r].data_ptr(), 0, stream)
    for ws in (wa, wb):
        sends = [sh.pack_to_rows(ws[r], r) for r in range(world)]
        for r in range(world):
            sh.unpack_rows(torch.stack([sends[q][r] for q in range(world)]), ws[r], r)
    for r in range(world):
        r0, rn = sh.rows(r)
        mmm.ntt_phase_dev(p, 1, d_a.data_ptr(), na, d_b.data_ptr(), nb, r0, rn, wa[r].data_ptr(),
                          wb[r].data_ptr(), 0, stream)
    sends = [sh.pack_to_cols(wa[r], r) for r in range(world)]
    for r in range(world):
        sh.unpack_cols(torch.stack([sends[q][r] for q in range(world)]), wa[r], r)
    f = torch.zeros(nf, dtype=torch.int64, device=d_a.device)
    for r in range(world):
        fr = torch.zeros(nf, dtype=torch.int32, device=d_a.device)
        c0, cn = sh.cols(r)
        mmm.ntt_phase_dev(p, 2, d_a.data_ptr(), na, d_b.data_ptr(), nb, c0, cn, wa[r].data_ptr(),
                          wb[r].data_ptr(), fr.data_ptr(), stream)
        f += fr.to(torch.int64)
    return f
