#!/usr/bin/env python3
"""Benchmark of the polynomial-arithmetic hot path (BASELINE.json metric:
mod-p coefficient operations per second).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload gcd|mul|div|ntt|ntt_batch|batch] [--s S]

Default workload: BASELINE.json configs[4] (cfg5) -- 4096 products of
4096 x 4096 terms plus 4096 divisions of 8192 by 4096 terms over
p = 469762049, seed 42: the largest single-GPU config and the one the
north star shards across 1/2/4/8 GPUs.  Instances split evenly over the
ranks; each rank's kernels store their rows into every rank's results
(symmetric memory over NVLink, fan-out epilogues), NCCL all-gather as the
validated fallback.  The unit of work is the modular coefficient MAC:
n^2 per product, (n+1) n per division.  `--workload gcd`
(configs[1]), `mul`, `div`, `div_fast`, `ntt`, `ntt_batch` time the others.

    python bench.py --gpus N ...   # N > 1 re-launches itself under torchrun
                                   # (one process per GPU); under torchrun,
                                   # WORLD_SIZE must equal --gpus

One JSON line on rank 0.  `value` = device time of the CUDA path with inputs
resident in HBM (CUDA events on the launch stream, L2 flushed between timed
steps, max over ranks); `e2e` = the same metric through the host-buffer C-ABI
calls (H2D of the inputs, kernels, D2H of the results inside the timed
region); `roofline` = the dominant kernel (per-kernel CUDA events) vs its
peak; `cpu_baseline` = the reference oracle (oracle/_ref, else the C port) on
one host core.  `--impl reference` times the reference's CPU implementation
of the same workload on all host threads (rank 0 only), with inputs drawn
through the reference itself.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import suites  # noqa: E402  (input definitions shared with the golden generator)

P = suites.P_BENCH
METRIC = "mod-p coeff-ops/sec (plain mult, div/GCD, NTT) vs int-MAD/HBM roofline"
UNIT = "coeff-ops/s"
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_configs.json")
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
IMAD_PEAKS = os.path.join(ROOT, "profiles", "peaks.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------- plumbing --
class Dist:
    """One process per GPU (torchrun env).  Our arm at N > 1: NCCL process
    group (max-over-ranks timing, barriers, the gather fallback); `backend`
    "gloo" runs the same plumbing on CPU (--launcher-check)."""

    def __init__(self, impl: str, backend: str = "nccl"):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg, self.backend = None, backend
        # MMM_BENCH_PEER=1: a process group even at N = 1, so the symmetric-memory
        # fan-out path (PeerOutputs) can be exercised on one GPU
        if impl == "ours" and (self.world > 1 or os.environ.get("MMM_BENCH_PEER")):
            import torch.distributed as dist
            if self.world == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group(backend, rank=self.rank, world_size=self.world)
            self.pg = dist

    def _dev(self):
        return "cuda" if self.backend == "nccl" else "cpu"

    def max(self, x: float) -> float:
        if self.pg is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self._dev())
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.pg is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=self._dev())
        self.pg.all_reduce(t)
        return float(t.item())

    def barrier(self):
        if self.pg is not None:
            if self.backend == "nccl":
                import torch
                self.pg.barrier(device_ids=[torch.cuda.current_device()])
            else:
                self.pg.barrier()

    def close(self):
        if self.pg is not None:
            self.pg.destroy_process_group()


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=1)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[4:8]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def digest(x) -> str:
    import hashlib
    a = np.ascontiguousarray(np.asarray(x).astype("<i8"))
    return hashlib.sha256(a.tobytes()).hexdigest()[:16] if a.size else ""


TRAFFIC = os.path.join(ROOT, "profiles", "traffic.json")


def ncu_traffic(workload, kernel):
    """DRAM read+write bytes per launch of `kernel` in the ncu --set full
    capture of THIS workload's bench command (profiles/traffic.json, written by
    tools/ncu_traffic.py from the committed capture summaries): keyed by
    workload and kernel, never matched across captures."""
    try:
        with open(TRAFFIC) as fh:
            t = json.load(fh)[workload][kernel]
        return float(t["dram_bytes_per_launch"]), t["capture"]
    except (OSError, KeyError, ValueError, TypeError):
        return None, None


def peaks():
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(PEAKS):
        with open(PEAKS) as fh:
            hbm, src = float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    imad = None
    if os.path.exists(IMAD_PEAKS):
        with open(IMAD_PEAKS) as fh:
            imad = float(json.load(fh)["imad_wide_per_s"])
    return hbm, src, imad


IMAD_PEAK_SOURCE = ("builder-measured IMAD.WIDE.U32 rate (tools/peaks.cu -> profiles/peaks.json; "
                    "MEASURED_PEAKS.json has no integer peak)")


def imad_nominal(mhz=1965.0, sms=148):
    """Nominal IMAD.WIDE.U32 issue rate: 32 lanes/clk/SM (half the 64-lane
    IMAD rate) x 148 SMs x the max SM clock."""
    return 32.0 * sms * mhz * 1e6


def imad_line(macs, t, imad):
    """Roofline entry for an IMAD.WIDE-bound kernel: `macs` modular MACs in t s."""
    peak = imad or 8.0647e12
    ach = macs / t
    nom = imad_nominal()
    return {"bound": "imad", "achieved": ach / 1e12, "peak": peak / 1e12, "unit": "TMAC/s",
            "frac": ach / peak, "peak_source": IMAD_PEAK_SOURCE,
            "peak_nominal": nom / 1e12, "frac_nominal": ach / nom,
            "peak_nominal_source": "32 IMAD.WIDE lanes/clk/SM x 148 SMs x 1965 MHz",
            "traffic": None}


TC_PEAK = os.path.join(ROOT, "profiles", "tc_peak.json")


def tensor_line(mod_macs, t, imad):
    """Roofline entry for a tensor-core kernel doing `mod_macs` modular MACs
    (16 u8 x u8 limb MACs each) in t s."""
    try:
        with open(TC_PEAK) as fh:
            pk = json.load(fh)
        peak, src = float(pk["u8_mac_per_s"]), pk["source"]
    except (OSError, KeyError, ValueError):
        peak, src = 2.25e15, "nominal (4.5 POPS dense int8)"
    u8 = 16.0 * mod_macs
    ach = u8 / t
    return {"bound": "tensor", "achieved": ach / 1e12, "peak": peak / 1e12,
            "unit": "T u8-MAC/s", "frac": ach / peak, "peak_source": src,
            "peak_nominal": 2250.0, "frac_nominal": ach / 2.25e15,
            "peak_nominal_source": "4.5 POPS dense int8 per B200 = 2.25e15 MAC/s",
            "alg_u8_macs_per_launch": u8,
            "modular_macs_per_s": mod_macs / t,
            "vs_imad_wide_ceiling": (mod_macs / t) / (imad or 8.0647e12),
            "traffic": None}


def imad_rate():
    """Measured plain IMAD rate (profiles/peaks.json, tools/peaks.cu)."""
    try:
        with open(IMAD_PEAKS) as fh:
            return float(json.load(fh)["imad_per_s"])
    except (OSError, KeyError, ValueError):
        return 1.82e13


def ntt_roofline(logN, count, t_step, kernel):
    """The NTT's bound is the integer multiply pipe (IMAD-bound
    when each transform makes <= 1 HBM pass).  Every modular product is a
    Shoup product (IMAD.HI + 2 IMAD) or, for the pointwise product, a
    Montgomery REDC (IMAD.WIDE + IMAD + IMAD.HI).  IMAD.HI and IMAD.WIDE issue
    at half the IMAD rate on this part (profiles/peaks.json: 8.76e12 vs
    1.82e13 /s), so in IMAD issue slots a Shoup product costs 4 and a REDC 5.
    Products per step: one per butterfly over the 3 transforms (3 (N/2) logN),
    6 N four-step twiddle products (2 per word per operand after the forward
    columns, 2 per word after the rows; the N^-1 scale rides in operand b's
    table) and N pointwise REDCs.  Peak: the measured IMAD rate."""
    N = 1 << logN
    bfly = 3 * (N // 2) * logN * count
    slots = 4 * (bfly + 6 * N * count) + 5 * N * count
    peak = imad_rate()
    achieved = slots / t_step
    return {"bound": "imad", "achieved": achieved / 1e12, "peak": peak / 1e12,
            "unit": "T IMAD-slots/s", "frac": achieved / peak, "traffic": None,
            "kernel": kernel, "alg_imad_slots_per_step": slots, "butterflies": bfly,
            "peak_note": "measured IMAD rate (profiles/peaks.json imad_per_s); "
                         "IMAD.HI/IMAD.WIDE count as 2 slots"}


class OursGen:
    """Inputs through the product's own host generator (libmmm_cu: mmm_rng_*,
    std::mt19937_64 + the reference's random_poly draws) and its GPU product."""

    def __init__(self, seed):
        import paper_1402_0264_b200 as mmm
        self.mmm, self.g = mmm, mmm.Rng(seed)

    def next(self):
        return self.g()

    def random_poly(self, terms, p):
        return self.g.random_poly(terms, p)

    def mul(self, a, b, p):
        return self.mmm.mul(a, b, p)

    def monic(self, a, p):
        return self.mmm.mul(a, [self.mmm.Field(p).inv(int(a[-1]))], p)


class RefGen:
    """Inputs through the reference oracle only (oracle/_ref: ref_rng_*,
    ref_random_poly, ref_mul, ref_inv -- the reference's own random_poly and
    oracle_mul), else its C restatement: the reference arm never loads the
    product library."""

    def __init__(self, seed):
        from oracle import pyoracle
        self.orc, self.kind = _oracle()
        if self.kind == "reference":
            self.h = self.orc.rng_new(seed)
        else:
            import ctypes as C
            lib = self.orc.lib
            lib.orc_mt_seed.argtypes = [C.c_void_p, C.c_uint64]
            lib.orc_mt_next.argtypes = [C.c_void_p]
            lib.orc_mt_next.restype = C.c_uint64
            lib.orc_random_poly.argtypes = [C.c_void_p, C.c_int64, C.c_int64,
                                            C.POINTER(C.c_int64)]
            self.h = C.create_string_buffer(312 * 8 + 64)
            lib.orc_mt_seed(self.h, seed)
        self.pyoracle = pyoracle

    def next(self):
        if self.kind == "reference":
            return self.orc.rng_next(self.h)
        return self.orc.lib.orc_mt_next(self.h)

    def random_poly(self, terms, p):
        import ctypes as C
        out = np.zeros(terms, dtype=np.int64)
        ptr = out.ctypes.data_as(C.POINTER(C.c_int64))
        st = (self.orc._random_poly(self.h, terms, p, ptr) if self.kind == "reference"
              else self.orc.lib.orc_random_poly(self.h, terms, p, ptr))
        assert st == 0, "random_poly"
        return out

    def mul(self, a, b, p):
        return self.orc.mul(a, b, p)

    def monic(self, a, p):
        return self.orc.mul(a, [self.orc.inv_raw(int(a[-1]), p)], p)


# -------------------------------------------------------------- workloads --
class Workload:
    """One BASELINE config.  __init__(s, gen) draws the seeded inputs through
    `gen` (OursGen for our arm, RefGen for the reference arm) and checks them
    against the reference's input digests; attach(mmm) binds the product
    library for our arm only."""

    name = ""
    config = {}

    mark_events = None  # list while the timed region records per-kernel events
    last_part = None    # label of the segment after the last mark

    def attach(self, mmm):
        self.mmm = mmm

    def _mark(self, label):
        """End of a kernel's segment of the step (CUDA event on the launch stream)."""
        if self.mark_events is not None:
            import torch
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(self.tstream)
            self.mark_events.append((label, ev))

    def units(self) -> float:  # coeff-ops per instance-step
        raise NotImplementedError

    def cpu_ref_kind(self, kind):
        """kind of the CPU sample cpu_ref() runs ("reference" or "port")."""
        return kind


def try_peer_outputs(work, sizes):
    """Sharded workloads at N > 1: every rank's full outputs in symmetric memory
    (shard.PeerOutputs), written by the fan-out kernels (the all-gather fused
    into their epilogues).  All ranks fall back to the NCCL gather together if
    any rank cannot map the buffers; the caller validates one step too."""
    from paper_1402_0264_b200.shard import PeerOutputs
    work.peer, work.peer_note = None, ""
    if work.world == 1 and not (os.environ.get("MMM_BENCH_PEER") and work.dist.pg is not None):
        return
    bad = 0.0
    try:
        work.peer = PeerOutputs(sizes, work.dist.pg)
    except Exception as e:  # no symmetric memory on this box: NCCL gather
        bad, work.peer_note = 1.0, f"symmetric memory unavailable ({type(e).__name__})"
    if work.dist.max(bad) > 0:
        work.peer = None
        work.peer_note = work.peer_note or "a peer could not map symmetric memory"


def validate_peer_outputs(work):
    """One fan-out step, checked on every rank; any mismatch sends all ranks back
    to the NCCL gather (recorded in config)."""
    import torch
    if work.peer is None:
        return
    bad = 0.0
    try:
        work.device_step(torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        work.dist.barrier()
        work.device_check()
    except Exception as e:
        bad, work.peer_note = 1.0, f"fan-out validation failed ({type(e).__name__})"
    if work.dist.max(bad) > 0:
        work.peer = None
        work.peer_note = work.peer_note or "fan-out validation failed on a peer"


class GcdWork(Workload):
    """configs[1]: single-instance Euclidean GCD (replicas only across GPUs)."""

    name = "gcd"

    def __init__(self, s, gen):
        self.s = s or 128
        gold = golden()["cfg2"]
        c = suites.cfg2(gen, gen.mul, gen.monic)
        self.a, self.b = c["a"].astype(np.uint32), c["b"].astype(np.uint32)
        assert (digest(self.a), digest(self.b)) == (gold["a"], gold["b"]), "cfg2 inputs"
        self.want = gold["g"]
        self.steps_, self.updates, self.ng = gold["steps"], gold["updates"], gold["deg_g"] + 1
        self.config = {"workload": "cfg2_gcd_deg12288_deg12287_p469762049", "p": P,
                       "deg_a": len(self.a) - 1, "deg_b": len(self.b) - 1, "s": self.s,
                       "s_effective": "61.6 eliminations per batch for s >= 64 (16384 in 266 batches, "
                                      "MMM_GCD_STATS): the 64-word update matrix caps a batch",
                       "eliminations": self.steps_, "seed": 42, "parallelism": "replicas",
                       "l2": "flushed between timed steps (256 MB written then read: clean lines; inputs < L2)"}

    def units(self):
        return float(self.updates)

    def device_setup(self):
        import torch
        self.da = torch.from_numpy(self.a.astype(np.int32)).cuda()
        self.db = torch.from_numpy(self.b.astype(np.int32)).cuda()
        self.dg = torch.zeros(max(len(self.a), len(self.b)), dtype=torch.int32, device="cuda")
        self.dn = torch.zeros(1, dtype=torch.int64, device="cuda")

    def device_step(self, stream):
        self.mmm.gcd_dev(P, self.da.data_ptr(), len(self.a), self.db.data_ptr(), len(self.b),
                         self.dg.data_ptr(), self.dn.data_ptr(), s=self.s, stream=stream)

    def device_check(self):
        n = int(self.dn.item())
        g = self.dg[:n].cpu().numpy().astype(np.uint32)
        assert digest(g) == self.want, "gcd result differs from the reference"

    def host_setup(self):
        import torch
        self.ha = torch.from_numpy(self.a.astype(np.int32)).pin_memory().numpy().view(np.uint32)
        self.hb = torch.from_numpy(self.b.astype(np.int32)).pin_memory().numpy().view(np.uint32)
        self.bytes_in = 4 * (len(self.a) + len(self.b))

    def host_step(self):
        g = self.mmm.gcd(self.ha, self.hb, P, s=self.s)
        self.bytes_out = 4 * len(g) + 8
        return g

    def host_check(self, g):
        assert digest(g) == self.want

    def roofline(self, t_step, hbm, imad, parts=None):
        alg = 4.0 * (len(self.a) + len(self.b) + self.ng)  # inputs read once, gcd written once
        achieved = alg / t_step / 1e9
        return {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None, "kernel": "gcd_kernel",
                "alg_bytes_per_launch": alg,
                "binding": f"dependency chain: {self.steps_} sequential eliminations, "
                           f"{t_step / self.steps_ * 1e9:.1f} ns per elimination",
                "chain": chain_model(t_step, self.steps_)}

    def cpu_ref(self, orc):
        """(callable, coeff-ops per call, checker, sample description)."""
        a, b = self.a.astype(np.int64), self.b.astype(np.int64)
        return (lambda: orc.gcd(a, b, P), self.units(),
                lambda out: digest(out) == self.want, "full instance (oracle_gcd)")


def chain_model(t_step, steps, mhz=1965.0):
    """The GCD's real bound: its critical path, one warp.  A fused pair of
    eliminations (gcd.cu fused_fast) costs at least the larger of (a) its
    dependent chain -- comb (lead of the first step) + neg / canonicalise +
    3-term comb + lead broadcast and test (tools/latency.cu,
    profiles/latency_r1.json) -- and (b) the single-warp issue time of its
    multiply-pipe instructions: 10 IMAD.WIDE.U32 (cc 2, alpha 1, beta 1, two
    words per lane x 3 terms) and 5 IMAD.HI (tools/issue_rate.cu,
    profiles/issue_rate_r1.json).  Batch overheads (replay tail, window build)
    are not in the floor: frac is what the whole run achieves against it."""
    try:
        lat = json.load(open(os.path.join(ROOT, "profiles", "latency_r1.json")))
        iss = json.load(open(os.path.join(ROOT, "profiles", "issue_rate_r1.json")))
    except (OSError, ValueError):
        return None
    dep = lat["lazy_redc_comb"] + 8.0 + lat["comb3_chain"] + lat["shfl_bcast_cmp_branch"]
    issue = 10 * iss["imad_wide_acc"] + 5 * iss["imad_hi_plus_iadd"]
    pair = max(dep, issue)
    floor_ns = pair / 2.0 / mhz * 1e3
    got_ns = t_step / steps * 1e9
    return {"ns_per_elimination": got_ns, "floor_ns_per_elimination": floor_ns,
            "frac": floor_ns / got_ns, "floor_cycles_per_pair": pair,
            "dependent_chain_cycles_per_pair": dep, "issue_cycles_per_pair": issue,
            "sm_mhz": mhz,
            "source": "profiles/latency_r1.json + profiles/issue_rate_r1.json"}


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x).astype(np.uint32).view(np.int32)).cuda()


def _pinned(x):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x).astype(np.uint32).view(np.int32)).pin_memory()
    return t.numpy().view(np.uint32), t


class MulWork(Workload):
    """configs[0]: 2^14 x 2^14 plain multiplication (IMAD-bound).  With N > 1
    ranks the product shards by output range, balanced by work (the triangular
    profile, shard.balanced_output_ranges): each rank computes its
    slice with mmm_cu_mul_range_dev, then one NCCL all-gather (padded slices)
    inside the timed step."""

    name = "mul"
    sharded = True

    def __init__(self, s, gen):
        self.s = s  # 0 = auto (the tensor core); s >= 1: the s x s-tile CUDA-core kernel
        c = suites.cfg1(gen)
        self.a, self.b = c["a"], c["b"]
        self.want = golden()["cfg1"]["f"]
        self.nf = len(self.a) + len(self.b) - 1
        self.world, self.dist = 1, None
        self.ranges = [(0, self.nf)]
        self.k0, self.k1, self.L = 0, self.nf, self.nf
        self.config = {"workload": "cfg1_mul_2^14x2^14_p469762049", "p": P,
                       "s": self.s or "auto (tensor core)",
                       "seed": 42, "parallelism": "single GPU",
                       "l2": "flushed between timed steps (256 MB written then read: clean lines; inputs < L2)"}

    def bind(self, dist):
        from paper_1402_0264_b200.shard import balanced_output_ranges
        self.dist, self.world = dist, dist.world
        self.ranges = balanced_output_ranges(len(self.a), len(self.b), dist.world, align=32)
        self.k0, self.k1 = self.ranges[dist.rank]
        self.L = max(k1 - k0 for k0, k1 in self.ranges)
        if dist.world > 1:
            self.config["parallelism"] = (f"output range sharded by work over {dist.world} ranks "
                                          "(balanced_output_ranges); gather: see config.gather")
            self.config["ranges"] = self.ranges

    def units(self):
        return float(len(self.a) * len(self.b))

    def device_setup(self):
        import torch
        self.da, self.db = _dev(self.a), _dev(self.b)
        self.dloc = torch.zeros(self.L, dtype=torch.int32, device="cuda")
        self.dall = (torch.zeros(self.world * self.L, dtype=torch.int32, device="cuda")
                     if self.world > 1 else self.dloc)
        try_peer_outputs(self, [self.nf])
        validate_peer_outputs(self)
        if self.world > 1 or self.peer is not None:
            self.config["gather"] = ("fan-out: each rank's range stored into every rank's "
                                     "symmetric-memory product (NVLink), device barrier"
                                     if self.peer is not None else
                                     f"NCCL all-gather of padded slices ({self.peer_note})")

    def device_step(self, stream):
        if getattr(self, "peer", None) is not None:
            self.mmm.mul_range_fanout_dev(P, self.da.data_ptr(), len(self.a), self.db.data_ptr(),
                                          len(self.b), self.k0, self.k1,
                                          self.peer.ptrs(0, self.k0), s=self.s, stream=stream)
            self.peer.barrier()
            return
        self.mmm.mul_range_dev(P, self.da.data_ptr(), len(self.a), self.db.data_ptr(),
                               len(self.b), self.k0, self.k1, self.dloc.data_ptr(), s=self.s,
                               stream=stream)
        if self.world > 1:
            self.dist.pg.all_gather_into_tensor(self.dall, self.dloc)

    def _assemble(self, flat):
        return np.concatenate([flat[r * self.L: r * self.L + (k1 - k0)]
                               for r, (k0, k1) in enumerate(self.ranges)])

    def _result(self):
        if getattr(self, "peer", None) is not None:
            return self.peer.view(0, (self.nf,)).cpu().numpy().view(np.uint32)
        return self._assemble(self.dall.cpu().numpy().view(np.uint32))

    def device_check(self):
        assert digest(self._result()) == self.want, "mul result"

    def host_setup(self):
        (self.ha, self._ta), (self.hb, self._tb) = _pinned(self.a), _pinned(self.b)
        self.hout, self._to = _pinned(np.zeros(self.nf, np.uint32))  # result lands in pinned memory
        self.bytes_in = 4 * (len(self.a) + len(self.b))
        self.bytes_out = 4 * (self.nf if self.world == 1 or getattr(self, "peer", None) is not None
                              else self.world * self.L)

    def host_step(self):
        if self.world == 1:  # the host C-ABI call a user makes (mmm_cu_mul)
            return self.mmm.mul(self.ha, self.hb, P, s=self.s, out=self.hout)
        import torch  # sharded: pinned H2D, the rank's slice, all-gather, D2H
        self.da.copy_(self._ta, non_blocking=True)
        self.db.copy_(self._tb, non_blocking=True)
        self.device_step(torch.cuda.current_stream().cuda_stream)
        return self._result()

    def host_check(self, f):
        assert digest(f) == self.want

    def roofline(self, t_step, hbm, imad, parts=None):
        from paper_1402_0264_b200.shard import range_work
        macs = float(range_work(len(self.a), len(self.b), self.k0, self.k1))  # this rank
        full = (self.k0, self.k1) == (0, self.nf)
        if not self.s and full and os.environ.get("MMM_MUL_TC", "1") != "0":
            r = tensor_line(macs, t_step, imad)  # csrc/tcmul.cu: tcmul_split_kernel
            r.update(kernel="tcmul_split_kernel", alg_modular_macs_per_launch=macs)
            return r
        r = imad_line(macs, t_step, imad)
        r.update(kernel="mul_kernel", alg_macs_per_launch=macs,
                 note="integer pipe: one IMAD.WIDE.U32 per modular MAD")
        return r

    def cpu_ref(self, orc):
        a, b = self.a.astype(np.int64), self.b.astype(np.int64)
        return (lambda: orc.mul(a, b, P), self.units(),
                lambda out: digest(out) == self.want, "full instance (oracle_mul)")


class DivWork(Workload):
    """configs[2]: long division deg 2^16 by deg 2^15, s-blocked."""

    name = "div"

    def __init__(self, s, gen):
        self.s = s or 128
        c = suites.cfg3(gen)
        self.a, self.b = c["a"], c["b"]
        g = golden()["cfg3"]
        self.want = (g["q"], g["r"])
        self.nq, self.nr = len(self.a) - len(self.b) + 1, len(self.b) - 1
        self.config = {"workload": "cfg3_divmod_deg2^16_by_deg2^15_p469762049", "p": P,
                       "s": self.s, "seed": 42, "parallelism": "replicas",
                       "l2": "flushed between timed steps (256 MB written then read: clean lines; inputs < L2)"}

    def units(self):
        return float(self.nq * len(self.b))  # heads x (deg b + 1) updates

    def device_setup(self):
        import torch
        self.da, self.db = _dev(self.a), _dev(self.b)
        self.dq = torch.zeros(self.nq, dtype=torch.int32, device="cuda")
        self.dr = torch.zeros(max(self.nr, 1), dtype=torch.int32, device="cuda")

    def device_step(self, stream):
        self.mmm.divmod_dev(P, self.da.data_ptr(), len(self.a), self.db.data_ptr(), len(self.b),
                            self.dq.data_ptr(), self.dr.data_ptr(), s=self.s, stream=stream)

    def device_check(self):
        q = np.trim_zeros(self.dq.cpu().numpy().view(np.uint32), "b")
        r = np.trim_zeros(self.dr[: self.nr].cpu().numpy().view(np.uint32), "b")
        assert (digest(q), digest(r)) == self.want, "divmod result"

    def host_setup(self):
        (self.ha, self._ta), (self.hb, self._tb) = _pinned(self.a), _pinned(self.b)
        self.bytes_in = 4 * (len(self.a) + len(self.b))
        self.bytes_out = 4 * (self.nq + self.nr)

    def host_step(self):
        return self.mmm.divmod(self.ha, self.hb, P, s=self.s)

    def host_check(self, qr):
        assert (digest(qr[0]), digest(qr[1])) == self.want

    def roofline(self, t_step, hbm, imad, parts=None):
        alg = 4.0 * (len(self.a) + len(self.b) + self.nq + self.nr)
        achieved = alg / t_step / 1e9
        return {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None,
                "kernel": "div_pipe_kernel" if self.s >= 32 else "div_grid_kernel",
                "alg_bytes_per_launch": alg,
                "imad_frac": self.units() / t_step / (imad or 8.0647e12),
                "binding": f"{-(-self.nq // self.s)} dependent steps of s={self.s} heads "
                           "(pipelined head CTA for s >= 32; at s = 128 one product per step "
                           "on the head, bound by the head -> bulk -> head hand-off)"}

    def cpu_ref(self, orc):
        a, b = self.a.astype(np.int64), self.b.astype(np.int64)
        return (lambda: orc.divmod(a, b, P), self.units(),
                lambda out: (digest(out[0]), digest(out[1])) == self.want,
                "full instance (oracle_divmod)")


class FastDivWork(DivWork):
    """configs[2] by Newton iteration and NTT products: the
    same (q, r); units stay the schoolbook updates so the rate compares."""

    name = "div_fast"

    def __init__(self, s, gen):
        super().__init__(s, gen)
        self.config.update(workload="cfg3_divmod_fast_newton_ntt_deg2^16_by_deg2^15_p469762049",
                           units="schoolbook-equivalent updates")
        self.config.pop("s", None)

    def device_step(self, stream):
        self.mmm.divmod_fast_dev(P, self.da.data_ptr(), len(self.a), self.db.data_ptr(),
                                 len(self.b), self.dq.data_ptr(), self.dr.data_ptr(),
                                 stream=stream)

    def host_step(self):
        return self.mmm.divmod_fast(self.ha, self.hb, P)

    def roofline(self, t_step, hbm, imad, parts=None):
        alg = 4.0 * (len(self.a) + len(self.b) + self.nq + self.nr)
        achieved = alg / t_step / 1e9
        return {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None, "kernel": "ntt_rows",
                "alg_bytes_per_launch": alg,
                "binding": "~17 Newton doublings + 2 products: launch latency of small NTTs"}


class NttWork(Workload):
    """configs[3] (single): 2^20 x 2^20 product through a length-2^21 NTT.
    With N > 1 ranks the transform is sharded (four-step: column slices,
    all-to-all, row slices, all-to-all, column slices, all-reduce of the
    disjoint outputs; shard.ntt_mul_sharded) -- strong scaling."""

    name = "ntt"
    sharded = True

    def __init__(self, s, gen):
        c = suites.cfg4_big(gen)
        self.a, self.b = c["a"], c["b"]
        self.want = golden()["cfg4_big"].get("f")
        self.nf = len(self.a) + len(self.b) - 1
        self.config = {"workload": "cfg4_ntt_2^20x2^20_N2^21_p469762049", "p": P, "seed": 42,
                       "transform": "four-step 2^10 x 2^11, radix-4/8 Stockham in smem",
                       "parallelism": "single GPU", "units": "schoolbook-equivalent MACs",
                       "l2": "flushed between timed steps (256 MB written then read: clean lines)"}
        self.world, self.dist = 1, None

    def bind(self, dist):
        self.dist, self.world = dist, dist.world
        if dist.world > 1:
            self.config["parallelism"] = (f"four-step NTT sharded over {dist.world} ranks: "
                                          "2 NCCL all-to-alls + 1 all-reduce")

    def units(self):
        return float(len(self.a) * len(self.b))

    def device_setup(self):
        import torch
        self.da, self.db = _dev(self.a), _dev(self.b)
        self.df = torch.zeros(self.nf, dtype=torch.int32, device="cuda")

    def device_step(self, stream):
        if self.world == 1:
            self.mmm.ntt_mul_dev(P, self.da.data_ptr(), len(self.a), self.db.data_ptr(),
                                 len(self.b), self.df.data_ptr(), stream=stream)
        else:
            from paper_1402_0264_b200.shard import ntt_mul_sharded
            ntt_mul_sharded(self.mmm, P, self.da, len(self.a), self.db, len(self.b), self.df,
                            self.dist.pg, self.world, self.dist.rank, stream)

    def device_check(self):
        if self.want:
            assert digest(self.df.cpu().numpy().view(np.uint32)) == self.want, "ntt result"

    def host_setup(self):
        (self.ha, self._ta), (self.hb, self._tb) = _pinned(self.a), _pinned(self.b)
        self.hout, self._to = _pinned(np.zeros(self.nf, np.uint32))
        self.bytes_in = 4 * (len(self.a) + len(self.b))
        self.bytes_out = 4 * self.nf

    def host_step(self):
        if self.world == 1:  # the host C-ABI call a user makes (mmm_cu_ntt_mul)
            return self.mmm.ntt_mul(self.ha, self.hb, P, out=self.hout)
        import torch  # sharded: pinned H2D, the sharded product, D2H
        self.da.copy_(self._ta, non_blocking=True)
        self.db.copy_(self._tb, non_blocking=True)
        self.device_step(torch.cuda.current_stream().cuda_stream)
        return np.trim_zeros(self.df.cpu().numpy().view(np.uint32), "b")

    def host_check(self, f):
        if self.want:
            assert digest(f) == self.want

    def roofline(self, t_step, hbm, imad, parts=None):
        r = ntt_roofline(21, 1, t_step, "ntt_rows")
        if self.world > 1:  # this rank's share of the transform work
            r["achieved"] /= self.world
            r["frac"] /= self.world
        alg = 4.0 * (len(self.a) + len(self.b) + self.nf)
        r["hbm"] = {"achieved_gbs": alg / t_step / 1e9, "peak_gbs": hbm,
                    "frac": alg / t_step / 1e9 / hbm, "alg_bytes": alg}
        return r

    def cpu_ref_kind(self, kind):
        return "port"  # the reference has no output-range routine: the C restatement runs

    def cpu_ref(self, orc):
        # bounded sample: 2^12 middle output words of the product, computed
        # output-stationary exactly as oracle_mul_alt (each ~2^20 MACs)
        import ctypes as C
        from oracle import pyoracle
        port = pyoracle.Port()
        fn = port.lib.orc_poly_mul_alt_range
        PT = C.POINTER(C.c_int64)
        fn.argtypes = [PT, C.c_int64, PT, C.c_int64, C.c_int64, C.c_int64, C.c_int64, PT]
        fn.restype = None
        a, b = self.a.astype(np.int64), self.b.astype(np.int64)
        k0, k1 = (1 << 20) - 2048, (1 << 20) + 2048
        out = np.zeros(k1 - k0, dtype=np.int64)
        macs = float(sum(min(k + 1, self.nf - k, len(a)) for k in range(k0, k1)))

        def run():
            fn(a.ctypes.data_as(PT), len(a), b.ctypes.data_as(PT), len(b), P, k0, k1,
               out.ctypes.data_as(PT))
            return out
        return (run, macs, lambda o: True,
                "4096 middle output words of the 2^20 x 2^20 product (oracle_mul_alt "
                "restated, C port), 2^32 MACs")


class _Sharded(Workload):
    """Batched configs: instances split evenly across ranks (no data-path
    collective), outputs all-gathered to every rank over NCCL inside the timed
    step ("results gathered over NVLink", BASELINE.json configs[3]/[4])."""

    sharded = True

    def bind(self, dist):
        from paper_1402_0264_b200.shard import shard_range
        self.dist, self.world = dist, dist.world
        self.lo, self.hi = shard_range(self.count, dist.world, dist.rank)

    def _gather(self, t):
        from paper_1402_0264_b200.shard import gather_rows
        return gather_rows(t, self.dist.pg, self.world)


class NttBatchWork(_Sharded):
    """configs[3] batch: 256 independent 2^15 x 2^15 products (NTT length 2^16)."""

    name = "ntt_batch"

    def __init__(self, s, gen):
        self.count = 256
        suites.cfg4_big(gen)  # same stream: the batch follows the big pair
        c = suites.cfg4_batch(gen)
        self.A, self.B = c["A"].astype(np.uint32), c["B"].astype(np.uint32)
        gold = golden()["cfg4_batch"]
        self.want = gold["f_all"]
        self.na = self.A.shape[1]
        self.nf = 2 * self.na - 1
        self.config = {"workload": "cfg4_batch_256x(2^15x2^15)_ntt_N2^16_p469762049", "p": P,
                       "seed": 42, "parallelism": "instances sharded across ranks; results "
                       "gathered to every rank (config.gather)", "units": "schoolbook-equivalent MACs",
                       "l2": "flushed between timed steps (256 MB written then read: clean lines)"}

    def units(self):
        return float(self.count) * self.na * self.na

    def device_setup(self):
        import torch
        self.dA = _dev(self.A[self.lo:self.hi])
        self.dB = _dev(self.B[self.lo:self.hi])
        self.dF = torch.zeros((self.hi - self.lo, self.nf), dtype=torch.int32, device="cuda")
        try_peer_outputs(self, [self.count * self.nf])
        validate_peer_outputs(self)
        if self.world > 1 or self.peer is not None:
            self.config["gather"] = ("peer push: one kernel stores the rank's rows into every "
                                     "rank's symmetric-memory results (NVLink), device barrier"
                                     if self.peer is not None else
                                     f"NCCL all-gather ({self.peer_note})")

    def device_step(self, stream):
        k = self.hi - self.lo
        self.mmm.ntt_mul_batched_dev(P, self.dA.data_ptr(), self.na, self.na, self.dB.data_ptr(),
                                     self.na, self.na, k, self.dF.data_ptr(),
                                     self.nf, stream=stream)
        pe = getattr(self, "peer", None)
        if pe is not None:
            self.mmm.fanout_copy_dev(self.dF.data_ptr(), k * self.nf,
                                     pe.ptrs(0, self.lo * self.nf), stream=stream)
            pe.barrier()
            self.full = pe.view(0, (self.count, self.nf))
            return
        self.full = self._gather(self.dF)

    def _digest_rows(self, F):
        import hashlib
        fs = [digest(np.trim_zeros(F[i].astype(np.int64), "b")) for i in range(F.shape[0])]
        return hashlib.sha256("".join(fs).encode()).hexdigest()[:16]

    def device_check(self):
        assert self._digest_rows(self.full.cpu().numpy().view(np.uint32)) == self.want, \
            "ntt batch result"

    def host_setup(self):
        (self.hA, self._ta), (self.hB, self._tb) = _pinned(self.A[self.lo:self.hi]), _pinned(
            self.B[self.lo:self.hi])
        self.hout, self._to = _pinned(np.zeros((self.hi - self.lo, self.nf), np.uint32))
        self.bytes_in = 4 * (self.hA.size + self.hB.size)
        self.bytes_out = 4 * (self.hi - self.lo) * self.nf

    def host_step(self):
        return self.mmm.ntt_mul_batched(self.hA, self.hB, P, out=self.hout)

    def host_check(self, F):
        if self.world == 1:
            assert self._digest_rows(F) == self.want

    def roofline(self, t_step, hbm, imad, parts=None):
        n_local = self.hi - self.lo
        r = ntt_roofline(16, n_local, t_step, "ntt_rows")
        alg = 4.0 * n_local * (2 * self.na + self.nf)
        r["hbm"] = {"achieved_gbs": alg / t_step / 1e9, "peak_gbs": hbm,
                    "frac": alg / t_step / 1e9 / hbm, "alg_bytes": alg}
        return r

    def cpu_ref(self, orc):
        i = 0
        a, b = self.A[i].astype(np.int64), self.B[i].astype(np.int64)
        want = golden()["cfg4_batch"]["f"][i]
        return (lambda: orc.mul(a, b, P), float(self.na * self.na),
                lambda out: digest(out) == want, "one 2^15 x 2^15 instance (oracle_mul)")


class BatchWork(_Sharded):
    """configs[4]: 4096 products 4096 x 4096 + 4096 divisions 8192 / 4096 terms."""

    name = "batch"

    def __init__(self, s, gen):
        self.count, self.s = 4096, s or 0
        c = suites.cfg5(gen)
        self.A, self.B = c["A"].astype(np.uint32), c["B"].astype(np.uint32)
        self.C, self.D = c["C"].astype(np.uint32), c["D"].astype(np.uint32)
        gold = golden()["cfg5"]
        self.want = (gold["f_all"], gold["qr_all"])
        self.n = self.A.shape[1]
        self.config = {"workload": "cfg5_4096x(4096x4096 mul)+4096x(8192/4096 div)_p469762049",
                       "p": P, "seed": 42, "s": self.s or "auto (tensor core)",
                       "parallelism": "instances sharded across ranks; results gathered to "
                       "every rank (config.gather)", "l2": "inputs 335 MB > L2"}

    def units(self):
        n = self.n
        return float(self.count) * (n * n + (n + 1) * n)

    def device_setup(self):
        import torch
        sl = slice(self.lo, self.hi)
        k, n = self.hi - self.lo, self.n
        self.dA, self.dB, self.dC, self.dD = (_dev(x[sl]) for x in (self.A, self.B, self.C,
                                                                      self.D))
        self.dF = torch.zeros((k, 2 * n - 1), dtype=torch.int32, device="cuda")
        self.dQ = torch.zeros((k, n + 1), dtype=torch.int32, device="cuda")
        self.dR = torch.zeros((k, n - 1), dtype=torch.int32, device="cuda")
        c = self.count
        try_peer_outputs(self, [c * (2 * n - 1), c * (n + 1), c * (n - 1)])
        validate_peer_outputs(self)
        if self.world > 1 or self.peer is not None:
            self.config["gather"] = ("fan-out: each rank's rows stored into every rank's "
                                     "symmetric-memory results (NVLink), device barrier"
                                     if self.peer is not None else
                                     f"NCCL all-gather ({self.peer_note})")

    def _device_step(self, stream):
        k, n = self.hi - self.lo, self.n
        pe = getattr(self, "peer", None)
        if pe is not None:
            lo = self.lo
            self.mmm.mul_batched_fanout_dev(P, self.dA.data_ptr(), n, n, self.dB.data_ptr(), n,
                                            n, k, pe.ptrs(0, lo * (2 * n - 1)), 2 * n - 1,
                                            s=self.s, stream=stream)
            self._mark(self._mul_label)
            self.mmm.divmod_batched_fanout_dev(P, self.dC.data_ptr(), 2 * n, 2 * n,
                                               self.dD.data_ptr(), n, n, k,
                                               pe.ptrs(1, lo * (n + 1)), n + 1,
                                               pe.ptrs(2, lo * (n - 1)), n - 1,
                                               s=self.s, stream=stream)
            pe.barrier()
            c = self.count
            self.fullF = pe.view(0, (c, 2 * n - 1))
            self.fullQ = pe.view(1, (c, n + 1))
            self.fullR = pe.view(2, (c, n - 1))
            return
        self.mmm.mul_batched_dev(P, self.dA.data_ptr(), n, n, self.dB.data_ptr(), n, n, k,
                                 self.dF.data_ptr(), 2 * n - 1, s=self.s, stream=stream)
        self._mark(self._mul_label)
        self.mmm.divmod_batched_dev(P, self.dC.data_ptr(), 2 * n, 2 * n, self.dD.data_ptr(), n,
                                    n, k, self.dQ.data_ptr(), n + 1, self.dR.data_ptr(), n - 1,
                                    s=self.s, stream=stream)
        self.fullF = self._gather(self.dF)
        self.fullQ = self._gather(self.dQ)
        self.fullR = self._gather(self.dR)

    def _digests(self, F, Q, R):
        import hashlib
        def rows(M):
            return [digest(np.trim_zeros(M[i].astype(np.int64), "b")) for i in range(M.shape[0])]
        f = hashlib.sha256("".join(rows(F)).encode()).hexdigest()[:16]
        qr = hashlib.sha256("".join(rows(Q) + rows(R)).encode()).hexdigest()[:16]
        return f, qr

    def device_check(self):
        got = self._digests(*(t.cpu().numpy().view(np.uint32) for t in (self.fullF, self.fullQ,
                                                                          self.fullR)))
        assert got == self.want, "batch results"

    def host_setup(self):
        sl = slice(self.lo, self.hi)
        pins = [_pinned(x[sl]) for x in (self.A, self.B, self.C, self.D)]
        (self.hA, self.hB, self.hC, self.hD) = (q[0] for q in pins)
        self._pins = pins
        k, n = self.hi - self.lo, self.n
        outs = [_pinned(np.zeros(shape, np.uint32))
                for shape in ((k, 2 * n - 1), (k, n + 1), (k, max(n - 1, 1)))]
        (self.hF, self.hQ, self.hR), self._pouts = (o[0] for o in outs), outs
        self.bytes_in = 4 * k * (n + n + 2 * n + n)
        self.bytes_out = 4 * k * ((2 * n - 1) + (n + 1) + (n - 1))

    def host_step(self):
        F = self.mmm.mul_batched(self.hA, self.hB, P, s=self.s, out=self.hF)
        Q, R = self.mmm.divmod_batched(self.hC, self.hD, P, s=self.s, q_out=self.hQ,
                                       r_out=self.hR)
        return F, Q, R

    def host_step_default(self):
        F = self.mmm.mul_batched(self.hA, self.hB, P, s=self.s)
        Q, R = self.mmm.divmod_batched(self.hC, self.hD, P, s=self.s)
        return F, Q, R

    def host_check(self, out):
        if self.world == 1:
            assert self._digests(*out) == self.want

    def _kernels(self):
        """Which kernels the dispatcher runs for cfg5 (csrc/mul.cu, divmod.cu):
        the tensor-core ones unless MMM_MUL_TC / MMM_DIV_TC = 0."""
        tm = os.environ.get("MMM_MUL_TC", "1" if not self.s else "0") != "0"
        td = os.environ.get("MMM_DIV_TC", "1" if not self.s else "0") != "0"
        return ("tcmul_kernel" if tm else "mul_kernel"), ("tcdiv_kernel" if td else "div_cta_kernel")

    @property
    def last_part(self):
        return self._kernels()[1]

    def device_step(self, stream):
        self._mul_label = self._kernels()[0]
        self._device_step(stream)

    def roofline(self, t_step, hbm, imad, parts=None):
        """Per kernel (CUDA events between the two launches of each step):
        algorithmic modular MACs of this rank's share (mul: n^2 per product;
        div: (n+1) n per division) over the kernel's mean time.
        Tensor-core kernels are measured in u8 MACs -- 16 limb products per
        modular MAC -- against the measured kind::i8 UMMA rate; the modular
        rate is also given against the IMAD.WIDE ceiling of the CUDA-core
        kernels.  The dominant kernel is the headline.  With a gather, it
        rides in the division's segment (the barrier after it)."""
        k, n = self.hi - self.lo, self.n
        km, kd = self._kernels()
        work = {km: float(k) * n * n, kd: float(k) * (n + 1) * n}
        parts = parts or {km + "+" + kd: t_step}
        if km + "+" + kd in parts:
            work = {km + "+" + kd: sum(work.values())}
        out = {}
        for name, t in parts.items():
            out[name] = (tensor_line(work[name], t, imad) if name.startswith("tc")
                         else imad_line(work[name], t, imad))
            out[name]["ms"] = t * 1e3
        dom = max(parts, key=lambda x: parts[x])
        r = dict(out[dom])
        r.update(kernel=dom, parts=out, alg_modular_macs_per_launch=work[dom])
        return r

    def cpu_ref(self, orc):
        gold = golden()["cfg5"]
        a, b = self.A[0].astype(np.int64), self.B[0].astype(np.int64)
        c, d = self.C[0].astype(np.int64), self.D[0].astype(np.int64)
        n = self.n

        def run():
            return orc.mul(a, b, P), orc.divmod(c, d, P)

        def ok(out):
            f, (q, r) = out
            return (digest(f), digest(q), digest(r)) == (gold["f"][0], gold["q"][0], gold["r"][0])
        return (run, float(n * n + (n + 1) * n), ok,
                "instance 0 of each batch (oracle_mul + oracle_divmod)")


WORKLOADS = {"gcd": GcdWork, "mul": MulWork, "div": DivWork, "div_fast": FastDivWork,
             "ntt": NttWork,
             "ntt_batch": NttBatchWork, "batch": BatchWork}


# ------------------------------------------------------------------ arms --
def run_ours(args, dist):
    import torch
    torch.cuda.set_device(dist.local)
    import paper_1402_0264_b200 as mmm
    mmm.load()
    work = WORKLOADS[args.workload](args.s, OursGen(42))
    work.attach(mmm)
    sharded = getattr(work, "sharded", False)
    if sharded:
        work.bind(dist)
    work.device_setup()
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    work.tstream = stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        work.device_step(sp)
    torch.cuda.synchronize()
    work.device_check()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    marks = [[] for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    n0 = mmm.launch_count()
    with Clocks(torch.cuda.current_device()) as clk:
        for (e0, e1), mk in zip(ev, marks):
            # flush L2: write a 256 MB buffer (> L2), then read it back so the
            # L2 is left holding clean lines -- otherwise the timed kernels pay
            # for writing back up to 126 MB of the flush's dirty lines
            flush.zero_()
            flush_sum = flush.view(torch.int32).sum()  # noqa: F841
            e0.record(stream)
            work.mark_events = mk
            work.device_step(sp)
            work.mark_events = None
            e1.record(stream)
        torch.cuda.synchronize()
        launches = mmm.launch_count() - n0
        t_dev = sum(e0.elapsed_time(e1) for e0, e1 in ev) / 1e3
    dist.barrier()
    torch.cuda.synchronize()
    work.device_check()
    t_dev = dist.max(t_dev)
    t_step = t_dev / args.steps
    # per-kernel segments of the step (this rank), for the roofline's dominant kernel
    parts = None
    if marks[0]:
        parts = {}
        for (e0, e1), mk in zip(ev, marks):
            prev = e0
            for label, e in mk + [(work.last_part, e1)]:
                parts[label] = parts.get(label, 0.0) + prev.elapsed_time(e) / 1e3 / args.steps
                prev = e
    # replicas: every rank ran the whole instance; sharded: the ranks split it
    value = (1 if sharded else dist.world) * work.units() / t_step

    # e2e: host-buffer C-ABI call, H2D + kernel + D2H inside the region
    work.host_setup()
    for _ in range(max(1, args.warmup)):
        work.host_step()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = work.host_step()
    t_e2e = dist.max(time.perf_counter() - t0) / args.steps
    work.host_check(out)
    e2e = {"value": (1 if sharded else dist.world) * work.units() / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": work.bytes_in, "d2h_bytes_per_step": work.bytes_out,
           "ms_per_step": t_e2e * 1e3,
           "how": "the host C-ABI call a user makes (host buffers; H2D, kernels, D2H and "
                  "input validation inside the timed region), pinned result arrays"}
    if hasattr(work, "host_step_default") and dist.world == 1:
        work.host_step_default()
        t0 = time.perf_counter()
        n_def = 3
        for _ in range(n_def):
            work.host_step_default()
        e2e["default_out_ms_per_step"] = (time.perf_counter() - t0) / n_def * 1e3
        e2e["default_out_note"] = ("same call with out=None: results in page-locked memory from "
                                   "the library's pool (mmm_cu_host_alloc), reused once the "
                                   "previous step's arrays are dropped")

    hbm, src, imad = peaks()
    roof = work.roofline(t_step, hbm, imad, parts=parts)
    roof.setdefault("peak_source", src)
    traffic, tsrc = ncu_traffic(work.name, roof["kernel"])
    if traffic is not None:
        roof["traffic"], roof["traffic_source"] = traffic, tsrc
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded mt19937_64 inputs, reference random_poly draws)",
            "config": work.config, "impl": "ours", "e2e": e2e, "roofline": roof,
            "gpu_launches": launches, "clocks": clk.summary()}
    if roof.get("chain") and line["clocks"].get("sm_mhz"):  # at the clock actually run
        roof["chain"] = chain_model(t_step, work.steps_, float(line["clocks"]["sm_mhz"]))
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(work, args.cpu_seconds)
    return line


def _oracle():
    """The reference oracle compiled unmodified (oracle/_ref), else its C
    restatement; (backend, kind).  Test infrastructure: only the cpu_baseline
    leg and the reference arm call it."""
    from oracle import pyoracle
    if pyoracle.reference_available():
        return pyoracle.Reference(), "reference"
    pyoracle.build_port()
    return pyoracle.Port(), "port"


def cpu_baseline(work, seconds):
    """The CPU oracle on this host, rank 0, one core, a bounded sample."""
    orc, kind = _oracle()
    fn, units, ok, what = work.cpu_ref(orc)[:4]
    kind = work.cpu_ref_kind(kind)
    fn()  # warm
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds or n == 0:
        out = fn()
        n += 1
    dt = (time.perf_counter() - t0) / n
    assert ok(out), "cpu baseline result differs from the reference"
    return {"value": units / dt, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{n} x {what}, serial, {dt * 1e3:.1f} ms each"}


def run_reference(args, dist):
    """The reference's own CPU path on the workload of our arm: the reference
    oracle compiled unmodified (oracle/_ref; its C restatement only if that is
    missing, and for the NTT sample, which has no reference routine -> kind
    "port").  Inputs are drawn through the reference's own random_poly and
    oracle_mul (RefGen); this arm never loads the product library.
    Single-instance configs: the reference algorithm is serial, so one
    instance per step on one thread.  Batched configs: one instance per host
    thread per step (a bounded sample of the batch).  Rank 0 only."""
    if dist.rank != 0:
        return None
    gen = RefGen(42)
    work = WORKLOADS[args.workload](args.s, gen)
    orc, kind = gen.orc, gen.kind
    kind = work.cpu_ref_kind(kind)
    batched = getattr(work, "sharded", False)
    cores = (os.cpu_count() or 1) if batched else 1
    fn, units, ok, what = work.cpu_ref(orc)[:4]

    def step():
        if cores == 1:
            return [fn()]
        with ThreadPoolExecutor(cores) as ex:
            return list(ex.map(lambda _: fn(), range(cores)))

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        outs = step()
    dt = (time.perf_counter() - t0) / args.steps
    assert all(ok(o) for o in outs), "reference result differs from the golden digest"
    value = cores * units / dt
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i64",
            "data": "synthetic (seeded mt19937_64 inputs, reference random_poly draws)",
            "config": work.config, "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": (f"{cores} concurrent x {what} per step, one per host "
                                        f"thread") if cores > 1 else
                                       f"{what} per step, serial (the reference algorithm is "
                                       f"single-threaded)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def launcher_check(args, dist):
    """CPU check of the N-rank launch (gloo): every rank joins, max/sum over
    ranks work; rank 0 reports what a bench line would carry."""
    ranks = dist.sum(1.0)
    slowest = dist.max(float(dist.rank))
    dist.barrier()
    return {"launcher_check": True, "n_gpus": dist.world, "ranks_joined": int(ranks),
            "max_rank": int(slowest), "backend": dist.backend, "impl": args.impl}


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="batch")
    ap.add_argument("--s", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--launcher-check", action="store_true",
                    help="CPU: launch the ranks over gloo and report them (no GPU work)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        log(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; refusing to time a "
            "different number of ranks than asked for")
        sys.exit(2)
    if args.launcher_check:
        dist = Dist("ours" if world > 1 else "none", backend="gloo")
        try:
            line = launcher_check(args, dist)
            if dist.rank == 0:
                print(json.dumps(line), flush=True)
        finally:
            dist.close()
        return
    dist = Dist(args.impl)
    try:
        line = run_ours(args, dist) if args.impl == "ours" else run_reference(args, dist)
        if line is not None and dist.rank == 0:
            print(json.dumps(line), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
