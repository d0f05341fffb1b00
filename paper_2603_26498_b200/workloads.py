"""Sweep grids of BASELINE.json's configs and the replica-sharding layer.

A replica = one engine (trace x load x policy parameters).  Replicas never interact
("many engines may run concurrently on independent inputs"), so a sweep
shards across GPUs with no data-path collective: global replica g = seed*n_cells + cell goes to
rank seed mod G
(seed rows dealt cyclically so every rank holds every cell); only the int64 a6 histograms
and counters are all-reduced (NCCL), which is bit-exact for any G.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import tcm

try:  # the generator is the shared seeded-input module (repo root)
    import tracegen as T
except ImportError:  # pragma: no cover - repo root not on sys.path
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import tracegen as T


@dataclass
class Sweep:
    name: str
    gen: np.ndarray          # tracegen.TG_REPLICA_DTYPE [R]
    params: np.ndarray       # tcm.PARAMS_DTYPE [R]
    n_cells: int
    cells: list              # human-readable description of each cell
    ids: np.ndarray = None   # global replica id of each replica, in load order

    @property
    def n_replicas(self) -> int:
        return len(self.gen)

    @property
    def n_requests(self) -> int:
        return int(self.gen["n_requests"].sum())


def rank_ids(n_cells: int, seeds_total: int, rank: int, world: int) -> list:
    """Global replica ids g = seed * n_cells + cell owned by `rank`: seed rows are dealt
    cyclically (seed % world == rank), so every rank holds every cell in equal measure (load
    balance: cells differ ~100x in cost); ids are ordered cell-major so a warp's 32 replicas
    share one cell's parameters (SIMT coherence)."""
    return [s * n_cells + c for c in range(n_cells) for s in range(rank, seeds_total, world)]


def _grid(name, cells, replicas_per_cell, n_requests, seed, replica_ids):
    """cells: list of dicts(rate, mix, kv, policy, alpha, budget). Global replica g belongs to
    cell g % n_cells and seed row g // n_cells."""
    nc = len(cells)
    R = len(replica_ids)
    gen = np.zeros(R, dtype=T.TG_REPLICA_DTYPE)
    params = tcm.make_params(R)
    for j, g in enumerate(replica_ids):
        c = cells[g % nc]
        gen[j] = T.make_replica(seed, int(g), n_requests, c["rate"], c["mix"], c.get("gen_kv", c["kv"]))
        params[j]["policy"] = c["policy"]
        params[j]["kv_capacity"] = c["kv"]
        params[j]["aging_alpha"] = c["alpha"]
        params[j]["chunk_budget"] = c["budget"]
        params[j]["cell_id"] = g % nc
        params[j]["flags"] = c.get("flags", 0)
    return Sweep(name, gen, params, nc, cells, np.asarray(replica_ids, dtype=np.int64))


ALPHAS = [0.0] + [2.0 ** e for e in range(-7, 8)]          # R14: {0} U {2^-7 .. 2^7}


def c1(policy=tcm.POLICY_TCM, seed=1):
    """1 replica x 1,000 requests, 70/25/5, 2 req/s, KV 131072, B 2048."""
    cells = [dict(rate=2.0, mix=(0.70, 0.25, 0.05), kv=131072, policy=policy, alpha=1.0, budget=2048)]
    return _grid("C1", cells, 1, 1000, seed, [0])


def c3(rank=0, world=1, replicas=4096, n_requests=10_000, seed=2026):
    """4,096 replicas x 10k: lambda in {0.25..4.0} (16) x alpha (16) x 16 seeds, 70/25/5, TCM."""
    cells = [dict(rate=0.25 * (i + 1), mix=(0.70, 0.25, 0.05), kv=131072, policy=tcm.POLICY_TCM,
                  alpha=a, budget=2048) for i in range(16) for a in ALPHAS]
    nc = len(cells)
    return _grid("C3", cells, replicas // nc, n_requests, seed, rank_ids(nc, replicas // nc, rank, world))


def c4_cells():
    return [dict(rate=lam, mix=(0.50, 0.20, 0.30), kv=kv, policy=pol, alpha=1.0, budget=2048)
            for pol in (tcm.POLICY_FCFS, tcm.POLICY_TCM) for lam in (0.5, 1.0, 2.0, 4.0)
            for kv in (131072, 65536, 32768, 16384)]


def c4(rank=0, world=1, replicas_per_gpu=65536, n_requests=10_000, seed=4044):
    """Memory-pressure sweep (video-heavy 50/20/30, tight KV): KV {128k,64k,32k,16k} x lambda
    {0.5,1,2,4} x {FCFS,TCM} x seeds.  Weak scaling: every rank simulates replicas_per_gpu
    replicas; global replica ids rank, rank+G, ... (cyclic over the 32 cells)."""
    cells = c4_cells()
    seeds_total = replicas_per_gpu * world // len(cells)
    ids = rank_ids(len(cells), seeds_total, rank, world)
    # warp layout: 16 lanes of an FCFS cell next to 16 lanes of the TCM cell with the same (lambda, KV)
    # (cells c and c + 16): the FCFS half finishes early and leaves each warp 16 TCM replicas instead of
    # 32, 2 % faster on the fused engine than cell-major; needs 16 | replicas per cell
    per = len(ids) // len(cells)
    if per % 16 == 0 and per > 0:
        blk = np.asarray(ids).reshape(len(cells), per // 16, 16)
        ids = np.stack([blk[:16], blk[16:]], axis=2).reshape(-1).tolist()
    return _grid("C4", cells, seeds_total, n_requests, seed, ids)


def c4_growth(rank=0, world=1, replicas_per_gpu=4096, n_requests=2000, seed=4045,
              policies=(tcm.POLICY_FCFS, tcm.POLICY_TCM, tcm.POLICY_EDF)):
    """NEXT-1 memory-pressure sweep: the C4 grid (KV x lambda) under FCFS, TCM and EDF (with its
    priority-inversion preemption, R34) with decode KV growth and preemption (tcm.KV_GROWTH,
    readings R28-R32) on the stepwise engine -- the three policies of fig:preemptions
    (PAPER.md:620-623).  Footprints are clamped to kv - 2048 so that footprint + out - 1 fits the
    KV capacity (R28)."""
    base = [c for c in c4_cells() if c["policy"] == tcm.POLICY_FCFS]
    cells = [dict(c, policy=pol, gen_kv=c["kv"] - 2048, flags=tcm.KV_GROWTH) for pol in policies for c in base]
    seeds_total = replicas_per_gpu * world // len(cells)
    return _grid("C4-growth", cells, seeds_total, n_requests, seed, rank_ids(len(cells), seeds_total, rank, world))


def c5_cells():
    mixes = [T.MIXES[k] for k in ("TO", "ML", "MH", "70/25/5", "50/20/30", "80/20/0", "80/0/20", "40/40/20")]
    budgets = [256 << i for i in range(8)]                      # 256 .. 32768
    return [dict(rate=0.25 * (i + 1), mix=mx, kv=131072, policy=tcm.POLICY_TCM, alpha=a, budget=b)
            for i in range(16) for mx in mixes for a in ALPHAS for b in budgets]


def c5(rank=0, world=8, replicas=1 << 20, n_requests=10_000, seed=5055):
    """1M replicas x 10k: 16 lambda x 8 mixes x 16 alpha x 8 budgets (16,384 cells) x 64 seeds."""
    cells = c5_cells()
    nc = len(cells)
    return _grid("C5", cells, replicas // nc, n_requests, seed, rank_ids(nc, replicas // nc, rank, world))


def c2prime(replicas=65536, pending=1024, seed=2222):
    """C2': many replicas x ~1k pending requests, for the per-step kernels' HBM
    roofline.  Request 0 of each replica carries 60 s of inline encode time, so when the second
    iteration starts every other request (arrivals spread over ~60 s) is pending with a
    distinct waiting time."""
    rate = pending / 60.0
    cells = [dict(rate=rate, mix=(0.70, 0.25, 0.05), kv=131072, policy=tcm.POLICY_TCM, alpha=1.0, budget=2048)]
    sw = _grid("C2'", cells, replicas, pending, seed, range(replicas))
    return sw


def stage_c2prime(trace_np):
    """Make request 0 of every replica a 60 s-inline image so the clock jumps past all arrivals."""
    off = trace_np.offset
    first = off[:-1].astype(np.int64)
    trace_np.inline_us[first] = 60_000_000
    trace_np.modality[first] = 1
    trace_np.footprint[first] = 800
    return trace_np


def allreduce_aggregate(hist, cnt):
    """Sum the int64 a6 histograms / counters over all ranks (NCCL on GPUs, gloo on CPU).
    Integer sums are order-independent, so the result is bit-identical for any world size."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(hist)
        dist.all_reduce(cnt)
    return hist, cnt
