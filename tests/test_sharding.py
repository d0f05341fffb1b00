"""Replica sharding across ranks: shards are disjoint, cover the sweep,
balance the cells, and the all-reduced int64 aggregation equals the single-process one
bit-exactly.  Runs world_size 2 over gloo on CPU; per-replica results come from the oracle
(the GPU path is exercised by tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import tracegen as T
from paper_2603_26498_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def aggregate_shard(sw):
    """Run every replica of a shard through the oracle and aggregate into (hist, cnt)."""
    tr = T.generate(sw.gen)
    H = np.zeros((sw.n_cells, O.GROUPS, O.HIST_BINS), np.int64)
    C = np.zeros((sw.n_cells, O.GROUPS, O.NCNT), np.int64)
    for r in range(sw.n_replicas):
        p = sw.params[r]
        res = O.simulate_trace(tr, r, policy=int(p["policy"]), alpha=float(p["aging_alpha"]),
                               kv_capacity=int(p["kv_capacity"]), chunk_budget=int(p["chunk_budget"]))
        assert res.status == 0
        cell = int(p["cell_id"])
        O.aggregate(tr.replica(r), res, chunk_budget=int(p["chunk_budget"]), hist=H[cell], cnt=C[cell])
    return H, C


def small_c4(rank, world):
    return W.c4(rank, world, replicas_per_gpu=64 // world, n_requests=120)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sw = small_c4(rank, world)
    H, C = aggregate_shard(sw)
    h, c = torch.from_numpy(H), torch.from_numpy(C)
    W.allreduce_aggregate(h, c)
    if rank == 0:
        q.put((h.numpy().copy(), c.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_shards_partition_the_sweep():
    full = small_c4(0, 1)
    parts = [small_c4(r, 2) for r in range(2)]
    seeds = np.concatenate([p.gen["seed"] for p in parts])
    assert len(seeds) == full.n_replicas and set(seeds.tolist()) == set(full.gen["seed"].tolist())
    for p in parts:                               # cyclic assignment keeps every cell on every rank
        assert set(p.params["cell_id"].tolist()) == set(range(32))
    assert W.rank_ids(2, 4, 1, 2) == [1 * 2 + 0, 3 * 2 + 0, 1 * 2 + 1, 3 * 2 + 1]
    for p in parts:                               # equal share of every cell
        assert np.all(np.bincount(p.params["cell_id"], minlength=32) == 1)


def test_allreduce_equals_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    h, c = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    H, C = aggregate_shard(small_c4(0, 1))
    np.testing.assert_array_equal(h, H)
    np.testing.assert_array_equal(c, C)


def test_c5_and_growth_sweeps_shard_cleanly():
    # C5 (1M replicas at 8 GPUs): rank r holds seeds r, r+8, ... of every one of the 16,384 cells;
    # shards are disjoint and together equal the single-process sweep (checked at 1/64 scale)
    nc = len(W.c5_cells())
    assert nc == 16 * 8 * 16 * 8
    full = set(W.rank_ids(nc, 16, 0, 1))
    parts = [set(W.rank_ids(nc, 16, r, 8)) for r in range(8)]
    assert sum(len(p) for p in parts) == len(full) and set().union(*parts) == full
    for r, p in enumerate(parts):
        assert {g % nc for g in p} == set(range(nc)) and all((g // nc) % 8 == r for g in p)
    # NEXT-1 sweep: every replica has the growth flag and footprint + out - 1 fits its KV (R28)
    sw = W.c4_growth(0, 1, replicas_per_gpu=64, n_requests=200)
    assert np.all(sw.params["flags"] == 2)
    tr = T.generate(sw.gen)
    for r in range(sw.n_replicas):
        a, b = int(tr.offset[r]), int(tr.offset[r + 1])
        kv = int(sw.params["kv_capacity"][r])
        assert np.all(tr.footprint[a:b].astype(np.int64) + tr.out_tokens[a:b] - 1 <= kv)


def test_c4_sweep_ids_cover_the_rank_ids():
    """Sweep.ids (the global replica id of each loaded replica, after the C4 warp layout) is a permutation
    of the rank's rank_ids, and the ranks of a world partition the single-rank sweep."""
    full = W.c4(0, 1, replicas_per_gpu=1024, n_requests=10)
    assert sorted(full.ids.tolist()) == sorted(W.rank_ids(len(full.cells), 1024 // len(full.cells), 0, 1))
    parts = [W.c4(r, 2, replicas_per_gpu=512, n_requests=10).ids.tolist() for r in range(2)]
    assert sorted(parts[0] + parts[1]) == sorted(full.ids.tolist())
    # every replica's cell and generator record follow its global id
    for j, g in enumerate(full.ids[:64]):
        assert int(full.params["cell_id"][j]) == int(g) % len(full.cells)
