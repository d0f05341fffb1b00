"""Replica sharding through libtcm: two ranks on one GPU, each simulating its shard
of a C4-shaped sweep with the fused engine, all-reduce their int64 a6 histograms / counters over
gloo (CUDA tensors) -- the bench's NCCL all-reduce with another backend -- and must reproduce a
single-process run of the whole sweep bit-exactly (integer sums are order-independent).  The
per-replica results of each shard must equal the corresponding replicas of the single run."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2603_26498_b200 import _build, tcm  # noqa: E402
from paper_2603_26498_b200 import workloads as W  # noqa: E402

REPLICAS, REQUESTS = 512, 800


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_shard(sw):
    dev = tcm.generate_device(sw.gen)
    dev["params"] = torch.from_numpy(sw.params.view(np.uint8)).cuda()
    res = tcm.alloc_results(sw.n_requests)
    sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells))
    sim.load(dev, res)
    sim.run()
    hist, cnt, st = sim.aggregate()
    out = {k: v.cpu().numpy() for k, v in res.items()}
    sim.close()
    return hist, cnt, out, st


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sw = W.c4(rank, world, replicas_per_gpu=REPLICAS // world, n_requests=REQUESTS)
    hist, cnt, out, st = run_shard(sw)
    W.allreduce_aggregate(hist, cnt)           # CUDA tensors over gloo
    q.put((rank, hist.cpu().numpy(), cnt.cpu().numpy(), out, st["requests_done"], sw.ids))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_through_libtcm_equal_one():
    _build.build()
    full = W.c4(0, 1, replicas_per_gpu=REPLICAS, n_requests=REQUESTS)
    H, C, out1, _ = run_shard(full)
    H, C = H.cpu().numpy(), C.cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got.sort(key=lambda g: g[0])
    assert sum(g[4] for g in got) == full.n_requests
    assert sorted(np.concatenate([g[5] for g in got]).tolist()) == sorted(full.ids.tolist())
    for rank, h, c, out, _, gids in got:
        np.testing.assert_array_equal(h, H)       # all-reduced = single process, bit-exact
        np.testing.assert_array_equal(c, C)
        # the shard's replicas by global id, located in the single run (both apply the C4 warp layout)
        pos = {int(g): j for j, g in enumerate(full.ids)}
        off1 = np.concatenate([[0], np.cumsum(full.gen["n_requests"].astype(np.int64))])
        off = 0
        for g in gids:
            j = pos[int(g)]
            a, b = int(off1[j]), int(off1[j + 1])
            for k in out:
                np.testing.assert_array_equal(out[k][off:off + b - a], out1[k][a:b], err_msg=f"rank {rank} g {g} {k}")
            off += b - a
