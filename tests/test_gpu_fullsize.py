"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

* C4 (bench workload): 65,536 replicas x 10,000 requests on one GPU (fused engine, device-generated
  trace).  Sampled replicas (every FCFS cell + the light TCM cells, which the oracle finishes in
  seconds) are compared bit-exactly with the oracle; properties that hold at any size are checked
  on all 655M requests.
* C3: 4,096 replicas x 10,000 requests (lambda x alpha sweep, TCM): sampled light replicas.
* C2: one queue with 100k pending requests: the first iterations of both engines vs the oracle
  (max_iters), which re-sorts all 100k keys every iteration.
* C2': 65,536 replicas x 1,024 pending, one paper-literal step on both engines vs the oracle.
* C5: rank 0's shard of the 1M-replica sweep (131,072 x 10,000) as `bench.py --workload c5` runs it.
* NEXT-1: the C4-growth sweep at the size bench.py times (stepwise engine), one replica per cell.
"""
import multiprocessing as mp
import os

import numpy as np
import pytest

import oracle as O
import tracegen as T

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2603_26498_b200 import _build, tcm  # noqa: E402
from paper_2603_26498_b200 import workloads as W  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()
    tcm.lib()


def _oracle_job(job):
    gen, pol, kv, alpha, budget, max_iters = job
    tr = T.generate(np.array([gen], dtype=T.TG_REPLICA_DTYPE))
    r = O.simulate_trace(tr, 0, policy=pol, alpha=alpha, kv_capacity=kv, chunk_budget=budget,
                         max_iters=max_iters)
    return r.status, r.admit_seq, r.first_token_us, r.done_us


def oracle_many(sw, idx, max_iters=0, gen=None):
    gen = sw.gen if gen is None else gen
    jobs = [(gen[i], int(sw.params[i]["policy"]), int(sw.params[i]["kv_capacity"]),
             float(sw.params[i]["aging_alpha"]), int(sw.params[i]["chunk_budget"]), max_iters) for i in idx]
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        return pool.map(_oracle_job, jobs, chunksize=1)


def run_sweep(sw, engine=tcm.ENGINE_FUSED):
    dev = tcm.generate_device(sw.gen)
    dev["params"] = torch.from_numpy(sw.params.view(np.uint8)).cuda()
    res = tcm.alloc_results(sw.n_requests)
    sim = tcm.Simulation(tcm.config(engine=engine, n_cells=sw.n_cells))
    sim.load(dev, res)
    return sim, dev, res


def compare(sw, res, idx, orc):
    off = np.zeros(sw.n_replicas + 1, np.int64)
    np.cumsum(sw.gen["n_requests"].astype(np.int64), out=off[1:])
    for i, (st, seq, ft, dn) in zip(idx, orc):
        assert st == 0
        a, b = int(off[i]), int(off[i + 1])
        np.testing.assert_array_equal(res["admit_seq"][a:b].cpu().numpy(), seq, err_msg=f"replica {i}")
        np.testing.assert_array_equal(res["first_token_us"][a:b].cpu().numpy(), ft, err_msg=f"replica {i}")
        np.testing.assert_array_equal(res["done_us"][a:b].cpu().numpy(), dn, err_msg=f"replica {i}")


def test_c4_bench_workload_sampled_bit_exact_and_properties():
    sw = W.c4(0, 1, replicas_per_gpu=65536, n_requests=10_000)
    sim, dev, res = run_sweep(sw)
    sim.run()
    st = sim.stats()
    N, R = sw.n_requests, sw.n_replicas
    assert st["requests_done"] == N and st["replicas_done"] == R and st["first_bad_replica"] == -1
    # properties on all 655M requests: every request admitted once, first token after its
    # isolated TTFT, completion after the first token, admit_seq a permutation per replica
    off = dev["req_offset"].to(torch.int64)
    n = (off[1:] - off[:-1])
    seq = res["admit_seq"].to(torch.int64)
    assert int(seq.max()) < 10_000
    rep = torch.repeat_interleave(torch.arange(R, device="cuda"), n)
    s = torch.zeros(R, dtype=torch.int64, device="cuda").index_add_(0, rep, seq)
    assert torch.equal(s, n * (n - 1) // 2)
    arr = dev["arrival_us"].to(torch.int64)
    ft = res["first_token_us"].to(torch.int64)
    dn = res["done_us"].to(torch.int64)
    f = dev["footprint"].to(torch.int64)
    iso = dev["inline_us"].to(torch.int64) + (f + 2047) // 2048 * 5000 + 20 * f
    assert bool(((ft - arr) >= iso).all()) and bool((dn >= ft).all())
    # sampled replicas vs the oracle: every FCFS cell and the light TCM cells
    cells = sw.params["cell_id"]
    light = [c for c, cell in enumerate(sw.cells) if cell["policy"] == tcm.POLICY_FCFS or
             (cell["rate"] <= 1.0 and cell["kv"] >= 65536)]
    idx = [int(np.nonzero(cells == c)[0][k]) for c in light for k in (0, 977)]
    compare(sw, res, idx, oracle_many(sw, idx))
    # a6 aggregation: per-cell counts add up
    hist, cnt, _ = sim.aggregate()
    assert int(cnt[:, 3, 0].sum()) == N and int(hist[:, 3].sum()) == N


def test_c3_sweep_sampled_bit_exact():
    sw = W.c3(0, 1, replicas=4096, n_requests=10_000)
    sim, dev, res = run_sweep(sw)
    sim.run()
    assert sim.stats()["requests_done"] == sw.n_requests
    lam = np.array([sw.cells[c]["rate"] for c in sw.params["cell_id"]])
    idx = [int(i) for i in np.nonzero(lam <= 1.5)[0][::97]][:24]
    compare(sw, res, idx, oracle_many(sw, idx))


def _stage_c2(replicas, pending, engine):
    sw = W.c2prime(replicas=replicas, pending=pending)
    tr = T.generate(sw.gen)
    W.stage_c2prime(tr)
    dev = tcm.to_device(tr, sw.params)
    res = tcm.alloc_results(tr.n_requests)
    sim = tcm.Simulation(tcm.config(engine=engine))
    sim.load(dev, res)
    return sw, tr, sim, res


@pytest.mark.parametrize("engine", [tcm.ENGINE_FUSED, tcm.ENGINE_STEPWISE], ids=["fused", "stepwise"])
def test_c2_single_queue_100k_first_steps(engine):
    iters = 6
    sw, tr, sim, res = _stage_c2(1, 100_000, engine)
    for _ in range(iters):
        sim.step(1)
    o = O.simulate_trace(tr, 0, policy=O.TCM, max_iters=iters)
    assert o.counters["iterations"] == iters
    np.testing.assert_array_equal(res["admit_seq"].cpu().numpy(), o.admit_seq)
    np.testing.assert_array_equal(res["first_token_us"].cpu().numpy(), o.first_token_us)
    np.testing.assert_array_equal(res["done_us"].cpu().numpy(), o.done_us)
    st = sim.stats()
    assert st["decisions"] == o.counters["decisions"] and st["sum_pending"] == o.counters["sum_pending"]


def test_c2prime_one_step_both_engines_and_oracle():
    iters = 4
    outs = []
    for engine in (tcm.ENGINE_FUSED, tcm.ENGINE_STEPWISE):
        sw, tr, sim, res = _stage_c2(65536, 1024, engine)
        for _ in range(iters):
            sim.step(1)
        outs.append({k: v.cpu().numpy() for k, v in res.items()})
        sim.close()
    for k in outs[0]:
        np.testing.assert_array_equal(outs[0][k], outs[1][k])
    for r in (0, 12345, 65535):
        a, b = int(tr.offset[r]), int(tr.offset[r + 1])
        o = O.simulate_trace(tr, r, policy=O.TCM, max_iters=iters)
        np.testing.assert_array_equal(outs[1]["admit_seq"][a:b], o.admit_seq)
        np.testing.assert_array_equal(outs[1]["first_token_us"][a:b], o.first_token_us)


def test_c5_per_gpu_shard_sampled_bit_exact():
    # C5 (configs[4]) at full size per GPU: rank 0's shard of the 1M-replica sweep (131,072
    # replicas x 10,000 requests), as `bench.py --workload c5` runs it; light sampled cells
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    sw = W.c5(0, 8, replicas=1 << 20, n_requests=10_000)
    assert sw.n_replicas == 131072
    sim, dev, res = run_sweep(sw)
    sim.run()
    st = sim.stats()
    assert st["requests_done"] == sw.n_requests and st["first_bad_replica"] == -1
    cells = sw.params["cell_id"]
    light = [c for c, cell in enumerate(sw.cells) if cell["rate"] <= 0.5 and cell["budget"] >= 2048][::97][:12]
    idx = [int(np.nonzero(cells == c)[0][0]) for c in light]
    compare(sw, res, idx, oracle_many(sw, idx))
    sim.close()
    del dev, res
    gc.collect()
    torch.cuda.empty_cache()


def _oracle_growth_job(job):
    gen, pol, kv, alpha, budget = job
    tr = T.generate(np.array([gen], dtype=T.TG_REPLICA_DTYPE))
    r = O.simulate_trace_growth(tr, 0, policy=pol, alpha=alpha, kv_capacity=kv, chunk_budget=budget)
    return r.status, r.admit_seq, r.first_token_us, r.done_us, r.preempt_count, r.preempted_us


def test_c4_growth_bench_config_sampled_bit_exact():
    # NEXT-1 at the size bench.py times (C4-growth, 1,024 x 1,000, stepwise engine): one replica per cell
    sw = W.c4_growth(0, 1, replicas_per_gpu=1024, n_requests=1000)
    dev = tcm.generate_device(sw.gen)
    dev["params"] = torch.from_numpy(sw.params.view(np.uint8)).cuda()
    res = tcm.alloc_results(sw.n_requests, preemption=True)
    sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_STEPWISE, n_cells=sw.n_cells))
    sim.load(dev, res)
    sim.run()
    st = sim.stats()
    assert st["requests_done"] == sw.n_requests and st["preemptions"] > 0
    cells = sw.params["cell_id"]
    idx = [int(np.nonzero(cells == c)[0][3]) for c in range(sw.n_cells)]
    jobs = [(sw.gen[i], int(sw.params[i]["policy"]), int(sw.params[i]["kv_capacity"]),
             float(sw.params[i]["aging_alpha"]), int(sw.params[i]["chunk_budget"])) for i in idx]
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        orc = pool.map(_oracle_growth_job, jobs, chunksize=1)
    off = np.zeros(sw.n_replicas + 1, np.int64)
    np.cumsum(sw.gen["n_requests"].astype(np.int64), out=off[1:])
    for i, (s_, seq, ft, dn, pc, pt) in zip(idx, orc):
        assert s_ == 0
        a, b = int(off[i]), int(off[i + 1])
        for k, v in (("admit_seq", seq), ("first_token_us", ft), ("done_us", dn), ("preempt_count", pc),
                     ("preempted_us", pt)):
            np.testing.assert_array_equal(res[k][a:b].cpu().numpy(), v, err_msg=f"replica {i} {k}")
    sim.close()
