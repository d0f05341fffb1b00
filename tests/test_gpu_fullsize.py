"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

* C4 (bench workload): 65,536 replicas x 10,000 requests on one GPU (fused engine, device-generated
  trace).  Two replicas of EVERY one of the 32 cells -- the heavy TCM cells (lambda 4, KV 16k)
  included, where the closed-form windows L4/L4c/L5 (FP32 bounds) decide ~98 % of the decisions --
  are compared bit-exactly with the full-length oracle, per request (admit_seq, first_token_us,
  done_us) and per replica (iterations, decisions, sum of pending sizes); properties that hold at
  any size are checked on all 655M requests.
* C3: 4,096 replicas x 10,000 requests (lambda x alpha sweep, TCM): the heaviest cells (lambda 4) and
  a spread of the others, full length.
* C2: one queue with 100k pending requests: the first iterations of both engines vs the oracle
  (max_iters), which re-sorts all 100k keys every iteration.
* C2': 65,536 replicas x 1,024 pending, one paper-literal step on both engines vs the oracle.
* C5: rank 0's shard of the 1M-replica sweep (131,072 x 10,000) as `bench.py --workload c5` runs it:
  light cells at full length, and the heaviest cells (lambda 4, MH mix, B = 256) on an oracle
  prefix covering >= 50 % of each replica's iterations.
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
    return r.status, r.admit_seq, r.first_token_us, r.done_us, r.counters


def oracle_many(sw, idx, max_iters=0, gen=None):
    """Oracle runs of replicas idx (max_iters: an int for all, or a list per replica; 0 = full
    length), one single-threaded process per replica on every host core, heaviest first."""
    gen = sw.gen if gen is None else gen
    mi = max_iters if isinstance(max_iters, (list, tuple)) else [max_iters] * len(idx)
    jobs = [(gen[i], int(sw.params[i]["policy"]), int(sw.params[i]["kv_capacity"]),
             float(sw.params[i]["aging_alpha"]), int(sw.params[i]["chunk_budget"]), m) for i, m in zip(idx, mi)]
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        return pool.map(_oracle_job, jobs, chunksize=1)


def run_sweep(sw, engine=tcm.ENGINE_FUSED):
    dev = tcm.generate_device(sw.gen)
    dev["params"] = torch.from_numpy(sw.params.view(np.uint8)).cuda()
    res = tcm.alloc_results(sw.n_requests)
    sim = tcm.Simulation(tcm.config(engine=engine, n_cells=sw.n_cells))
    sim.load(dev, res)
    return sim, dev, res


def compare(sw, res, idx, orc, counters=None, prefix=False):
    """Bit-exact per-request comparison of replicas idx with oracle results orc.  With counters
    (tcm_replica_counters of the GPU run), the per-replica work counters are compared too: iterations,
    decisions (R17) and the sum of pending-set sizes -- the GPU's closed-form decisions plus its
    scanned ones must add up to the oracle's iteration-by-iteration count.  prefix: the oracle ran
    only its first max_iters iterations; every request it stamped must match, and every request it
    did not stamp must be stamped by the GPU after the oracle's final clock."""
    off = np.zeros(sw.n_replicas + 1, np.int64)
    np.cumsum(sw.gen["n_requests"].astype(np.int64), out=off[1:])
    for i, (st, seq, ft, dn, oc) in zip(idx, orc):
        assert st == 0
        a, b = int(off[i]), int(off[i + 1])
        g_seq = res["admit_seq"][a:b].cpu().numpy()
        g_ft = res["first_token_us"][a:b].cpu().numpy()
        g_dn = res["done_us"][a:b].cpu().numpy()
        if not prefix:
            np.testing.assert_array_equal(g_seq, seq, err_msg=f"replica {i}")
            np.testing.assert_array_equal(g_ft, ft, err_msg=f"replica {i}")
            np.testing.assert_array_equal(g_dn, dn, err_msg=f"replica {i}")
            if counters is not None:
                for k in ("iterations", "decisions", "sum_pending"):
                    assert int(counters[k][i]) == int(oc[k]), (i, k, int(counters[k][i]), int(oc[k]))
                assert int(counters["requests_done"][i]) == b - a
            continue
        T_end = int(oc["final_clock"])
        adm = seq != 0xFFFFFFFF
        assert adm.sum() > 0
        np.testing.assert_array_equal(g_seq[adm], seq[adm], err_msg=f"replica {i} (prefix)")
        assert (g_seq[~adm] >= adm.sum()).all()
        for g, o in ((g_ft, ft), (g_dn, dn)):
            m = o != 0
            np.testing.assert_array_equal(g[m], o[m], err_msg=f"replica {i} (prefix)")
            assert (g[~m] > T_end).all(), f"replica {i}: GPU stamped a request the oracle prefix did not"
        if counters is not None:
            assert int(counters["iterations"][i]) >= int(oc["iterations"])


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
    cnt_r = sim.replica_counters(R)
    assert int(cnt_r["requests_done"].sum()) == N
    assert int(cnt_r["decisions"].sum()) == st["decisions"]
    # a6 aggregation: per-cell counts add up
    hist, cnt, _ = sim.aggregate()
    assert int(cnt[:, 3, 0].sum()) == N and int(hist[:, 3].sum()) == N
    # two replicas of EVERY cell vs the full-length oracle, heavy TCM cells included (the oracle keys
    # and sorts every pending request at every decision: minutes per heavy replica, all host cores)
    cells = sw.params["cell_id"]
    idx = [int(np.nonzero(cells == c)[0][k]) for c in range(sw.n_cells) for k in (0, 977)]
    heavy_first = sorted(idx, key=lambda i: -int(cnt_r["sum_pending"][i]))
    # the sampled heavy TCM cells really are the ones the closed-form windows carry
    tcm_heavy = [i for i in idx if sw.cells[cells[i]]["policy"] == tcm.POLICY_TCM and sw.cells[cells[i]]["rate"] == 4.0]
    assert all(int(cnt_r["scanned_decisions"][i]) * 4 < int(cnt_r["decisions"][i]) for i in tcm_heavy)
    compare(sw, res, heavy_first, oracle_many(sw, heavy_first), counters=cnt_r)


def test_c3_sweep_sampled_bit_exact():
    sw = W.c3(0, 1, replicas=4096, n_requests=10_000)
    sim, dev, res = run_sweep(sw)
    sim.run()
    assert sim.stats()["requests_done"] == sw.n_requests
    cnt_r = sim.replica_counters(sw.n_replicas)
    lam = np.array([sw.cells[c]["rate"] for c in sw.params["cell_id"]])
    # the heaviest cells (lambda 4, every alpha), plus a spread of the rest
    heavy = [int(i) for i in np.nonzero(lam == 4.0)[0][::16]]
    idx = heavy + [int(i) for i in np.nonzero(lam < 4.0)[0][::173]][:16]
    idx = sorted(idx, key=lambda i: -int(cnt_r["sum_pending"][i]))
    compare(sw, res, idx, oracle_many(sw, idx), counters=cnt_r)


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
    cnt_r = sim.replica_counters(sw.n_replicas)
    cells = sw.params["cell_id"]
    light = [c for c, cell in enumerate(sw.cells) if cell["rate"] <= 0.5 and cell["budget"] >= 2048][::97][:12]
    idx = [int(np.nonzero(cells == c)[0][0]) for c in light]
    compare(sw, res, idx, oracle_many(sw, idx), counters=cnt_r)
    # the heaviest cells (lambda 4, MH mix, B = 256): an oracle prefix of >= 50 % of each replica's
    # iterations (a full-length oracle run keys thousands of pending requests per decision for hours)
    mh = T.MIXES["MH"]
    heavy = [c for c, cell in enumerate(sw.cells) if cell["rate"] == 4.0 and cell["budget"] == 256 and
             tuple(cell["mix"]) == tuple(mh)][::4]
    idx = [int(np.nonzero(cells == c)[0][0]) for c in heavy]
    mi = [int((int(cnt_r["iterations"][i]) + 1) // 2) for i in idx]
    compare(sw, res, idx, oracle_many(sw, idx, max_iters=mi), counters=cnt_r, prefix=True)
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
    # NEXT-1 at the size bench.py times (C4-growth, 1,536 x 1,000, stepwise engine; FCFS, TCM and EDF
    # cells): one replica per cell
    sw = W.c4_growth(0, 1, replicas_per_gpu=1536, n_requests=1000)
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


def test_c4_heavy_subset_fused_equals_stepwise_full_length():
    # 1,024 replicas of the heaviest C4 TCM cells (lambda 4 at every KV, lambda 2 at KV 16k/32k) at
    # the full 10,000 requests: the fused engine (closed-form windows L3-L5, FP32-bound ordering)
    # against the paper-literal stepwise engine (every pending request re-keyed in exact FP64 each
    # iteration, no L4/L5), on every request and every per-replica counter but `scanned`
    import gc
    full = W.c4(0, 1, replicas_per_gpu=65536, n_requests=10_000)
    cells = full.params["cell_id"]
    heavy = [c for c, cell in enumerate(full.cells) if cell["policy"] == tcm.POLICY_TCM and
             (cell["rate"] == 4.0 or (cell["rate"] == 2.0 and cell["kv"] <= 32768))]
    idx = np.concatenate([np.nonzero(cells == c)[0][: 1024 // len(heavy) + 1] for c in heavy])[:1024]
    sw = W.Sweep("C4-heavy", full.gen[idx], full.params[idx], full.n_cells, full.cells)
    outs = []
    for engine in (tcm.ENGINE_FUSED, tcm.ENGINE_STEPWISE):
        sim, dev, res = run_sweep(sw, engine)
        sim.run()
        c = sim.replica_counters(sw.n_replicas)
        outs.append(({k: v.cpu().numpy() for k, v in res.items()}, c))
        sim.close()
        del dev, res
        gc.collect()
    for k in outs[0][0]:
        np.testing.assert_array_equal(outs[0][0][k], outs[1][0][k], err_msg=k)
    for k in ("iterations", "decisions", "sum_pending", "requests_done"):
        np.testing.assert_array_equal(outs[0][1][k], outs[1][1][k], err_msg=k)
    assert int(outs[0][1]["scanned_decisions"].sum()) * 10 < int(outs[0][1]["decisions"].sum())


def test_c4_growth_fused_full_size_sampled_bit_exact():
    # NEXT-1 at the C4 size bench.py's `next1` leg times: 65,536 replicas x 10,000 requests, FCFS and
    # TCM cells with KV growth, fused engine (k_fgrow).  Two replicas of every cell against the
    # full-length growth oracle, per request (admit_seq, first token, done, preempt count, preempted
    # time); properties on all requests.
    sw = W.c4_growth(0, 1, replicas_per_gpu=65536, n_requests=10_000,
                     policies=(tcm.POLICY_FCFS, tcm.POLICY_TCM))
    dev = tcm.generate_device(sw.gen)
    dev["params"] = torch.from_numpy(sw.params.view(np.uint8)).cuda()
    res = tcm.alloc_results(sw.n_requests, preemption=True)
    sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells))
    sim.load(dev, res)
    sim.run()
    st = sim.stats()
    assert st["requests_done"] == sw.n_requests and st["first_bad_replica"] == -1 and st["preemptions"] > 0
    cells = sw.params["cell_id"]
    idx = [int(i) for c in range(sw.n_cells) for i in np.nonzero(cells == c)[0][[5, 1000]]]
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
    # every request admitted once, first token before done, preempted time within its E2E
    assert bool((res["done_us"].view(torch.int64) >= res["first_token_us"].view(torch.int64)).all())
    assert int(res["preempt_count"].view(torch.int32).to(torch.int64).sum()) == st["preemptions"]
    sim.close()
