"""GPU parity for NEXT-1 (decode KV growth + preemption by recomputation, readings R28-R32) on
the stepwise engine through the C ABI: bit-exact per-request admit_seq, first_token_us, done_us,
preempt_count and preempted_us, and equal work / preemption counters, against the CPU oracle."""
import json
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

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "preemption.json")))


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()
    tcm.lib()


def run_gpu(tr, params, engine=tcm.ENGINE_STEPWISE, step=None):
    sim = tcm.Simulation(tcm.config(engine=engine))
    dev = tcm.to_device(tr, params)
    res = tcm.alloc_results(tr.n_requests, preemption=True)
    sim.load(dev, res)
    if step is None:
        sim.run()
    else:
        while sim.step(step) > 0:
            pass
    out = {k: v.cpu().numpy() for k, v in res.items()}
    st = sim.stats()
    sim.close()
    return out, st


def growth_sweep(R, n, seed, kvs=(16384, 32768), rates=(1.0, 3.0, 6.0), mixes=((0.5, 0.2, 0.3), (0.7, 0.25, 0.05)),
                 policies=(tcm.POLICY_FCFS, tcm.POLICY_TCM)):
    rng = np.random.default_rng(seed)
    reps, params = [], tcm.make_params(R)
    for r in range(R):
        kv = int(rng.choice(kvs))
        mix = mixes[rng.integers(len(mixes))]
        nr = int(rng.integers(max(1, n // 3), n + 1))
        reps.append(T.make_replica(seed, r, nr, float(rng.choice(rates)), mix, kv - 2048))   # f + out - 1 <= kv
        params[r]["kv_capacity"] = kv
        params[r]["policy"] = rng.choice(list(policies))
        params[r]["aging_alpha"] = rng.choice([0.0, 2.0**-7, 1.0, 16.0])
        params[r]["chunk_budget"] = rng.choice([256, 2048, 8192])
        params[r]["flags"] = tcm.KV_GROWTH
    return T.generate(np.array(reps)), params


def check(tr, params, out, replicas):
    tot_pre = tot_forced = dec = sp = it = 0
    for r in replicas:
        a, b = int(tr.offset[r]), int(tr.offset[r + 1])
        kw = dict(policy=int(params["policy"][r]), alpha=float(params["aging_alpha"][r]),
                  kv_capacity=int(params["kv_capacity"][r]), chunk_budget=int(params["chunk_budget"][r]))
        if params["flags"][r] & tcm.KV_GROWTH:
            o = O.simulate_trace_growth(tr, r, **kw)
            np.testing.assert_array_equal(out["preempt_count"][a:b], o.preempt_count, err_msg=f"replica {r} pcount")
            np.testing.assert_array_equal(out["preempted_us"][a:b], o.preempted_us, err_msg=f"replica {r} ptime")
            tot_pre += o.counters["preemptions"]
            tot_forced += o.counters["forced_preemptions"]
        else:
            o = O.simulate_trace(tr, r, **kw)
            assert not out["preempt_count"][a:b].any()
        assert o.status == 0
        np.testing.assert_array_equal(out["admit_seq"][a:b], o.admit_seq, err_msg=f"replica {r} admit_seq")
        np.testing.assert_array_equal(out["first_token_us"][a:b], o.first_token_us, err_msg=f"replica {r} first")
        np.testing.assert_array_equal(out["done_us"][a:b], o.done_us, err_msg=f"replica {r} done")
        dec += o.counters["decisions"]
        sp += o.counters["sum_pending"]
        it += o.counters["iterations"]
    return dict(preemptions=tot_pre, forced=tot_forced, decisions=dec, sum_pending=sp, iterations=it)


# every golden on the stepwise engine; FCFS / TCM ones also on the fused engine (k_fgrow) -- EDF is
# not class-monotone and runs on the stepwise engine only
_CASES = [(c, tcm.ENGINE_STEPWISE) for c in GOLD["cases"]] + \
         [(c, tcm.ENGINE_FUSED) for c in GOLD["cases"] if c["policy"] != "EDF"]


@pytest.mark.parametrize("case,engine", _CASES,
                         ids=[c["name"] + ("-fused" if e == tcm.ENGINE_FUSED else "-stepwise") for c, e in _CASES])
def test_hand_worked_preemption_gpu(case, engine):
    tr = T.from_requests(case["requests"])
    params = tcm.make_params(1, kv_capacity=case["kv"])
    params["policy"] = {"FCFS": tcm.POLICY_FCFS, "TCM": tcm.POLICY_TCM, "EDF": tcm.POLICY_EDF}[case["policy"]]
    params["chunk_budget"] = case.get("B", 2048)
    params["flags"] = tcm.KV_GROWTH
    out, st = run_gpu(tr, params, engine=engine)
    e = case["expect"]
    assert out["first_token_us"].tolist() == e["first"]
    assert out["done_us"].tolist() == e["done"]
    assert out["admit_seq"].tolist() == e["admit_seq"]
    assert out["preempt_count"].tolist() == e["preempt_count"]
    assert out["preempted_us"].tolist() == e["preempted_us"]
    assert st["preemptions"] == e["preemptions"] and st["forced_preemptions"] == e["forced"]


@pytest.mark.parametrize("step", [None, 7])
def test_random_growth_replicas_bit_exact(step):
    tr, params = growth_sweep(96, 500, 71)
    out, st = run_gpu(tr, params, step=step)
    assert st["requests_done"] == tr.n_requests and st["first_bad_replica"] == -1
    c = check(tr, params, out, range(96))
    assert c["preemptions"] > 0
    assert st["preemptions"] == c["preemptions"] and st["forced_preemptions"] == c["forced"]
    assert st["decisions"] == c["decisions"] and st["sum_pending"] == c["sum_pending"]
    assert st["iterations"] == c["iterations"]


def test_mixed_growth_and_plain_replicas():
    # growth and R7 replicas in one load: the growth instantiation must keep plain replicas exact
    tr, params = growth_sweep(64, 400, 72)
    params["flags"][::2] = 0
    out, st = run_gpu(tr, params)
    check(tr, params, out, range(64))


def test_warp_per_replica_path_sampled():
    # >= 2x the resident warp slots -> one warp per replica (k_step<1, true>)
    tr, params = growth_sweep(8192, 120, 73, kvs=(4096,), rates=(8.0,))
    out, st = run_gpu(tr, params)
    assert st["requests_done"] == tr.n_requests
    c = check(tr, params, out, range(0, 8192, 128))
    assert st["preemptions"] > 0 and c["preemptions"] > 0


def test_growth_rejections():
    tr, params = growth_sweep(4, 100, 74)
    params["policy"] = tcm.POLICY_EDF
    with pytest.raises(tcm.TcmError) as e:          # EDF keys are not class-monotone: stepwise only
        run_gpu(tr, params, engine=tcm.ENGINE_FUSED)
    assert e.value.code == -1
    tr = T.from_requests([[0, 400, 0, 102, 0]])      # R28: 400 + 102 - 1 > 500
    params = tcm.make_params(1, kv_capacity=500)
    params["flags"] = tcm.KV_GROWTH
    with pytest.raises(tcm.TcmError) as e:
        run_gpu(tr, params)
    assert e.value.code == -3


def test_growth_edge_cases():
    # empty replica, a lone request, out = 1 everywhere (no growth), B = 1, KV exactly f + out - 1
    reqs = [
        [],
        [[0, 100, 0, 1, 0]],
        [[0, 50, 0, 1, 0], [0, 60, 0, 1, 1], [5, 70, 0, 1, 2]],
        [[0, 8, 0, 5, 0], [0, 10, 0, 3, 0], [1, 4, 0, 4, 1]],
        [[0, 200, 0, 301, 0]],
        [[0, 3, 0, 8, 0], [0, 3, 0, 6, 1]],
    ]
    kvs = [100, 100, 100, 14, 500, 16]
    budgets = [2048, 2048, 1, 1, 2048, 2]
    tr = T.concat([T.from_requests(r) for r in reqs]) if hasattr(T, "concat") else None
    if tr is None:
        pytest.skip("tracegen.concat not available")
    params = tcm.make_params(len(reqs))
    params["kv_capacity"] = kvs
    params["chunk_budget"] = budgets
    params["flags"] = tcm.KV_GROWTH
    for pol in (tcm.POLICY_FCFS, tcm.POLICY_TCM):
        params["policy"] = pol
        out, st = run_gpu(tr, params)
        c = check(tr, params, out, range(len(reqs)))
        assert st["requests_done"] == tr.n_requests
        assert c["preemptions"] > 0 and st["preemptions"] == c["preemptions"]


@pytest.mark.parametrize("mode", ["1", "8", "cluster"])
def test_growth_launch_modes_bit_exact(mode, monkeypatch):
    monkeypatch.setenv("TCM_SW_GROUP", mode)
    tr, params = growth_sweep(24, 400, 75)
    out, st = run_gpu(tr, params)
    c = check(tr, params, out, range(24))
    assert c["preemptions"] > 0 and st["preemptions"] == c["preemptions"]


def test_device_preemption_stats_equal_oracle():
    # fig:preemptions counters (tcm_preemption_stats) per (cell, class): the device classifies with the
    # engine's a1 classifier; the oracle side sums its per-request results by orc_classify
    tr, params = growth_sweep(64, 400, 75)
    params["cell_id"] = np.arange(64) % 4
    sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_STEPWISE, n_cells=4))
    dev = tcm.to_device(tr, params)
    res = tcm.alloc_results(tr.n_requests, preemption=True)
    sim.load(dev, res)
    sim.run()
    got = sim.preemption_stats().cpu().numpy()
    sim.close()
    want = np.zeros((4, 4, 3), np.int64)
    for r in range(64):
        a, b = int(tr.offset[r]), int(tr.offset[r + 1])
        o = O.simulate_trace_growth(tr, r, policy=int(params["policy"][r]), alpha=float(params["aging_alpha"][r]),
                                    kv_capacity=int(params["kv_capacity"][r]),
                                    chunk_budget=int(params["chunk_budget"][r]))
        for i in range(b - a):
            if o.preempt_count[i]:
                g = O.classify(int(tr.modality[a + i]), int(tr.footprint[a + i]))
                for gg in (g, 3):
                    want[r % 4, gg] += (int(o.preempt_count[i]), int(o.preempted_us[i]), 1)
    assert want[:, 3, 0].sum() > 0
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("launch", [None, "1", "8"])
def test_edf_inversion_preemption_bit_exact(launch, monkeypatch):
    # NEXT-3 EDF with its priority-inversion preemption (R34) under KV growth, every
    # launch mode of the stepwise engine, against the oracle
    if launch:
        monkeypatch.setenv("TCM_SW_GROUP", launch)
    tr, params = growth_sweep(48, 400, 76, policies=(tcm.POLICY_EDF,))
    out, st = run_gpu(tr, params)
    c = check(tr, params, out, range(48))
    assert c["preemptions"] > 0 and st["preemptions"] == c["preemptions"]
    assert st["decisions"] == c["decisions"] and st["sum_pending"] == c["sum_pending"]


@pytest.mark.parametrize("step", [None, 5])
def test_fused_growth_random_replicas_bit_exact(step):
    # NEXT-1 on the fused engine (k_fgrow: class-FIFO merge + preempted stacks, R28-R32) vs the oracle
    tr, params = growth_sweep(96, 500, 81)
    out, st = run_gpu(tr, params, engine=tcm.ENGINE_FUSED, step=step)
    assert st["requests_done"] == tr.n_requests and st["first_bad_replica"] == -1
    c = check(tr, params, out, range(96))
    assert c["preemptions"] > 0
    assert st["preemptions"] == c["preemptions"] and st["forced_preemptions"] == c["forced"]
    assert st["decisions"] == c["decisions"] and st["sum_pending"] == c["sum_pending"]
    assert st["iterations"] == c["iterations"]


def test_fused_growth_mixed_with_plain_replicas():
    # k_fused runs the R7 replicas, k_fgrow the growth ones, in one load
    tr, params = growth_sweep(64, 400, 82)
    params["flags"][::2] = 0
    out, st = run_gpu(tr, params, engine=tcm.ENGINE_FUSED)
    c = check(tr, params, out, range(64))
    assert st["preemptions"] == c["preemptions"]


def test_fused_growth_tight_kv_many_preemptions():
    # heavy memory pressure: small KV, long outputs, both policies and the alpha grid
    tr, params = growth_sweep(64, 300, 83, kvs=(4096, 6144), rates=(4.0, 8.0))
    out, st = run_gpu(tr, params, engine=tcm.ENGINE_FUSED)
    c = check(tr, params, out, range(64))
    assert c["preemptions"] > 200 and st["preemptions"] == c["preemptions"]
    assert st["forced_preemptions"] == c["forced"]
