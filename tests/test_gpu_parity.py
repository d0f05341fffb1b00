"""GPU parity: libtcm (through the C ABI) vs the CPU oracle, bit-exact on per-request
admit_seq, first_token_us and done_us, plus K1, generator and aggregation parity."""
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

ENGINES = [tcm.ENGINE_FUSED, tcm.ENGINE_STEPWISE]
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "schedules.json")))


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()
    tcm.lib()


def run_gpu(tr, params, engine=tcm.ENGINE_FUSED, cfg=None, mem=tcm.MEM_DEVICE, step=None):
    cfg = cfg or tcm.config(engine=engine)
    cfg.engine = engine
    sim = tcm.Simulation(cfg)
    if mem == tcm.MEM_DEVICE:
        dev = tcm.to_device(tr, params)
        res = tcm.alloc_results(tr.n_requests)
        sim.load(dev, res)
    else:
        host = {"req_offset": tr.offset, "arrival_us": tr.arrival_us, "footprint": tr.footprint,
                "inline_us": tr.inline_us, "out_tokens": tr.out_tokens, "modality": tr.modality,
                "params": params}
        res = {"admit_seq": np.zeros(tr.n_requests, np.uint32),
               "first_token_us": np.zeros(tr.n_requests, np.uint64),
               "done_us": np.zeros(tr.n_requests, np.uint64)}
        sim.load(host, res, mem=tcm.MEM_HOST)
    if step is None:
        sim.run()
    else:
        while sim.step(step) > 0:
            pass
    out = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in res.items()}
    st = sim.stats()
    return sim, out, st


def check_replicas(tr, params, out, replicas, m=None):
    for r in replicas:
        a, b = int(tr.offset[r]), int(tr.offset[r + 1])
        o = O.simulate_trace(tr, r, policy=int(params["policy"][r]), alpha=float(params["aging_alpha"][r]),
                             kv_capacity=int(params["kv_capacity"][r]),
                             chunk_budget=int(params["chunk_budget"][r]), m=m)
        assert o.status == 0
        np.testing.assert_array_equal(out["admit_seq"][a:b], o.admit_seq, err_msg=f"replica {r} admit_seq")
        np.testing.assert_array_equal(out["first_token_us"][a:b], o.first_token_us, err_msg=f"replica {r} first")
        np.testing.assert_array_equal(out["done_us"][a:b], o.done_us, err_msg=f"replica {r} done")


# ------------------------------------------------------------------------------------ K1
def test_k1_bit_exact_vs_oracle():
    rng = np.random.default_rng(0)
    n = 200_000
    cls = rng.integers(0, 3, n).astype(np.uint8)
    w = (10 ** rng.uniform(0, 10.5, n)).astype(np.uint64)
    w[:100] = 0
    alpha = rng.choice([0.0, 2.0**-7, 0.25, 1.0, 3.0, 128.0], n)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    tcm.tcm_k1_eval(tcm.config(), torch.from_numpy(cls).cuda(), torch.from_numpy(w).cuda(),
                    torch.from_numpy(alpha).cuda(), out)
    got = out.cpu().numpy()
    idx = rng.choice(n, 20_000, replace=False)
    want = np.array([O.priority(int(cls[i]), int(w[i]), float(alpha[i])) for i in idx])
    np.testing.assert_array_equal(got[idx].view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("c", [0, 1, 2])
def test_k1_monotone_full_range(c):
    # Lemma L1 audit at every microsecond of [0, 2^33) (~2.4 h of waiting) per class.
    first = torch.empty(1, dtype=torch.uint64, device="cuda")
    tcm.tcm_k1_audit(tcm.config(), c, 1.0, 0, 2**33, first)
    assert int(first.cpu().numpy()[0]) == 2**64 - 1


@pytest.mark.parametrize("alpha", [2.0**-7, 2.0**-3, 0.5, 2.0, 8.0, 32.0, 128.0])
def test_k1_monotone_alpha_grid(alpha):
    first = torch.empty(1, dtype=torch.uint64, device="cuda")
    for c in range(3):
        tcm.tcm_k1_audit(tcm.config(), c, alpha, 0, 2**31, first)
        assert int(first.cpu().numpy()[0]) == 2**64 - 1, (c, alpha)


# ---------------------------------------------------------------------- hand-worked schedules
@pytest.mark.parametrize("engine", ENGINES, ids=["fused", "stepwise"])
def test_golden_schedules(engine):
    for case in GOLD["cases"]:
        for pol, code in (("FCFS", tcm.POLICY_FCFS), ("TCM", tcm.POLICY_TCM)):
            tr = T.from_requests(case["requests"])
            params = tcm.make_params(1, policy=code, chunk_budget=case["B"], kv_capacity=case["kv"])
            _, out, _ = run_gpu(tr, params, engine)
            exp = case["expect"][pol]
            assert (out["first_token_us"] - tr.arrival_us).tolist() == exp["ttft"], (case["name"], pol)
            assert out["admit_seq"].tolist() == exp["admit_seq"], (case["name"], pol)
            if "e2e" in exp:
                assert (out["done_us"] - tr.arrival_us).tolist() == exp["e2e"], (case["name"], pol)


# --------------------------------------------------------------------- random multi-replica
def sweep(R, n, seed, kvs=(131072, 32768, 16384), rates=(0.5, 2.0, 6.0), mixes=((0.7, 0.25, 0.05), (0.5, 0.2, 0.3))):
    rng = np.random.default_rng(seed)
    reps, params = [], tcm.make_params(R)
    for r in range(R):
        kv = int(rng.choice(kvs))
        mix = mixes[rng.integers(len(mixes))]
        nr = int(rng.integers(max(1, n // 3), n + 1))
        reps.append(T.make_replica(seed, r, nr, float(rng.choice(rates)), mix, kv))
        params[r]["kv_capacity"] = kv
        params[r]["policy"] = rng.choice([tcm.POLICY_FCFS, tcm.POLICY_TCM])
        params[r]["aging_alpha"] = rng.choice([0.0, 2.0**-7, 1.0, 16.0])
        params[r]["chunk_budget"] = rng.choice([256, 2048, 8192])
    return T.generate(np.array(reps)), params


@pytest.mark.parametrize("engine", ENGINES, ids=["fused", "stepwise"])
def test_random_replicas_bit_exact(engine):
    tr, params = sweep(256, 400, 17)
    _, out, st = run_gpu(tr, params, engine)
    assert st["replicas_active"] == 0 and st["first_bad_replica"] == -1
    assert st["requests_done"] == tr.n_requests
    check_replicas(tr, params, out, range(256))


def test_counters_match_oracle():
    tr, params = sweep(64, 300, 5)
    _, out, st = run_gpu(tr, params)
    dec = it = sp = 0
    for r in range(64):
        o = O.simulate_trace(tr, r, policy=int(params["policy"][r]), alpha=float(params["aging_alpha"][r]),
                             kv_capacity=int(params["kv_capacity"][r]), chunk_budget=int(params["chunk_budget"][r]))
        dec += o.counters["decisions"]
        it += o.counters["iterations"]
        sp += o.counters["sum_pending"]
    assert st["decisions"] == dec and st["iterations"] == it and st["sum_pending"] == sp


@pytest.mark.parametrize("engine", ENGINES, ids=["fused", "stepwise"])
@pytest.mark.parametrize("step", [1, 7, 1000])
def test_step_granularity_is_invisible(engine, step):
    tr, params = sweep(32, 150, 23)
    _, ref, _ = run_gpu(tr, params, engine)
    _, out, _ = run_gpu(tr, params, engine, step=step)
    for k in ref:
        np.testing.assert_array_equal(ref[k], out[k])


def test_host_buffers_equal_device_buffers():
    tr, params = sweep(48, 300, 31)
    _, a, _ = run_gpu(tr, params)
    _, b, _ = run_gpu(tr, params, mem=tcm.MEM_HOST)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])


def test_run_async_equals_run():
    """tcm_run_async + tcm_wait (the pipelined e2e path) gives tcm_run's results and counters, twice in a
    row on one context; calls during a pending run are refused; the stepwise engine refuses the call."""
    tr, params = sweep(48, 300, 37)
    _, a, sa = run_gpu(tr, params, mem=tcm.MEM_HOST)
    host = {"req_offset": tr.offset, "arrival_us": tr.arrival_us, "footprint": tr.footprint,
            "inline_us": tr.inline_us, "out_tokens": tr.out_tokens, "modality": tr.modality, "params": params}
    sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED))
    for rep in range(2):
        res = {k: np.zeros_like(v) for k, v in a.items()}
        sim.load(host, res, mem=tcm.MEM_HOST)
        sim.run_async()
        with pytest.raises(tcm.TcmError):
            sim.step(1)                                   # TCM_E_STATE while pending
        sim.wait(tcm.WAIT_ENGINE)
        sp = sim.stats()                                  # allowed before the copy-back is done
        sim.wait(tcm.WAIT_ALL)
        assert sp["decisions"] == sa["decisions"] and sp["requests_done"] == sa["requests_done"]
        sim.wait(tcm.WAIT_ALL)                            # nothing pending: a no-op
        for k in a:
            np.testing.assert_array_equal(res[k], a[k], err_msg=f"rep {rep} {k}")
        sb = sim.stats()
        for k in ("iterations", "decisions", "sum_pending", "requests_done", "scanned_decisions"):
            assert sb[k] == sa[k], k
    sim.close()
    sw = tcm.Simulation(tcm.config(engine=tcm.ENGINE_STEPWISE))
    sw.load(tcm.to_device(tr, params), tcm.alloc_results(tr.n_requests))
    with pytest.raises(tcm.TcmError):
        sw.run_async()
    sw.close()


def test_engines_agree_on_heavy_load():
    tr, params = sweep(64, 1500, 41, kvs=(16384,), rates=(4.0,), mixes=((0.5, 0.2, 0.3),))
    _, a, sa = run_gpu(tr, params, tcm.ENGINE_FUSED)
    _, b, sb = run_gpu(tr, params, tcm.ENGINE_STEPWISE)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])
    assert sa["decisions"] == sb["decisions"] and sa["sum_pending"] == sb["sum_pending"]
    check_replicas(tr, params, a, [0, 13, 63])


# ---------------------------------------------------------------------------- edge cases
@pytest.mark.parametrize("engine", ENGINES, ids=["fused", "stepwise"])
def test_edge_cases(engine):
    # empty replica, single request, all arrivals at t=0, out=1 everywhere, out=2048, B=1
    parts = [T.from_requests([]), T.from_requests([[5, 1, 0, 1, 0]])]
    z = T.generate(np.array([T.make_replica(3, 0, 600, 1.0, (0.5, 0.2, 0.3), 40000, T.FLAG_ALL_AT_ZERO)]))
    parts.append(z)
    o1 = T.generate(np.array([T.make_replica(4, 0, 300, 8.0, (0.7, 0.25, 0.05), 131072)]))
    o1.out_tokens[:] = 1
    parts.append(o1)
    o2 = T.generate(np.array([T.make_replica(5, 0, 50, 0.2, (0.7, 0.25, 0.05), 131072)]))
    o2.out_tokens[:] = 2048
    parts.append(o2)
    tr = T.concat(parts)
    params = tcm.make_params(len(parts))
    params["kv_capacity"] = [131072, 131072, 40000, 131072, 131072]
    params["chunk_budget"] = [2048, 1, 2048, 2048, 2048]
    for pol in (tcm.POLICY_FCFS, tcm.POLICY_TCM):
        params["policy"] = pol
        _, out, st = run_gpu(tr, params, engine)
        assert st["requests_done"] == tr.n_requests
        check_replicas(tr, params, out, range(len(parts)))


def test_validation_errors():
    tr = T.from_requests([[0, 500, 0, 1, 0]])
    with pytest.raises(tcm.TcmError) as e:
        run_gpu(tr, tcm.make_params(1, kv_capacity=400))
    assert e.value.code == -3                       # TCM_E_CAPACITY (R18)
    tr = T.from_requests([[0, 5, 0, 3000, 0]])
    with pytest.raises(tcm.TcmError) as e:
        run_gpu(tr, tcm.make_params(1))
    assert e.value.code == -1                       # out > 2048
    tr = T.from_requests([[10, 5, 0, 3, 0], [5, 5, 0, 3, 0]])
    with pytest.raises(tcm.TcmError) as e:
        run_gpu(tr, tcm.make_params(1))
    assert e.value.code == -1                       # arrivals out of order


# --------------------------------------------------------------------- generator, a6
def test_device_generator_bit_identical():
    reps = np.array([T.make_replica(99, r, 1000 + 37 * r, 0.5 + r, T.MIXES["MH"], 16384 << (r % 3))
                     for r in range(40)])
    host = T.generate(reps)
    dev = tcm.generate_device(reps)
    np.testing.assert_array_equal(dev["req_offset"].cpu().numpy(), host.offset)
    for k in ("arrival_us", "footprint", "inline_us", "out_tokens", "modality"):
        np.testing.assert_array_equal(dev[k].cpu().numpy(), getattr(host, k), err_msg=k)


def test_aggregation_matches_oracle():
    tr, params = sweep(96, 500, 77)
    params["cell_id"] = np.arange(96) % 5
    cfg = tcm.config(n_cells=5)
    sim, out, _ = run_gpu(tr, params, cfg=cfg)
    hist, cnt, _ = sim.aggregate()
    H = np.zeros((5, O.GROUPS, O.HIST_BINS), np.int64)
    C = np.zeros((5, O.GROUPS, O.NCNT), np.int64)
    for r in range(96):
        a, b = int(tr.offset[r]), int(tr.offset[r + 1])
        res = O.Result(out["admit_seq"][a:b], out["first_token_us"][a:b], out["done_us"][a:b], None, {}, None, 0)
        cell = int(params["cell_id"][r])
        O.aggregate(tr.replica(r), res, chunk_budget=int(params["chunk_budget"][r]), hist=H[cell], cnt=C[cell])
    np.testing.assert_array_equal(hist.cpu().numpy(), H)
    np.testing.assert_array_equal(cnt.cpu().numpy(), C)


@pytest.mark.parametrize("alpha", [1.0, 2.0**-7, 0.125, 8.0, 128.0])
def test_filter_bound_within_delta(alpha):
    # The stepwise engine skips the exact key of a request only when its FP32 bound proves it
    # cannot enter the top-32; that is exact iff |P~ - P| <= delta = 1e-4.  Audit every us of
    # [0, 2^28) and a 97-us lattice of [0, 2^36) per class (the design bound is < 1e-5).
    for c in range(3):
        e1 = tcm.tcm_k1_filter_error(tcm.config(), c, alpha, 0, 2**28, 1)
        e2 = tcm.tcm_k1_filter_error(tcm.config(), c, alpha, 0, 2**36, 97)
        assert max(e1, e2) < 1e-5, (c, alpha, e1, e2)


# ------------------------------------------------------------------------------- NEXT-3
def test_next3_policies_stepwise_bit_exact():
    # EDF, naive aging and first-fit admission on the stepwise
    # engine (general top-k path) vs the oracle
    tr, params = sweep(160, 400, 61, kvs=(131072, 16384), rates=(1.0, 4.0))
    rng = np.random.default_rng(3)
    params["policy"] = rng.choice([tcm.POLICY_EDF, tcm.POLICY_NAIVE_AGING, tcm.POLICY_TCM, tcm.POLICY_FCFS], 160)
    params["flags"] = rng.choice([0, tcm.ADMIT_SKIP], 160)
    _, out, st = run_gpu(tr, params, tcm.ENGINE_STEPWISE)
    assert st["requests_done"] == tr.n_requests
    for r in range(160):
        a, b = int(tr.offset[r]), int(tr.offset[r + 1])
        o = O.simulate_trace(tr, r, policy=int(params["policy"][r]), alpha=float(params["aging_alpha"][r]),
                             kv_capacity=int(params["kv_capacity"][r]), chunk_budget=int(params["chunk_budget"][r]),
                             admit_skip=bool(params["flags"][r]))
        assert o.status == 0
        np.testing.assert_array_equal(out["admit_seq"][a:b], o.admit_seq, err_msg=f"replica {r}")
        np.testing.assert_array_equal(out["first_token_us"][a:b], o.first_token_us, err_msg=f"replica {r}")
        np.testing.assert_array_equal(out["done_us"][a:b], o.done_us, err_msg=f"replica {r}")


def test_next3_naive_aging_fused_and_rejections():
    tr, params = sweep(32, 300, 62)
    params["policy"] = tcm.POLICY_NAIVE_AGING
    _, out, _ = run_gpu(tr, params, tcm.ENGINE_FUSED)
    check_replicas(tr, params, out, range(32))
    # the fused engine relies on Lemmas L1/L2, which EDF and first-fit break: refused loudly
    for pol, fl in ((tcm.POLICY_EDF, 0), (tcm.POLICY_TCM, tcm.ADMIT_SKIP)):
        p2 = params.copy()
        p2["policy"], p2["flags"] = pol, fl
        with pytest.raises(tcm.TcmError) as e:
            run_gpu(tr, p2, tcm.ENGINE_FUSED)
        assert e.value.code == -1


def test_calibrated_thresholds_bit_exact():
    # NEXT-4: thresholds learned by the calibration pipeline drive both engines (R13)
    from paper_2603_26498_b200 import calibration as K
    cal = T.generate(np.array([T.make_replica(42, r, 300, 1.0, (1 / 3, 1 / 3, 1 / 3), 131072) for r in range(3)]))
    thr, _, _ = K.calibrate(cal)
    tr, params = sweep(64, 300, 63)
    m = O.model(thresholds=thr)
    for engine in ENGINES:
        cfg = tcm.config(engine=engine, thresholds=thr)
        _, out, _ = run_gpu(tr, params, engine, cfg=cfg)
        check_replicas(tr, params, out, range(64), m=m)


@pytest.mark.parametrize("mode", ["1", "8", "cluster"])
def test_stepwise_launch_modes_bit_exact(mode, monkeypatch):
    # every group mode of k_step (warp, CTA, 8-CTA cluster per replica) on the same sweep; the
    # automatic choice depends on the replica count and size, so force each one (TCM_SW_GROUP)
    monkeypatch.setenv("TCM_SW_GROUP", mode)
    tr, params = sweep(40, 400, 81)
    _, out, st = run_gpu(tr, params, tcm.ENGINE_STEPWISE)
    assert st["requests_done"] == tr.n_requests
    check_replicas(tr, params, out, range(40))


# ------------------------------------------------------------------------ brute force
def _tiny_cases(outs=(1, 3)):
    """SURVEY.md 8(c) brute force on tiny queues (the grid of tests/test_oracle_engine.py)."""
    import itertools
    import random
    fps = [1, 17, 30]
    arrivals = [0, 1, 3_200_000, 47_000_000, 90_000_000]
    one = list(itertools.product(arrivals, fps, [0, 95_000_000], list(outs), [0, 1, 2]))
    rng = random.Random(9)
    cases = [[a] for a in one]
    cases += [sorted([rng.choice(one) for _ in range(k)]) for k in (2, 3, 4) for _ in range(600)]
    return [[list(r) for r in c] for c in cases]


@pytest.mark.parametrize("engine", ENGINES, ids=["fused", "stepwise"])
def test_brute_force_tiny_queues_as_replicas(engine):
    # every tiny trace x B in {1,3,8} x {FCFS, TCM} as one replica of a single GPU batch, each
    # compared bit-exactly with the oracle (thresholds that map the footprints to all classes)
    thr = ((10, 2**32 - 1), (0, 2**32 - 1), (0, 20))
    m = O.model(thresholds=thr)
    cases = _tiny_cases()
    combos = [(c, B, pol) for c in cases for B in (1, 3, 8) for pol in (tcm.POLICY_FCFS, tcm.POLICY_TCM)]
    tr = T.concat([T.from_requests(c) for c, _, _ in combos])
    params = tcm.make_params(len(combos), kv_capacity=40)
    params["chunk_budget"] = [B for _, B, _ in combos]
    params["policy"] = [p for _, _, p in combos]
    cfg = tcm.config(engine=engine, thresholds=thr)
    _, out, st = run_gpu(tr, params, engine, cfg=cfg)
    assert st["requests_done"] == tr.n_requests and st["first_bad_replica"] == -1
    for r, (c, B, pol) in enumerate(combos):
        a, b = int(tr.offset[r]), int(tr.offset[r + 1])
        o = O.simulate_trace(tr, r, policy=int(pol), kv_capacity=40, chunk_budget=B, m=m)
        assert o.status == 0
        assert out["admit_seq"][a:b].tolist() == o.admit_seq.tolist(), (c, B, pol)
        assert out["first_token_us"][a:b].tolist() == o.first_token_us.tolist(), (c, B, pol)
        assert out["done_us"][a:b].tolist() == o.done_us.tolist(), (c, B, pol)


def test_brute_force_tiny_queues_growth_stepwise():
    # the same batch under NEXT-1 (KV growth + preemption, R28-R32) on the stepwise engine
    thr = ((10, 2**32 - 1), (0, 2**32 - 1), (0, 20))
    m = O.model(thresholds=thr)
    # outputs up to 9 tokens so that decode growth exhausts the 40-token KV (17 + 8 twice > 40)
    combos = [(c, B, pol) for c in _tiny_cases(outs=(1, 9)) for B in (1, 3, 8)
              for pol in (tcm.POLICY_FCFS, tcm.POLICY_TCM)]
    tr = T.concat([T.from_requests(c) for c, _, _ in combos])
    params = tcm.make_params(len(combos), kv_capacity=40)
    params["chunk_budget"] = [B for _, B, _ in combos]
    params["policy"] = [p for _, _, p in combos]
    params["flags"] = tcm.KV_GROWTH
    sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_STEPWISE, thresholds=thr))
    dev = tcm.to_device(tr, params)
    res = tcm.alloc_results(tr.n_requests, preemption=True)
    sim.load(dev, res)
    sim.run()
    out = {k: v.cpu().numpy() for k, v in res.items()}
    npre = 0
    for r, (c, B, pol) in enumerate(combos):
        a, b = int(tr.offset[r]), int(tr.offset[r + 1])
        o = O.simulate_trace_growth(tr, r, policy=int(pol), kv_capacity=40, chunk_budget=B, m=m)
        assert o.status == 0
        for k, v in (("admit_seq", o.admit_seq), ("first_token_us", o.first_token_us), ("done_us", o.done_us),
                     ("preempt_count", o.preempt_count), ("preempted_us", o.preempted_us)):
            assert out[k][a:b].tolist() == v.tolist(), (k, c, B, pol)
        npre += o.counters["preemptions"]
    assert npre > 0 and sim.stats()["preemptions"] == npre
    sim.close()
