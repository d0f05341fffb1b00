"""Pins for the oracle's engine loop.

Each test pins the oracle to something other than itself: hand-worked schedules
(tests/golden/schedules.json), the isolated closed form, reductions
to FCFS / static priority, invariants on every iteration, and a declarative restatement
of the step (tests/spec_engine.py) on brute-forced tiny traces.
"""
import itertools
import json
import os
import random

import numpy as np
import pytest

import oracle as O
import tracegen as T
from tests import spec_engine

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "schedules.json")))


def run(reqs, policy, **kw):
    tr = T.from_requests(reqs)
    return tr, O.simulate(tr.arrival_us, tr.footprint, tr.inline_us, tr.out_tokens, tr.modality,
                          policy=policy, **kw)


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
@pytest.mark.parametrize("pol", ["FCFS", "TCM"])
def test_hand_worked_schedules(case, pol):
    tr, r = run(case["requests"], O.FCFS if pol == "FCFS" else O.TCM,
                kv_capacity=case["kv"], chunk_budget=case["B"])
    assert r.status == 0
    exp = case["expect"][pol]
    assert (r.first_token_us - tr.arrival_us).tolist() == exp["ttft"]
    assert r.admit_seq.tolist() == exp["admit_seq"]
    if "e2e" in exp:
        assert (r.done_us - tr.arrival_us).tolist() == exp["e2e"]


def test_iteration_time_examples():
    # SPEC.md:137-139 re-derived in integer us (R9; App. B corrects the third example):
    # dt(400 tok, 0 dec, 0 inline) = 13000 ; dt(0 tok, 8 dec) = 9000 ; dt(2048, 4 dec, 1 s) = 1047960
    tr, r = run([[0, 400, 0, 1, 0]], O.FCFS)
    assert r.first_token_us[0] == 13000
    reqs = [[0, 1, 0, 3, 0]] * 8
    tr, r = run(reqs, O.FCFS, log=True)
    it = r.iters
    assert it[1]["n_dec"] == 8 and it[1]["tokens"] == 0
    assert it[1]["clock_end"] - it[1]["clock_start"] == 9000
    reqs = [[0, 1, 0, 3, 0]] * 4 + [[1, 2048, 1_000_000, 1, 2]]
    tr, r = run(reqs, O.FCFS, log=True, chunk_budget=2052)
    it = r.iters
    assert it[1]["n_dec"] == 4 and it[1]["tokens"] == 2048
    assert it[1]["clock_end"] - it[1]["clock_start"] == 1_047_960


@pytest.mark.parametrize("mod", [0, 1, 2])
def test_single_request_equals_isolated_closed_form(mod):
    # SPEC.md:478 / acceptance 4: a single-request simulation equals isolated_e2e exactly.
    rng = random.Random(100 + mod)
    for _ in range(100):
        f = rng.randint(1, 60000)
        inl = 0 if mod == 0 else rng.randint(0, 3_000_000)
        out = rng.randint(1, 2048)
        B = rng.choice([1, 7, 512, 2048, 8192])
        for pol in (O.FCFS, O.TCM):
            tr, r = run([[rng.randint(0, 10**9), f, inl, out, mod]], pol, chunk_budget=B,
                        kv_capacity=65536)
            assert r.first_token_us[0] - tr.arrival_us[0] == O.iso_ttft(f, inl, B)
            assert r.done_us[0] - tr.arrival_us[0] == O.iso_e2e(f, inl, out, B)
            # closed form written out here as well
            assert O.iso_e2e(f, inl, out, B) == inl + -(-f // B) * 5000 + 20 * f + (out - 1) * 5500


def _gen(n, rate, mix, kv, seed, replica=0):
    return T.generate(np.array([T.make_replica(seed, replica, n, rate, mix, kv)]))


def test_reduction_one_class_equals_fcfs():
    # (i) all requests in one class -> priority is FIFO (Lemma L1) -> TCM == FCFS bit-exactly
    for seed in range(6):
        tr = _gen(600, 3.0, (1.0, 0.0, 0.0), 131072, seed)
        tr.footprint[:] = np.minimum(tr.footprint, 4095)          # every text stays a motorcycle
        a = O.simulate_trace(tr, 0, policy=O.FCFS, kv_capacity=20000)
        b = O.simulate_trace(tr, 0, policy=O.TCM, kv_capacity=20000)
        assert np.array_equal(a.admit_seq, b.admit_seq)
        assert np.array_equal(a.first_token_us, b.first_token_us)
        assert np.array_equal(a.done_us, b.done_us)


def test_reduction_equal_params_equals_fcfs():
    # (iii) S, k, p equal for all classes -> the key depends on waiting time only -> FCFS
    m = O.model(S=(0.1, 0.1, 0.1), k=(0.003,) * 3, p=(2.5,) * 3)
    for seed in range(4):
        tr = _gen(500, 2.0, (0.5, 0.2, 0.3), 32768, seed)
        a = O.simulate_trace(tr, 0, policy=O.FCFS, kv_capacity=32768, m=m)
        b = O.simulate_trace(tr, 0, policy=O.TCM, kv_capacity=32768, m=m)
        assert np.array_equal(a.admit_seq, b.admit_seq)
        assert np.array_equal(a.first_token_us, b.first_token_us)


def test_reduction_alpha_zero_is_strict_class_order():
    # (ii) alpha = 0: static priority M -> C -> T, FCFS within a class:
    # the declarative engine with key (class, arrival, id) must agree exactly.
    for seed in range(4):
        tr = _gen(300, 3.0, (0.5, 0.2, 0.3), 32768, seed)
        r = O.simulate_trace(tr, 0, policy=O.TCM, alpha=0.0, kv_capacity=32768)
        reqs = list(zip(tr.arrival_us.tolist(), tr.footprint.tolist(), tr.inline_us.tolist(),
                        tr.out_tokens.tolist(), tr.modality.tolist()))
        s = spec_engine.run(reqs, 1, alpha=0.0, kv=32768)
        assert r.admit_seq.tolist() == s["admit_seq"]
        assert r.first_token_us.tolist() == s["first"]


def test_reduction_infinite_resources_policy_independent():
    # (iv) infinite KV and budget: every arrival is admitted in its first iteration, so
    # TTFT and E2E do not depend on the policy.
    for seed in range(4):
        tr = _gen(400, 4.0, (0.5, 0.2, 0.3), 2**31, seed)
        a = O.simulate_trace(tr, 0, policy=O.FCFS, kv_capacity=2**31, chunk_budget=10**8)
        b = O.simulate_trace(tr, 0, policy=O.TCM, kv_capacity=2**31, chunk_budget=10**8)
        assert np.array_equal(a.first_token_us, b.first_token_us)
        assert np.array_equal(a.done_us, b.done_us)


@pytest.mark.parametrize("pol", [O.FCFS, O.TCM])
@pytest.mark.parametrize("kv,rate,mix", [(131072, 2.0, (0.7, 0.25, 0.05)),
                                         (16384, 4.0, (0.5, 0.2, 0.3)),
                                         (32768, 1.0, (0.6, 0.25, 0.15))])
def test_invariants_every_iteration(pol, kv, rate, mix):
    tr = _gen(800, rate, mix, kv, 11)
    B = 2048
    r = O.simulate_trace(tr, 0, policy=pol, kv_capacity=kv, chunk_budget=B, log=True)
    assert r.status == 0                                  # no deadlock under R6 (acceptance 10)
    it = r.iters
    n = len(tr.arrival_us)
    assert np.all(it["tokens"] <= it["budget"])           # chunk budget
    assert np.all(it["budget"] == np.maximum(0, B - it["n_dec"].astype(np.int64)))
    assert np.all(it["kv_free_admit"] <= kv)              # reserve-on-admit never overdraws
    assert np.all(it["clock_end"] > it["clock_start"])    # clock strictly advances
    assert np.all(it["clock_start"][1:] >= it["clock_end"][:-1])
    assert np.all(it["n_partial_after"] <= (3 if pol == O.TCM else 1))   # Lemma L2
    assert sorted(r.admit_seq.tolist()) == list(range(n))  # admit_seq is a permutation
    assert np.all(r.first_token_us > tr.arrival_us)       # first token exactly once, after arrival
    assert np.all(r.done_us >= r.first_token_us)
    iso_t = np.array([O.iso_ttft(int(f), int(i), B) for f, i in zip(tr.footprint, tr.inline_us)])
    assert np.all(r.first_token_us - tr.arrival_us >= iso_t)   # TTFT >= isolated TTFT
    assert it["n_first_tokens"].sum() == n
    # work conservation: a pending request that fits is never left idle
    assert np.all((it["n_pending"] == 0) | (it["tokens"] > 0) | (it["budget"] == 0)
                  | (it["kv_free_start"] < 1) | (it["n_dec"] > 0))
    # determinism
    r2 = O.simulate_trace(tr, 0, policy=pol, kv_capacity=kv, chunk_budget=B)
    assert np.array_equal(r.first_token_us, r2.first_token_us)
    assert r.counters == r2.counters


def test_random_traces_match_declarative_engine():
    # Whole-engine pin: moderate random traces vs the declarative restatement.
    rng = random.Random(5)
    checked = 0
    for trial in range(40):
        n = rng.randint(5, 60)
        kv = rng.choice([3000, 12000, 40000, 131072])
        B = rng.choice([64, 512, 2048])
        tr = _gen(n, rng.choice([0.5, 2.0, 8.0]), (0.5, 0.25, 0.25), kv, 1000 + trial)
        reqs = list(zip(tr.arrival_us.tolist(), tr.footprint.tolist(), tr.inline_us.tolist(),
                        tr.out_tokens.tolist(), tr.modality.tolist()))
        for pol in (O.FCFS, O.TCM):
            for alpha in ([1.0] if pol == O.FCFS else [1.0, 0.125, 16.0]):
                s = spec_engine.run(reqs, pol, alpha=alpha, kv=kv, B=B)
                if s["near_tie"]:
                    continue
                r = O.simulate_trace(tr, 0, policy=pol, alpha=alpha, kv_capacity=kv, chunk_budget=B)
                assert r.admit_seq.tolist() == s["admit_seq"]
                assert r.first_token_us.tolist() == s["first"]
                assert r.done_us.tolist() == s["done"]
                checked += 1
    assert checked >= 150


def test_brute_force_tiny_traces():
    # SURVEY.md 8(c) "Brute force on tiny queues": enumerate small traces over a grid of
    # classes, footprints {1, fits, misfits}, waits spanning the crossovers, budgets and outs.
    kv = 40
    fps = [1, 17, 30]                         # two of 30 never fit together
    arrivals = [0, 1, 3_200_000, 47_000_000, 90_000_000]
    inlines = [0, 95_000_000]
    mods = [0, 1, 2]
    thr = ((10, 2**32 - 1), (0, 2**32 - 1), (0, 20))   # footprints map to all three classes
    m = O.model(thresholds=thr)
    one = list(itertools.product(arrivals, fps, inlines, [1, 3], mods))
    rng = random.Random(9)
    cases = [[a] for a in one]
    cases += [sorted([rng.choice(one) for _ in range(k)]) for k in (2, 3, 4) for _ in range(600)]
    checked = 0
    for reqs in cases:
        reqs = [list(r) for r in reqs]
        for B in (1, 3, 8):
            for pol in (O.FCFS, O.TCM):
                s = spec_engine.run(reqs, pol, kv=kv, B=B, thr=thr)
                if s["near_tie"]:
                    continue
                tr, r = run(reqs, pol, kv_capacity=kv, chunk_budget=B, m=m)
                assert r.status == 0
                assert r.admit_seq.tolist() == s["admit_seq"], (reqs, B, pol)
                assert r.first_token_us.tolist() == s["first"], (reqs, B, pol)
                assert r.done_us.tolist() == s["done"], (reqs, B, pol)
                checked += 1
    assert checked > 10000


def test_rejects_capacity_violation():
    # SPEC.md:456 CapacityImpossible / R18: a footprint above KV capacity is an input error
    tr, r = run([[0, 500, 0, 1, 0]], O.FCFS, kv_capacity=400)
    assert r.status == -1
