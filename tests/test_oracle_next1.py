"""NEXT-1 pins for the oracle: decode KV growth and preemption by recomputation
(readings R28-R32), against hand-worked schedules (tests/golden/preemption.json), the reduction
to the R7 engine when KV never runs out, invariants on tight-KV traces, and the declarative
restatement (tests/spec_engine.py, growth=True) on brute-forced tiny traces."""
import json
import os
import random

import numpy as np
import pytest

import oracle as O
import tracegen as T
from tests import spec_engine

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "preemption.json")))


def run(reqs, policy, **kw):
    tr = T.from_requests(reqs)
    return tr, O.simulate_growth(tr.arrival_us, tr.footprint, tr.inline_us, tr.out_tokens, tr.modality,
                                 policy=policy, **kw)


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
def test_hand_worked_preemption(case):
    pol = {"FCFS": O.FCFS, "TCM": O.TCM, "EDF": O.EDF}[case["policy"]]
    tr, r = run(case["requests"], pol, kv_capacity=case["kv"], chunk_budget=case.get("B", 2048))
    e = case["expect"]
    assert r.status == 0
    assert r.first_token_us.tolist() == e["first"]
    assert r.done_us.tolist() == e["done"]
    assert r.admit_seq.tolist() == e["admit_seq"]
    assert r.preempt_count.tolist() == e["preempt_count"]
    assert r.preempted_us.tolist() == e["preempted_us"]
    assert r.counters["preemptions"] == e["preemptions"]
    assert r.counters["forced_preemptions"] == e["forced"]


def test_capacity_rule():
    # R28: footprint + out - 1 must fit on its own
    _, r = run([[0, 400, 0, 102, 0]], O.FCFS, kv_capacity=500)
    assert r.status == -1
    _, r = run([[0, 400, 0, 101, 0]], O.FCFS, kv_capacity=500)
    assert r.status == 0 and r.counters["preemptions"] == 0


def _trace(seed, n, kv, mix=(0.5, 0.2, 0.3), rate=4.0):
    rep = T.make_replica(seed, 0, n, rate, mix, kv - 2048)    # f + out - 1 <= kv by construction
    return T.generate(np.array([rep]))


@pytest.mark.parametrize("policy", [O.FCFS, O.TCM])
def test_reduces_to_r7_engine_without_memory_pressure(policy):
    # KV larger than every footprint + output together: no preemption, no KV block -> the R7 engine
    tr = _trace(3, 300, 131072)
    big = int(tr.footprint.astype(np.int64).sum() + tr.out_tokens.astype(np.int64).sum()) + 1
    g = O.simulate_trace_growth(tr, 0, policy=policy, kv_capacity=big)
    b = O.simulate_trace(tr, 0, policy=policy, kv_capacity=big)
    assert g.status == 0 and b.status == 0 and g.counters["preemptions"] == 0
    assert np.array_equal(g.admit_seq, b.admit_seq)
    assert np.array_equal(g.first_token_us, b.first_token_us)
    assert np.array_equal(g.done_us, b.done_us)


@pytest.mark.parametrize("policy", [O.FCFS, O.TCM])
@pytest.mark.parametrize("kv", [16384, 32768])
def test_invariants_under_memory_pressure(policy, kv):
    tr = _trace(11, 400, kv, rate=3.0)
    a, b = int(tr.offset[0]), int(tr.offset[1])
    r = O.simulate_trace_growth(tr, 0, policy=policy, kv_capacity=kv)
    assert r.status == 0
    n = b - a
    assert sorted(r.admit_seq.tolist()) == list(range(n))               # every request admitted once
    arr = tr.arrival_us[a:b]
    assert np.all(r.done_us >= r.first_token_us) and np.all(r.first_token_us > arr)
    iso = np.array([O.iso_ttft(int(f), int(il)) for f, il in zip(tr.footprint[a:b], tr.inline_us[a:b])])
    assert np.all(r.first_token_us - arr >= iso)
    assert np.all(r.preempted_us <= r.done_us - arr)
    assert np.all((r.preempt_count == 0) <= (r.preempted_us == 0))
    assert int(r.preempt_count.sum()) == r.counters["preemptions"]
    if policy == O.TCM:   # motorcycles only when every running request is one (R29)
        assert int(r.preempt_count[r.cls == 0].sum()) <= r.counters["forced_preemptions"]
    assert r.counters["preemptions"] > 0                                 # the pressure is real


def test_tcm_spares_motorcycles_vs_fcfs():
    # PAPER.md:620-623 (fig:preemptions): FCFS preempts motorcycles, TCM (almost) never does
    tr = _trace(5, 600, 16384, rate=4.0)
    f = O.simulate_trace_growth(tr, 0, policy=O.FCFS, kv_capacity=16384)
    t = O.simulate_trace_growth(tr, 0, policy=O.TCM, kv_capacity=16384)
    fm = int(f.preempt_count[f.cls == 0].sum())
    tm = int(t.preempt_count[t.cls == 0].sum())
    assert fm > 0 and tm <= t.counters["forced_preemptions"] and tm < fm


def test_brute_force_vs_declarative_engine():
    rng = random.Random(2027)
    checked = edf_pre = 0
    for case in range(400):
        n = rng.randint(1, 6)
        kv = rng.choice([40, 64, 100])
        reqs, t = [], 0
        for _ in range(n):
            t += rng.choice([0, 0, 1, 3000, 40000, 3_000_000])
            f = rng.randint(1, 30)
            out = rng.randint(1, kv - f + 1)
            reqs.append([t, f, rng.choice([0, 0, 700]), out, rng.randint(0, 2)])
        pol = rng.choice([O.FCFS, O.TCM, O.EDF])          # EDF: R34 priority-inversion preemption
        B = rng.choice([1, 3, 8, 64])
        alpha = rng.choice([0.0, 1.0, 64.0])
        sp = spec_engine.run([tuple(x) for x in reqs], pol, alpha=alpha, kv=kv, B=B, growth=True)
        if sp["near_tie"]:
            continue
        _, r = run(reqs, pol, kv_capacity=kv, chunk_budget=B, alpha=alpha)
        assert r.status == 0
        assert r.admit_seq.tolist() == sp["admit_seq"], (case, reqs)
        assert r.first_token_us.tolist() == sp["first"], (case, reqs)
        assert r.done_us.tolist() == sp["done"], (case, reqs)
        assert r.preempt_count.tolist() == sp["preempt_count"], (case, reqs)
        assert r.preempted_us.tolist() == sp["preempted_us"], (case, reqs)
        checked += 1
        edf_pre += pol == O.EDF and r.counters["preemptions"] > 0
    assert checked > 350
    assert edf_pre > 10
