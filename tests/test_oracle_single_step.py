"""SURVEY.md 8(c) "Brute force on tiny queues": single-step states enumerated exhaustively, with
EXPLICIT partial/waiting flags and decode counts, checked against a declarative restatement.

`orc_decide` is the very code the oracle's engine loop runs for each decision (steps 3-6,
oracle/tcm_oracle.c `orc_admit_step`).  Each state: <= 5 pending requests, each with a class
(M/C/T), a waiting time on a 6-point grid that spans the cross-class crossovers (SURVEY.md 8(c)
"Cross-class order"), a footprint in {1, fits alone, misfits}, and a flag waiting / partial
(a partial already holds its KV and has `rem` < footprint left, R5/R7); chunk budget
B in {1, 3, 8} and n_dec in {0, 1, B} (R8).  The declarative side below is written from
PAPER.md:315, 447-461, 572 and SPEC.md:369-371, 401-403, 421 with readings R3-R8: sort the
pending set by the policy's comparator (priority from the paper's formula with Python's math
library, not K1), then a literal greedy scan.  States whose order hinges on a cross-class
near-tie (|dP| < 1e-11) are skipped, as in tests/spec_engine.py.
"""
import itertools
import random

import numpy as np
import pytest

import oracle as O
from tests.spec_engine import paper_priority

CLOCK = 200_000_000                                   # us; every arrival is CLOCK - wait
WAITS = [0, 2_000_000, 3_112_976, 15_900_000, 46_578_040, 89_614_596]   # spans the crossovers
KV_FREE = 40
FPS = [1, 25, 50]                                     # 1 | fits alone (two do not) | misfits
INL = (0, 170_000, 2_000_000)                         # per class: text / image / video encode
OUT = 3


def spec_decide(reqs, n_dec, B, policy, alpha, skip):
    """reqs: list of dicts (id, arr, f, inl, cls, partial, rem) in id (= arrival) order."""
    budget = max(0, B - n_dec)                                        # R8
    near_tie = False
    if policy == O.TCM:                                               # R3, R4: (P desc, arr, id)
        P = {r["id"]: max(paper_priority(r["cls"], CLOCK - r["arr"], alpha), 1e-12) for r in reqs}
        vals = sorted(reqs, key=lambda r: -P[r["id"]])
        for a, b in zip(vals, vals[1:]):
            if a["cls"] != b["cls"] and P[a["id"]] != P[b["id"]] and abs(P[a["id"]] - P[b["id"]]) < 1e-11:
                near_tie = True
        order = sorted(reqs, key=lambda r: (-P[r["id"]], r["arr"], r["id"]))
    elif policy == O.EDF:                                             # R27: arrival + 5 x iso E2E
        dl = lambda r: r["arr"] + 5 * (r["inl"] + -(-r["f"] // B) * 5000 + 20 * r["f"] + (OUT - 1) * 5500)
        order = sorted(reqs, key=lambda r: (dl(r), r["arr"], r["id"]))
    else:                                                             # FCFS
        order = sorted(reqs, key=lambda r: (r["arr"], r["id"]))
    free, left, blocked = KV_FREE, budget, False
    chunk = {r["id"]: 0 for r in reqs}
    admitted = []
    inl = 0
    for r in order:                                                   # R5-R7 greedy scan
        if left == 0:
            break
        if not r["partial"]:
            if blocked:
                continue
            if r["f"] > free:
                blocked = not skip
                continue
            free -= r["f"]
            admitted.append(r["id"])
            inl += r["inl"]
        chunk[r["id"]] = min(r["rem"], left)
        left -= chunk[r["id"]]
    return chunk, admitted, inl, free, budget, near_tie


def one_state_options():
    for c, w, f, part in itertools.product(range(3), WAITS, FPS, (False, True)):
        if part and f > KV_FREE + 50:
            continue
        yield dict(cls=c, wait=w, f=f, partial=part, rem=(max(1, f // 2) if part else f), inl=INL[c])


OPTS = list(one_state_options())


def build(state):
    # ids in arrival order: longest wait first; equal waits keep their enumeration order
    st = sorted(state, key=lambda o: -o["wait"])
    return [dict(o, id=i, arr=CLOCK - o["wait"]) for i, o in enumerate(st)]


def check(reqs, n_dec, B, policy, alpha=1.0, skip=False):
    chunk, admitted, inl, free, budget, tie = spec_decide(reqs, n_dec, B, policy, alpha, skip)
    if tie:
        return 0
    got = O.decide([r["arr"] for r in reqs], [r["f"] for r in reqs], [r["inl"] for r in reqs],
                   [OUT] * len(reqs), [r["cls"] for r in reqs], [r["rem"] for r in reqs],
                   [1 if r["partial"] else 0 for r in reqs], CLOCK, KV_FREE, n_dec,
                   policy=policy, alpha=alpha, chunk_budget=B, admit_skip=skip)
    ch, adm, tok, inl_o, free_o, bp = got
    assert bp == budget
    assert ch.tolist() == [chunk[r["id"]] for r in reqs], (reqs, n_dec, B, policy)
    assert [i for i in np.argsort(np.where(adm < 0, 1 << 40, adm), kind="stable") if adm[i] >= 0] == admitted
    assert sorted(adm[adm >= 0].tolist()) == list(range(len(admitted)))
    assert tok == sum(chunk.values()) <= budget
    assert inl_o == inl and free_o == free >= 0
    return 1


def _grid(B):
    return sorted({0, 1, B})


@pytest.mark.parametrize("B", [1, 3, 8])
def test_every_state_of_one_and_two_requests(B):
    checked = 0
    for k in (1, 2):
        for state in itertools.product(OPTS, repeat=k):
            reqs = build(state)
            for n_dec in _grid(B):
                for pol, alpha in ((O.FCFS, 1.0), (O.TCM, 1.0), (O.TCM, 0.0)):
                    checked += check(reqs, n_dec, B, pol, alpha)
    assert checked > 0.99 * 3 * len(_grid(B)) * (len(OPTS) + len(OPTS) ** 2)


@pytest.mark.parametrize("k", [3, 4, 5])
def test_sampled_states_of_three_to_five_requests(k):
    rng = random.Random(100 + k)
    checked = 0
    for _ in range(1500):
        reqs = build([rng.choice(OPTS) for _ in range(k)])
        B = rng.choice([1, 3, 8])
        for n_dec in _grid(B):
            for pol, alpha, skip in ((O.FCFS, 1.0, False), (O.TCM, 1.0, False), (O.TCM, 8.0, False),
                                     (O.TCM, 2.0**-7, False), (O.EDF, 1.0, False), (O.TCM, 1.0, True)):
                checked += check(reqs, n_dec, B, pol, alpha, skip)
    assert checked > 20000


def test_decide_is_the_engine_loop():
    # orc_decide and orc_simulate share orc_admit_step: the first decision of a trace whose requests
    # all arrive by the first iteration equals the engine's first iteration (admit order, tokens).
    reqs = [[0, 30, 0, 2, 2], [0, 3, 0, 2, 0], [0, 25, 0, 2, 1], [0, 1, 0, 2, 0]]
    m = O.model(thresholds=((10, 2**32 - 1), (0, 2**32 - 1), (0, 20)))
    a = [r[0] for r in reqs]
    f = [r[1] for r in reqs]
    cls = [O.classify(r[4], r[1], m) for r in reqs]
    for pol in (O.FCFS, O.TCM):
        r = O.simulate(np.array(a), np.array(f), np.zeros(4), np.full(4, 2), np.array([q[4] for q in reqs]),
                       policy=pol, kv_capacity=40, chunk_budget=8, m=m, log=True, max_iters=1)
        ch, adm, tok, _, free, _ = O.decide(a, f, [0] * 4, [2] * 4, cls, f, [0] * 4, 0, 40, 0, policy=pol,
                                            chunk_budget=8, m=m)
        assert int(r.iters[0]["tokens"]) == tok
        assert int(r.iters[0]["kv_free_admit"]) == free
        assert [int(x) for x in r.admit_seq[adm >= 0]] == adm[adm >= 0].tolist()
