"""Pins for the a6 aggregation (PAPER.md:579 SLO = 5x isolated E2E)."""
import numpy as np

import oracle as O
import tracegen as T


def test_bucket_properties():
    # HDR-style log buckets: exact below 16, then 8 sub-buckets per power of two.
    assert [O.ttft_bucket(t) for t in range(16)] == list(range(16))
    for k in range(4, 64):
        assert O.ttft_bucket(2**k) == 16 + 8 * (k - 4)          # closed form at powers of two
    assert O.ttft_bucket(2**64 - 1) == O.HIST_BINS - 1
    rng = np.random.default_rng(0)
    ts = np.unique(np.concatenate([rng.integers(0, 2**40, 5000, dtype=np.int64),
                                   np.arange(0, 5000)]))
    b = np.array([O.ttft_bucket(int(t)) for t in ts])
    assert np.all(np.diff(b) >= 0)                              # monotone
    # relative bucket width <= 1/8: all values in one bucket lie within [lo, lo * 9/8)
    for bk in np.unique(b):
        v = ts[b == bk]
        if v.min() >= 16:
            assert v.max() < v.min() * 9 / 8 + 1


def test_aggregate_matches_definition():
    tr = T.generate(np.array([T.make_replica(3, 0, 2000, 2.5, (0.5, 0.2, 0.3), 32768)]))
    r = O.simulate_trace(tr, 0, policy=O.TCM, kv_capacity=32768)
    hist, cnt = O.aggregate(tr, r)
    # independent vectorised restatement of SPEC.md:515-523 / PAPER.md:579
    a = tr.arrival_us.astype(np.int64)
    ttft = r.first_token_us.astype(np.int64) - a
    e2e = r.done_us.astype(np.int64) - a
    f = tr.footprint.astype(np.int64)
    iso = (tr.inline_us.astype(np.int64) + -(-f // 2048) * 5000 + 20 * f
           + (tr.out_tokens.astype(np.int64) - 1) * 5500)
    viol = e2e > 5 * iso
    cls = np.array([O.classify(int(m), int(x)) for m, x in zip(tr.modality, tr.footprint)])
    for g in range(4):
        sel = np.ones(len(a), bool) if g == 3 else cls == g
        assert cnt[g, 0] == sel.sum()
        assert cnt[g, 1] == ttft[sel].sum()
        assert cnt[g, 2] == e2e[sel].sum()
        assert cnt[g, 3] == viol[sel].sum()
        assert cnt[g, 4] == (e2e - 5 * iso)[sel & viol].sum()
        assert cnt[g, 5] == (e2e // tr.out_tokens.astype(np.int64))[sel].sum()
        assert hist[g].sum() == sel.sum()
    assert np.array_equal(hist[3], hist[0] + hist[1] + hist[2])   # overall = union of classes


def test_summary_examples():
    # SPEC.md:521 one record: arrival 0, first 0.013, completion 0.5575, out 100, slo 2.7875
    # -> no violation; SPEC.md:522 e2e 10 vs slo 4 -> violation, severity 6 s.
    tr = T.from_requests([[0, 400, 0, 100, 0]])
    r = O.simulate(tr.arrival_us, tr.footprint, tr.inline_us, tr.out_tokens, tr.modality)
    hist, cnt = O.aggregate(tr, r)
    assert cnt[3, 3] == 0 and cnt[3, 1] == 13000 and cnt[3, 2] == 557500
    assert cnt[3, 5] == 5575                                    # 0.005575 s/token
    fake = O.Result(np.zeros(1, np.uint32), np.array([13000], np.uint64),
                    np.array([10_000_000], np.uint64), None, {}, None, 0)
    tr2 = T.from_requests([[0, 400, 0, 100, 0]])
    m = O.model(slo_num=4_000_000, slo_den=557_500)            # slo = 4 s exactly for iso 0.5575 s
    hist, cnt = O.aggregate(tr2, fake, m=m)
    assert cnt[3, 3] == 1
    assert cnt[3, 4] == 10_000_000 * 557_500 - 4_000_000 * 557_500   # severity 6 s x den


def _check_golden(case, policy):
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "histogram.json")))[case]
    tr = T.from_requests(g["requests"])
    r = O.simulate(tr.arrival_us, tr.footprint, tr.inline_us, tr.out_tokens, tr.modality, policy=policy)
    assert r.status == 0
    hist, cnt = O.aggregate(tr, r)
    col = {"n": 0, "sum_ttft": 1, "sum_e2e": 2, "viol": 3, "severity": 4, "sum_norm": 5}
    for gname, exp in g["expect"].items():
        gi = {"M": 0, "C": 1, "T": 2, "All": 3}[gname]
        for k, v in exp.items():
            if k == "bins":
                nz = {str(b): int(hist[gi, b]) for b in np.nonzero(hist[gi])[0]}
                assert nz == v, (case, gname)
            elif k == "rate":
                assert cnt[gi, 3] / cnt[gi, 0] == v
            else:
                assert cnt[gi, col[k]] == v, (case, gname, k)


def test_hand_worked_histogram_isolated_requests():
    # tests/golden/histogram.json: SPEC.md:147-149 isolated requests, buckets derived by hand
    _check_golden("isolated_three", O.FCFS)
    _check_golden("isolated_three", O.TCM)


def test_hand_worked_violation_rates():
    # SPEC.md:523 overall rate 0.25 from class rates 0.5 (n=2) and 0.0 (n=2), via SURVEY H1 under FCFS
    _check_golden("violation_rates", O.FCFS)
