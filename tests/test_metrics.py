"""NEXT-2 metrics on the a6 counters: bucket bounds, quantiles, summaries and
the goodput search, pinned to SPEC's worked examples and to the oracle's bucket function."""
import numpy as np
import pytest

import oracle as O
import tracegen as T
from paper_2603_26498_b200 import metrics as M


def test_bucket_bounds_invert_the_oracle_bucket():
    lo, hi = M.bucket_bounds()
    rng = np.random.default_rng(1)
    for t in np.concatenate([np.arange(0, 300), rng.integers(0, 2**45, 3000)]):
        b = O.ttft_bucket(int(t))
        assert lo[b] <= t <= hi[b]
    # buckets tile the integers (checked where float64 is exact)
    assert np.all(lo[1:400] == hi[:399] + 1)


def test_quantile_bounds_contain_the_true_quantile():
    rng = np.random.default_rng(2)
    t = np.floor(10 ** rng.uniform(3, 9, 5000)).astype(np.int64)
    h = np.zeros(M.HIST_BINS, np.int64)
    for x in t:
        h[O.ttft_bucket(int(x))] += 1
    for q in (0.5, 0.9, 0.99):
        true = np.sort(t)[int(np.ceil(q * len(t))) - 1]   # nearest rank
        a, b = M.quantile_from_hist(h, q)
        assert a <= true <= b and b <= a * 1.125 + 1


def test_summary_spec_examples():
    # SPEC.md:521 one record: ttft 0.013, e2e 0.5575, out 100 -> norm 0.005575 s/token, no violation
    tr = T.from_requests([[0, 400, 0, 100, 0]])
    r = O.simulate(tr.arrival_us, tr.footprint, tr.inline_us, tr.out_tokens, tr.modality)
    h, c = O.aggregate(tr, r)
    s = M.summarize(c[None], h[None])[0]["all"]
    assert s["mean_ttft_s"] == pytest.approx(0.013) and s["mean_norm_latency_s_per_token"] == pytest.approx(0.005575)
    assert s["slo_violation_rate"] == 0.0 and s["mean_severity_s"] == 0.0
    assert s["p50_ttft_s"][0] <= 0.013 <= s["p50_ttft_s"][1]
    # SPEC.md:522 e2e 10 s vs slo 4 s -> severity 6 s (den = 557500 as in test_oracle_aggregate)
    cnt = np.zeros((1, 4, 6), np.int64)
    cnt[0, 3] = [1, 13000, 10_000_000, 1, (10_000_000 - 4_000_000) * 557_500, 100_000]
    assert M.summarize(cnt, slo_den=557_500)[0]["all"]["mean_severity_s"] == pytest.approx(6.0)
    # SPEC.md:523 two classes with violation rates 0.5 (n=2) and 0.0 (n=2) -> overall 0.25
    cnt = np.zeros((1, 4, 6), np.int64)
    cnt[0, 0, [0, 3]] = [2, 1]
    cnt[0, 1, [0, 3]] = [2, 0]
    cnt[0, 3, [0, 3]] = [4, 1]
    s = M.summarize(cnt)[0]
    assert s["M"]["slo_violation_rate"] == 0.5 and s["C"]["slo_violation_rate"] == 0.0
    assert s["all"]["slo_violation_rate"] == 0.25


def test_goodput_binary_search_spec_examples():
    # monotone attainment crossing the threshold at 3.0 -> 3.0 +- 0.05
    att = lambda r: 1.0 if r <= 3.0 + 1e-9 else 0.5
    g = M.binary_search_goodput(att, 0.5, 8.0, 0.9, 0.05)
    assert abs(g - 3.0) <= 0.05
    # oracle: linear scan at 0.05 resolution gives the same answer
    grid = [round(0.5 + 0.05 * k, 10) for k in range(151)]
    assert g == max(r for r in grid if att(r) >= 0.9)
    # threshold 1.0 with violations at every rate -> the low bound (R26)
    assert M.binary_search_goodput(lambda r: 0.95, 0.5, 8.0, 1.0, 0.05) == 0.5
    with pytest.raises(ValueError):
        M.binary_search_goodput(lambda r: 1.0, 0.5, 8.0, 0.9, 0.05)
    # goodput is non-increasing in the attainment threshold
    att2 = lambda r: max(0.0, 1.0 - 0.1 * r)
    gs = [M.binary_search_goodput(att2, 0.0, 9.0, th, 0.05) for th in (0.3, 0.5, 0.7, 0.9)]
    assert gs == sorted(gs, reverse=True)


def _oracle_counters(reqs, res):
    """[4, 3] fig:preemptions counters from oracle results, classes from the oracle's classifier."""
    import numpy as np
    import oracle as O
    c = np.zeros((4, 3), np.int64)
    for m, f, pc, pt in zip(reqs["modality"], reqs["footprint"], res.preempt_count, res.preempted_us):
        if pc:
            for g in (O.classify(m, f), 3):
                c[g] += (int(pc), int(pt), 1)
    return c


def test_preemption_summary_golden_p2():
    # tests/golden/preemption.json P2: FCFS preempts the text (motorcycle) once for 517,000 us,
    # TCM preempts the image (car) once for 792,000 us
    import oracle as O
    from paper_2603_26498_b200 import metrics as M
    reqs = dict(arrival_us=[0, 0], footprint=[150, 300], inline_us=[0, 0], out_tokens=[100, 150], modality=[1, 0])
    f = O.simulate_growth(**reqs, policy=O.FCFS, kv_capacity=460)
    t = O.simulate_growth(**reqs, policy=O.TCM, kv_capacity=460)
    sf = M.preemption_summary(_oracle_counters(reqs, f))
    st = M.preemption_summary(_oracle_counters(reqs, t)[None])      # [cells, 4, 3] sums over cells
    assert sf["M"] == {"preemptions": 1, "preempted_s": 0.517, "requests_preempted": 1}
    assert sf["C"]["preemptions"] == 0 and st["M"]["preemptions"] == 0
    assert st["C"] == {"preemptions": 1, "preempted_s": 0.792, "requests_preempted": 1}
    assert st["all"]["preemptions"] == 1 and st["T"]["requests_preempted"] == 0
