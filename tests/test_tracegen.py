"""Synthetic workload generator checks (SPEC.md:192-216 properties; SURVEY.md 8(d) recipe)."""
import numpy as np
import pytest
from scipy import stats

import tracegen as T


def gen(n, rate=2.0, mix=(0.6, 0.25, 0.15), kv=131072, seed=1, replica=0, flags=0):
    return T.generate(np.array([T.make_replica(seed, replica, n, rate, mix, kv, flags)]))


def test_deterministic_and_replica_distinct():
    a, b = gen(3000), gen(3000)
    for f in ("arrival_us", "footprint", "inline_us", "out_tokens", "modality"):
        assert np.array_equal(getattr(a, f), getattr(b, f))          # SPEC.md:199 bit-identical
    c = gen(3000, replica=1)
    assert not np.array_equal(a.footprint, c.footprint)


def test_poisson_arrivals():
    t = gen(20000, rate=2.0)
    gaps = np.diff(t.arrival_us.astype(np.int64)) / 1e6
    assert t.arrival_us[0] == 0 and np.all(gaps >= 0)
    assert abs(gaps.mean() - 0.5) < 0.025                            # SPEC.md:215 (+-5 %)
    # exponential gaps (SPEC.md:197 chi-square/KS at alpha = 0.01), floor to 1 us is negligible
    assert stats.kstest(gaps, "expon", args=(0, 0.5)).pvalue > 0.01


def test_mix_fractions():
    t = gen(2000, mix=(0.6, 0.25, 0.15))
    frac = np.bincount(t.modality, minlength=3) / 2000
    assert np.all(np.abs(frac - [0.6, 0.25, 0.15]) < 0.03)
    t = gen(2000, mix=(1.0, 0.0, 0.0))
    assert np.all(t.modality == 0) and np.all(t.inline_us == 0)      # SPEC.md:197 text-only


def test_ranges_and_shapes():
    t = gen(40000, mix=(0.34, 0.33, 0.33), kv=131072)
    m = t.modality
    ft, fi, fv = t.footprint[m == 0], t.footprint[m == 1], t.footprint[m == 2]
    assert ft.min() >= 10 and ft.max() <= 10000                      # PAPER.md:148 text 10..1e4
    assert abs(np.median(ft) - 200) < 15
    assert fi.min() >= 1 + 665 and fi.max() <= 512 + 793             # ~10^2..10^3
    assert fv.max() <= 131072 and fv.min() >= 1 + 196 * 8            # videos >> images
    assert np.all(t.out_tokens >= 1) and np.all(t.out_tokens <= 2048)
    assert abs(np.median(t.out_tokens) - 128) < 8
    ii = t.inline_us[m == 1]
    assert ii.min() >= 140000 and ii.max() < 290000                  # 0.13 + 0.04*MP s, MP in [0.25, 4)
    frames = (fv - 1) // 196
    iv = t.inline_us[m == 2]
    assert np.all(iv >= 300000 + 16000 * 8) and np.all(iv <= 300000 + 16000 * 512)


@pytest.mark.parametrize("kv", [16384, 32768])
def test_video_clamped_to_kv(kv):
    t = gen(5000, mix=(0.0, 0.0, 1.0), kv=kv)
    assert np.all(t.footprint <= kv)                                 # R18 generator clamps
    assert t.footprint.max() > kv - 196 - 512


def test_all_at_zero_flag():
    t = gen(1000, flags=T.FLAG_ALL_AT_ZERO)
    assert np.all(t.arrival_us == 0)


def test_multi_replica_csr():
    reps = np.array([T.make_replica(7, r, 100 + r, 1.0) for r in range(5)])
    t = T.generate(reps)
    assert t.offset.tolist() == [0, 100, 201, 303, 406, 510]
    one = gen(103, rate=1.0, mix=(0.7, 0.25, 0.05), seed=7, replica=3)
    s = t.replica(3)
    assert np.array_equal(s.footprint, one.footprint) and np.array_equal(s.arrival_us, one.arrival_us)
