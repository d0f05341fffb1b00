"""Pins for the oracle's K1 priority key.

The oracle's K1 is a specified-arithmetic evaluation of the paper's formula
    Priority_c = StaticPriority_c + (1 - e^{-k_c * waiting_time^{p_c}})
with waiting_time in seconds (R1).  Here it is pinned against an independent
high-precision evaluation (mpmath, 50 digits) of the paper's formula, against the
paper's constants, against exact-microsecond crossovers derived in closed form, and
against Lemma L1 (monotone in the waiting time within a class).
"""
import math
import random

import mpmath as mp
import pytest

import oracle as O

mp.mp.dps = 50
S, K, P = O.PAPER_S, O.PAPER_K, O.PAPER_P


def paper_priority(c, w_us, alpha=1.0):
    """PAPER.md:457 with PAPER.md:580 constants, w in seconds (R1), 50 digits."""
    if w_us == 0 or alpha == 0:
        return mp.mpf(S[c])
    w = mp.mpf(int(w_us)) / 10**6
    return mp.mpf(S[c]) + (1 - mp.e ** (-mp.mpf(alpha) * mp.mpf(K[c]) * w ** mp.mpf(P[c])))


# Values quoted in SURVEY.md 8(c) "Priority formula" row (mpmath, 50 digits), correcting
# SPEC.md:381-382, 407 (Appendix B errata).
GOLDEN = [
    (0, 2_000_000, 0.5320292880),      # M @ 2 s    (SPEC.md:381 prints 0.53202)
    (2, 100_000_000, 0.1120741036),    # T @ 100 s  (SPEC.md:382 prints 0.11212: erratum)
    (0, 500_000, 0.1044096661),        # M @ 0.5 s  (SPEC.md:407 prints 0.10880: erratum)
    (2, 10_000_000, 0.0093975054),     # T @ 10 s
]


@pytest.mark.parametrize("c,w,val", GOLDEN)
def test_paper_values(c, w, val):
    got = O.priority(c, w)
    assert abs(got - val) < 1e-10
    assert abs(got - float(paper_priority(c, w))) < 1e-14


def test_fresh_and_saturated():
    # waiting_time 0 -> age term vanishes ("Motorcycle, waiting_time 0 -> 0.1")
    for c in range(3):
        assert O.priority(c, 0) == S[c]
    # alpha = 0 (static priority) -> constant S_c
    for c in range(3):
        assert O.priority(c, 123456789, alpha=0.0) == S[c]
    # bounded above by S_c + 1 and reaching it exactly once e^{-x} underflows
    assert O.priority(0, 10**9) == S[0] + 1.0
    assert O.priority(1, 10**9) == S[1] + 1.0
    assert O.priority(2, 10**13) == 1.0
    # a fresh truck has P = 0 and gets the epsilon clamp (R3)
    assert O.key_bits(O.priority(2, 0)) == O.key_bits(1e-12)


def test_random_against_mpmath():
    rng = random.Random(1234)
    alphas = [0.0] + [2.0**e for e in range(-7, 8)]
    worst = 0.0
    for _ in range(3000):
        c = rng.randrange(3)
        a = rng.choice(alphas)
        w = int(10 ** rng.uniform(0, 10.5))
        got = O.priority(c, w, alpha=a)
        want = paper_priority(c, w, alpha=a)
        worst = max(worst, abs(got - float(want)))
    # Error budget: y = p*L + C carries <= ~1e-14 relative error
    # into x = e^y; |d e^{-x}| <= x e^{-x} * 1e-14 <= 3.7e-15; plus 2 roundings of P <= 2.1.
    assert worst < 5e-15, worst


def test_ln_exp_accuracy_every_table_interval():
    rng = random.Random(7)
    # LN: 16 table intervals x several binades, relative error vs mpmath
    for j in range(16):
        for e in (-30, -5, 0, 1, 20, 40):
            for _ in range(20):
                m = 1 + (j + rng.random()) / 16
                v = math.ldexp(m, e)
                got = O.ln(v)
                want = mp.log(mp.mpf(v))
                assert abs(got - float(want)) <= 4e-16 * max(1.0, abs(float(want))) + 1e-300
    # EXP across its domain, relative error (EXP.1 cut-offs are part of the spec)
    for _ in range(4000):
        y = rng.uniform(-700, 700)
        got = O.exp(y)
        want = mp.e ** mp.mpf(y)
        # T[j] (0.5 ulp) + Taylor-6 truncation on |r| <= ln2/32 (2 ulp) + 2 roundings
        assert abs(got - float(want)) <= 1e-15 * float(want)
    assert O.exp(-800.0) == 0.0 and O.exp(701.0) == math.inf and O.exp(0.0) == 1.0


def _crossover(ca, cb_fresh):
    """Waiting time (us, exact real) at which class ca's priority equals fresh class cb's S."""
    target = mp.mpf(S[cb_fresh]) - mp.mpf(S[ca])
    # S_a + 1 - exp(-k w^p) = S_b  ->  w = (-ln(1 - (S_b - S_a)) / k)^(1/p)
    w_s = (-mp.log(1 - target) / mp.mpf(K[ca])) ** (1 / mp.mpf(P[ca]))
    return w_s * 10**6


# SURVEY.md 8(c) "Cross-class order": exact-us crossovers (loses at floor, wins at ceil).
CROSS = [(2, 0, 89_614_595), (2, 1, 46_578_039), (1, 0, 3_112_975)]


@pytest.mark.parametrize("ca,cb,floor_us", CROSS)
def test_cross_class_crossovers(ca, cb, floor_us):
    w = _crossover(ca, cb)
    assert int(mp.floor(w)) == floor_us
    fresh = O.key_bits(O.priority(cb, 0))
    assert O.key_bits(O.priority(ca, floor_us)) < fresh
    assert O.key_bits(O.priority(ca, floor_us + 1)) > fresh


def test_motorcycle_beats_any_truck_threshold():
    # P_M(w) >= 1 = sup P_T  <=>  w >= (ln 10 / 0.05)^(1/3.5) s  (= 2.98685 s)
    w = (mp.log(10) / mp.mpf(K[0])) ** (1 / mp.mpf(P[0])) * 10**6
    assert abs(float(w) / 1e6 - 2.98685) < 1e-5
    truck_max = O.key_bits(O.priority(2, 10**14))
    assert O.key_bits(O.priority(0, int(mp.ceil(w)) + 1)) > truck_max
    assert O.key_bits(O.priority(0, int(mp.floor(w)) - 1)) < truck_max


def test_key_order_equals_score_order():
    # Score = -log(Priority): lower score first == higher key first (R3).
    rng = random.Random(3)
    for _ in range(2000):
        a, b = rng.uniform(0, 2.1), rng.uniform(0, 2.1)
        sa, sb = -math.log(max(a, 1e-12)), -math.log(max(b, 1e-12))
        if sa != sb:
            assert (O.key_bits(a) > O.key_bits(b)) == (sa < sb)
    assert abs(-math.log(1e-12) - 27.6310211) < 1e-7     # SPEC.md:387 score(eps)
    assert abs(-math.log(0.1) - 2.3025851) < 1e-7


@pytest.mark.parametrize("c,lo,hi", [(0, 0, 8_000_000), (1, 0, 3_000_000), (2, 0, 3_000_000),
                                     (1, 40_000_000, 46_000_000), (2, 89_000_000, 92_000_000)])
def test_monotone_in_waiting_time(c, lo, hi):
    # Lemma L1: key non-decreasing at every microsecond (full-range audit runs on the GPU)
    assert O.audit_monotone(c, lo, hi) is None


@pytest.mark.parametrize("alpha", [2.0**-7, 0.5, 4.0, 128.0])
def test_monotone_alpha_grid(alpha):
    for c in range(3):
        assert O.audit_monotone(c, 0, 400_000, alpha=alpha) is None


# ---------------------------------------------------------------------------------------------
# 10^6-sample pins (SURVEY.md 8(c) "K1" row) against an independent extended-precision evaluation:
# numpy's long double (x87 80-bit, 64-bit significand: 11 bits more than binary64) through libm's
# logl / expl / powl.  Stage by stage, then the whole key against the paper's formula.
# (A final-P bound of 4 ulp is not attainable by ANY binary64 evaluation through ln(w in us):
# 0.5 ulp of L ~ 20 is 1.8e-15 absolute, times p = 3.5 -- see DESIGN.md reading R33.)
import numpy as np

_LD = np.longdouble
_N6 = 1_000_000


def _ulp(x):
    return np.spacing(np.abs(np.asarray(x, dtype=np.float64))).astype(_LD)


def test_ln_million_samples_within_1_5_ulp():
    L = O.lib()
    rng = np.random.default_rng(61)
    v = np.ldexp(1 + rng.random(_N6), rng.integers(-60, 61, _N6))
    got = np.fromiter((L.orc_ln(float(x)) for x in v), np.float64, _N6).astype(_LD)
    ref = np.log(v.astype(_LD))
    # absolute error in ulps of max(|ln v|, 1): LN.5's table + series sum is absolute-accurate
    err = np.abs(got - ref) / _ulp(np.maximum(np.abs(ref), 1))
    assert float(err.max()) <= 1.5, float(err.max())


def test_exp_million_samples_within_6_ulp():
    L = O.lib()
    rng = np.random.default_rng(62)
    y = rng.uniform(-740.0, 700.0, _N6)
    got = np.fromiter((L.orc_exp(float(x)) for x in y), np.float64, _N6)
    ref = np.exp(y.astype(_LD))
    ok = got >= 2.0**-1022                        # EXP.7 flushes the subnormal range by spec
    assert np.all(ref[~ok] < _LD(2.0**-1021))
    err = np.abs(got[ok].astype(_LD) - ref[ok]) / _ulp(got[ok])
    # T[j] 0.5 ulp + degree-6 Taylor truncation r^7/7! <= 2 ulp on |r| <= ln2/32 + 3 roundings
    assert float(err.max()) <= 6.0, float(err.max())
    assert float(np.median(err.astype(np.float64))) <= 1.0


def test_priority_million_samples_vs_paper_formula():
    # PAPER.md:457 with PAPER.md:580 constants, w in seconds (R1), alpha on the sweep grid (R14):
    # P_ref = S + (1 - exp(-alpha k (w/1e6)^p)) in long double.  Bound: every stage of K1 within
    # 4 ulp of its exact result, propagated forward (dP = e x dy): dL, dC -> dy -> dx/x -> de.
    L = O.lib()
    rng = np.random.default_rng(63)
    alphas = np.array([0.0] + [2.0**e for e in range(-7, 8)])
    c = rng.integers(0, 3, _N6)
    a = alphas[rng.integers(0, len(alphas), _N6)]
    w = np.floor(10 ** rng.uniform(0, 10.5, _N6)).astype(np.uint64)
    Sv, Kv, Pv = np.array(S)[c], np.array(K)[c], np.array(P)[c]
    consts = {}
    got = np.empty(_N6)
    for i in range(_N6):
        key = (int(c[i]), float(a[i]))
        if key not in consts:
            consts[key] = O.k1_const(a[i], Kv[i], Pv[i])
        C, z = consts[key]
        got[i] = L.orc_priority(Sv[i], Pv[i], C, z, int(w[i]))
    wl = w.astype(_LD) / _LD(10**6)
    x = (a.astype(_LD) * Kv.astype(_LD)) * wl ** Pv.astype(_LD)
    e = np.exp(-x)
    ref = Sv.astype(_LD) + (_LD(1) - e)
    ref = np.where((w == 0) | (a == 0), Sv.astype(_LD), ref)
    lnw = np.log(np.maximum(w, 1).astype(_LD))
    yv = np.where(x > 0, np.log(np.where(x > 0, x, _LD(1))), _LD(0))
    dy = 4 * (Pv * _ulp(np.maximum(lnw, 1)) + _ulp(np.maximum(np.abs(yv), 1))
              + Pv * _ulp(np.log(1e6)) + _ulp(np.maximum(np.abs(np.log(np.maximum(a * Kv, 1e-300))), 1)))
    de = e * x * (dy + 4 * _LD(2.0**-52)) + 4 * _ulp(e)
    bound = de + 2 * _ulp(ref)
    err = np.abs(got.astype(_LD) - ref)
    assert np.all(err <= bound), float(np.max(err / bound))
    assert float(err.max()) < 5e-15                    # the absolute budget of the 3,000-sample pin
