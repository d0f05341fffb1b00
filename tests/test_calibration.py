"""NEXT-4 pins: Workload Profiler -> Impact Estimator -> Request Classifier -> kernel thresholds
(SPEC.md:224-356 worked examples)."""
import numpy as np
import pytest

import oracle as O
import tracegen as T
from paper_2603_26498_b200 import calibration as K


def test_profile_isolated_examples():
    # text P=400 -> (0, 0, 0.013, 400) with noise 0
    tr = T.from_requests([[0, 400, 0, 1, 0], [0, 779, 170000, 1, 1]])
    s = K.profile(tr)
    assert s.prefill_s[0] == pytest.approx(0.013) and s.encode_s[0] == 0.0 and s.footprint[0] == 400
    # image stages (0.17 s inline) + prefill-only remainder 0.005 + 779 x 2e-5
    assert s.encode_s[1] == pytest.approx(0.17) and s.prefill_s[1] == pytest.approx(0.005 + 779 * 2e-5)


def test_ols_recovers_noiseless_line():
    x = np.arange(10, 5000, 37, dtype=np.float64)
    a, b = K.ols(x, 0.005 + 2e-5 * x)
    assert abs(a - 0.005) < 1e-9 and abs(b - 2e-5) < 1e-12
    with pytest.raises(ValueError):
        K.ols(np.full(5, 3.0), np.arange(5.0))                  # DegenerateDesign


def test_quantile_regression_pins():
    rng = np.random.default_rng(0)
    y = rng.normal(size=1000)
    a, b = K.quantile_regression(np.zeros(1000), y, 0.9)        # SPEC.md:252 constant predictor
    ys = np.sort(y)
    assert ys[899] - 1e-9 <= a <= ys[900] + 1e-9
    x = rng.uniform(0, 100, 1000)                               # SPEC.md:253 coverage
    y = 1.0 + 0.5 * x + rng.normal(size=1000)
    a, b = K.quantile_regression(x, y, 0.9)
    cov = np.mean(y - (a + b * x) <= 1e-12)
    assert 0.87 <= cov <= 0.93


def test_kmeans_three_blobs_and_degenerate():
    rng = np.random.default_rng(1)
    centers = np.array([[-2, -2], [0, 0], [2, 2]], dtype=np.float64)
    X = np.concatenate([c + 0.1 * rng.normal(size=(200, 2)) for c in centers[[2, 0, 1]]])
    C, _ = K.kmeans(X, 3, 10, 7)
    assert np.all(np.abs(C - centers) < 0.1)                   # labelled ascending: M, C, T
    with pytest.raises(ValueError):
        K.kmeans(np.ones((10, 2)), 3)                           # DegenerateClusters


@pytest.fixture(scope="module")
def default_model():
    tr = T.generate(np.array([T.make_replica(42, r, 300, 1.0, (1 / 3, 1 / 3, 1 / 3), 131072) for r in range(3)]))
    thr, est, model = K.calibrate(tr)
    return tr, thr, est, model


def test_default_profile_classification(default_model):
    tr, thr, est, model = default_model
    s = K.profile(tr)
    lat = np.array([est.latency(m, f) for m, f in zip(s.modality, s.footprint)]).ravel()
    cls = K.classify_smart(model, lat, s.footprint)
    assert np.mean(cls[s.modality == K.TEXT] == 0) >= 0.95
    assert K.classify_smart(model, est.latency(K.TEXT, 9000), 9000)[0] == 1
    assert K.classify_smart(model, est.latency(K.VIDEO, 800), 800)[0] == 1
    assert K.classify_smart(model, est.latency(K.IMAGE, 779), 779)[0] == 1


def test_thresholds_reproduce_the_classifier(default_model):
    tr, thr, est, model = default_model
    m = O.model(thresholds=thr)
    rng = np.random.default_rng(5)
    for mod in (0, 1, 2):
        f = rng.integers(1, 131072, 400)
        want = K.classify_smart(model, est.latency(mod, f), f)
        got = [O.classify(mod, int(x), m) for x in f]
        assert list(want) == got
