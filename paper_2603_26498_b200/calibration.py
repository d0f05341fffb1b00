"""NEXT-4: smart-classifier calibration (offline, host) -> the per-modality footprint thresholds
that the scheduling kernels classify with (reading R13).

PAPER.md:337-347 (Workload Profiler), 364 (Impact Estimator: linear regression for text, quantile
regression at tau = 0.9 for image/video), 395 (Request Classifier: clustering on estimated prefill
latency and KV footprint).  SPEC.md:224-356 gives the operational form followed here:

  profile()        isolated execution of every request of a sample trace under the integer-us
                   cost model (R9): (modality, footprint, preprocess+encode, prefill) per request,
                   optional multiplicative log-normal noise (SPEC.md:118 noise_cv);
  fit_estimators() text: ordinary least squares of prefill time on footprint; image/video: affine
                   quantile regression at tau = 0.9 of TTFT (encode + prefill) on footprint, solved
                   exactly as a linear programme (scipy HiGHS);
  train_clusters() k-means, k = 3, 10 seeded restarts, on standardised (log10 estimated latency,
                   log10 footprint); centroids labelled by ascending coordinate sum -> M, C, T;
  classify_smart() nearest centroid, ties toward the larger class;
  thresholds()     the classifier as (thr_mc, thr_ct) per modality: with the estimators the class
                   is a function of the footprint alone, so it is evaluated at every footprint and
                   the two class boundaries are read off (monotonicity is checked).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TEXT, IMAGE, VIDEO = 0, 1, 2


@dataclass
class Samples:
    modality: np.ndarray     # u8
    footprint: np.ndarray    # tokens
    encode_s: np.ndarray     # preprocess + encode (s)
    prefill_s: np.ndarray    # prefill (s), isolated, chunked at B


def profile(trace, chunk_budget=2048, c0_us=5000, cp_us=20, noise_cv=0.0, seed=0) -> Samples:
    """Isolated execution of every request: prefill = ceil(f/B) c0 + cp f."""
    f = trace.footprint.astype(np.float64)
    pre = (np.ceil(f / chunk_budget) * c0_us + cp_us * f) / 1e6
    enc = trace.inline_us.astype(np.float64) / 1e6
    if noise_cv > 0:
        rng = np.random.default_rng(seed)
        s = np.sqrt(np.log1p(noise_cv ** 2))
        pre = pre * rng.lognormal(-s * s / 2, s, len(pre))
        enc = enc * rng.lognormal(-s * s / 2, s, len(enc))
    return Samples(trace.modality.copy(), f, enc, pre)


def ols(x: np.ndarray, y: np.ndarray) -> tuple[float, float]:
    """Ordinary least squares y ~ a + b x (PAPER.md:364 'lightweight linear regression')."""
    if len(x) < 2 or np.all(x == x[0]):
        raise ValueError("DegenerateDesign" if len(x) >= 2 else "InsufficientData")
    A = np.stack([np.ones_like(x), x], 1)
    (a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
    return float(a), float(b)


def quantile_regression(x: np.ndarray, y: np.ndarray, tau: float = 0.9) -> tuple[float, float]:
    """Affine quantile regression minimising the pinball loss at tau, exactly as the
    LP  min sum tau u+ + (1 - tau) u-  s.t.  a + b x + u+ - u- = y,  u+- >= 0."""
    from scipy.optimize import linprog
    n = len(x)
    if n < 10:
        raise ValueError("InsufficientData")
    xs = x / max(1.0, float(np.abs(x).max()))             # conditioning; slope rescaled below
    c = np.concatenate([[0.0, 0.0], np.full(n, tau), np.full(n, 1.0 - tau)])
    A = np.hstack([np.ones((n, 1)), xs[:, None], np.eye(n), -np.eye(n)])
    bounds = [(None, None), (None, None)] + [(0, None)] * (2 * n)
    r = linprog(c, A_eq=A, b_eq=y, bounds=bounds, method="highs")
    if not r.success:
        raise RuntimeError(r.message)
    a, b = r.x[0], r.x[1] / max(1.0, float(np.abs(x).max()))
    return float(a), float(b)


@dataclass
class Estimators:
    coef: dict   # modality -> (a, b): estimated latency (s) = a + b * footprint, clamped at 0

    def latency(self, modality, footprint):
        a, b = self.coef[int(modality)]
        return np.maximum(a + b * np.asarray(footprint, dtype=np.float64), 0.0)


def fit_estimators(s: Samples, tau: float = 0.9) -> Estimators:
    """Text: OLS of prefill time on footprint; image/video: tau-quantile regression of TTFT
    (encode + prefill) on footprint -- the latency feature must include encode time to separate
    images from equally long texts (SURVEY.md R13 note)."""
    coef = {}
    t = s.modality == TEXT
    coef[TEXT] = ols(s.footprint[t], s.prefill_s[t])
    for m in (IMAGE, VIDEO):
        k = s.modality == m
        coef[m] = quantile_regression(s.footprint[k], s.encode_s[k] + s.prefill_s[k], tau)
    return Estimators(coef)


@dataclass
class ClusterModel:
    centroids: np.ndarray    # [3, 2] standardised, rows ordered M, C, T
    mean: np.ndarray
    std: np.ndarray


def _features(lat, fp):
    return np.stack([np.log10(np.maximum(lat, 1e-9)), np.log10(np.maximum(fp, 1.0))], 1)


def kmeans(X: np.ndarray, k: int = 3, restarts: int = 10, seed: int = 0, iters: int = 100):
    """Lloyd's algorithm, k-means++ seeding, best of `restarts`."""
    if len(np.unique(X, axis=0)) < k:
        raise ValueError("DegenerateClusters")
    rng = np.random.default_rng(seed)
    best, best_obj = None, np.inf
    for _ in range(restarts):
        C = [X[rng.integers(len(X))]]
        for _ in range(1, k):
            d = np.min(((X[:, None, :] - np.array(C)[None]) ** 2).sum(-1), 1)
            C.append(X[rng.choice(len(X), p=d / d.sum())])
        C = np.array(C)
        prev = np.inf
        for _ in range(iters):
            lab = np.argmin(((X[:, None, :] - C[None]) ** 2).sum(-1), 1)
            C = np.array([X[lab == j].mean(0) if np.any(lab == j) else C[j] for j in range(k)])
            obj = ((X - C[lab]) ** 2).sum()
            if obj >= prev - 1e-12:
                break
            prev = obj
        if obj < best_obj:
            best, best_obj = C, obj
    return best[np.argsort(best.sum(1))], best_obj


def train_clusters(s: Samples, est: Estimators, seed: int = 0) -> ClusterModel:
    lat = np.array([est.latency(m, f) for m, f in zip(s.modality, s.footprint)]).ravel()
    X = _features(lat, s.footprint)
    mean, std = X.mean(0), X.std(0)
    std[std == 0] = 1.0
    C, _ = kmeans((X - mean) / std, 3, 10, seed)
    return ClusterModel(C, mean, std)


def classify_smart(model: ClusterModel, latency, footprint) -> np.ndarray:
    """Nearest centroid; ties toward the larger class."""
    Z = (_features(np.asarray(latency, np.float64).ravel(), np.asarray(footprint, np.float64).ravel())
         - model.mean) / model.std
    d = ((Z[:, None, :] - model.centroids[None]) ** 2).sum(-1)
    # argmin with ties resolved to the largest index: reverse, argmin, map back
    return (2 - np.argmin(d[:, ::-1], 1)).astype(np.int64)


def thresholds(model: ClusterModel, est: Estimators, max_footprint: int = 1 << 18):
    """(thr_mc, thr_ct) per modality for the kernels' classify() (R13): class(f) is evaluated at
    every footprint 1..max_footprint; it must be non-decreasing in f."""
    INF = 0xFFFFFFFF
    f = np.arange(1, max_footprint + 1, dtype=np.float64)
    out = []
    for m in (TEXT, IMAGE, VIDEO):
        cls = classify_smart(model, est.latency(m, f), f)
        if np.any(np.diff(cls) < 0):
            raise ValueError(f"class is not monotone in the footprint for modality {m}")
        mc = int(f[np.argmax(cls >= 1)]) if np.any(cls >= 1) else INF
        ct = int(f[np.argmax(cls >= 2)]) if np.any(cls >= 2) else INF
        out.append((mc if cls[0] == 0 else 0, ct))
    return tuple(out)


def calibrate(trace, chunk_budget=2048, noise_cv=0.1, seed=0):
    """Profile -> estimators -> clusters -> thresholds, end to end."""
    s = profile(trace, chunk_budget, noise_cv=noise_cv, seed=seed)
    est = fit_estimators(s)
    model = train_clusters(s, est, seed)
    return thresholds(model, est), est, model
