"""Paper metrics from the a6 aggregation.

Everything here is host arithmetic on the int64 counters and histograms that `tcm_stats`
produces on the device (and that the NCCL all-reduce sums across GPUs):

  cnt[cell][group][k], group in (M, C, T, all), k:
     0 n, 1 sum TTFT (us), 2 sum E2E (us), 3 SLO violations, 4 sum (e2e*den - num*iso) over
     violators, 5 sum floor(e2e / out) (us per output token)
  hist[cell][group][496]: TTFT log buckets

* mean TTFT, mean normalized latency ("seconds/token"), SLO violation rate and
  mean severity over violators (R19), P-quantiles of TTFT from the histogram
  (bucket bounds, <= 1/8 relative width);
* goodput: the largest request rate whose SLO attainment is >= a threshold (PAPER.md:768
  `fig:slo-ablation`), found by SPEC's binary search at 0.05 req/s resolution.
  Every probe rate is simulated at once as one batch of replicas (one tcm_run).
"""
from __future__ import annotations

import numpy as np

GROUPS = ("M", "C", "T", "all")
HIST_BINS = 496


def bucket_bounds() -> tuple[np.ndarray, np.ndarray]:
    """[lo, hi] microsecond range of each of the 496 TTFT buckets."""
    lo = np.zeros(HIST_BINS, dtype=np.float64)
    hi = np.zeros(HIST_BINS, dtype=np.float64)
    for b in range(16):
        lo[b] = hi[b] = b
    for b in range(16, HIST_BINS):
        e = 4 + (b - 16) // 8
        sub = (b - 16) % 8
        lo[b] = (8 + sub) * 2.0 ** (e - 3)
        hi[b] = (9 + sub) * 2.0 ** (e - 3) - 1
    return lo, hi


def quantile_from_hist(h: np.ndarray, q: float) -> tuple[float, float]:
    """Bounds [lo, hi] (us) on the q-quantile of TTFT given one histogram row (nearest-rank)."""
    n = int(h.sum())
    if n == 0:
        return float("nan"), float("nan")
    rank = max(1, int(np.ceil(q * n)))
    b = int(np.searchsorted(np.cumsum(h), rank))
    lo, hi = bucket_bounds()
    return float(lo[b]), float(hi[b])


def summarize(cnt: np.ndarray, hist: np.ndarray | None = None, slo_den: int = 1) -> list[dict]:
    """Per (cell, group) summary."""
    cnt = np.asarray(cnt, dtype=np.int64)
    out = []
    for cell in range(cnt.shape[0]):
        row = {}
        for g, name in enumerate(GROUPS):
            n, st, se, nv, sev, snl = (int(x) for x in cnt[cell, g])
            d = {"n": n}
            if n:
                d["mean_ttft_s"] = st / n / 1e6
                d["mean_e2e_s"] = se / n / 1e6
                d["mean_norm_latency_s_per_token"] = snl / n / 1e6
                d["slo_violation_rate"] = nv / n
                d["slo_attainment"] = 1.0 - nv / n
                d["mean_severity_s"] = (sev / slo_den / nv / 1e6) if nv else 0.0
                if hist is not None:
                    d["p50_ttft_s"] = [x / 1e6 for x in quantile_from_hist(np.asarray(hist[cell, g]), 0.50)]
                    d["p90_ttft_s"] = [x / 1e6 for x in quantile_from_hist(np.asarray(hist[cell, g]), 0.90)]
            row[name] = d
        out.append(row)
    return out


def binary_search_goodput(attainment_at, lo: float, hi: float, threshold: float = 0.9,
                          res: float = 0.05) -> float:
    """the largest probed rate with attainment >= threshold, to `res` resolution.
    attainment_at(rate) -> float; requires attainment(lo) >= threshold > attainment(hi)
    (BracketInvalid otherwise).  Rates are probed on the grid lo + k*res."""
    steps = int(round((hi - lo) / res))
    # R26: SPEC.md:532 returns the low bound when even it misses the threshold ("degenerate"),
    # although SPEC.md:528 asks for a bracket; only an unreached threshold at hi is an error.
    if not attainment_at(lo) >= threshold:
        return lo
    if attainment_at(hi) >= threshold:
        raise ValueError("BracketInvalid: the threshold is still met at the high bound")
    a, b = 0, steps                     # invariant: ok(a), not ok(b)
    while b - a > 1:
        mid = (a + b) // 2
        if attainment_at(lo + mid * res) >= threshold:
            a = mid
        else:
            b = mid
    return round(lo + a * res, 10)


def goodput_sweep(lo: float, hi: float, res: float, seeds: int, n_requests: int, mix, kv=131072,
                  policy=1, alpha=1.0, budget=2048, seed=777):
    """Replicas for every probe rate on the grid (cell k = rate lo + k*res, `seeds` replicas each);
    rate -> seed derivation is fixed ("fixed seed derivation rate->seed")."""
    import tracegen as T

    from . import tcm
    from .workloads import Sweep
    rates = [round(lo + k * res, 10) for k in range(int(round((hi - lo) / res)) + 1)]
    nc = len(rates)
    gen = np.zeros(nc * seeds, dtype=T.TG_REPLICA_DTYPE)
    params = tcm.make_params(nc * seeds, policy=policy, chunk_budget=budget, kv_capacity=kv, aging_alpha=alpha)
    for c, rate in enumerate(rates):
        for s in range(seeds):
            j = c * seeds + s
            gen[j] = T.make_replica(seed + int(round(rate * 1000)) * 1_000_003, s, n_requests, rate, mix, kv)
            params[j]["cell_id"] = c
    cells = [dict(rate=r, mix=mix, kv=kv, policy=policy, alpha=alpha, budget=budget) for r in rates]
    return Sweep("goodput", gen, params, nc, cells), rates


def goodput(lo: float, hi: float, res: float = 0.05, threshold: float = 0.9, seeds: int = 64,
            n_requests: int = 1000, mix=(0.60, 0.25, 0.15), kv=131072, policy=1, alpha=1.0,
            budget=2048, group: int = 3, cfg=None, device="cuda") -> dict:
    """Goodput on the GPU: one batched simulation over every grid rate, then SPEC's binary search
    on the measured attainment of `group` (0 M, 1 C, 2 T, 3 all)."""
    import torch

    from . import tcm
    sw, rates = goodput_sweep(lo, hi, res, seeds, n_requests, mix, kv, policy, alpha, budget)
    cfg = cfg or tcm.config(n_cells=sw.n_cells)
    cfg.n_cells = sw.n_cells
    trace = tcm.generate_device(sw.gen, device=device)
    trace["params"] = tcm.to_device_params(sw.params, device)
    sim = tcm.Simulation(cfg)
    sim.load(trace, None)
    sim.run()
    hist, cnt, _ = sim.aggregate(device=device)
    cnt = cnt.cpu().numpy()
    sim.close()
    att = {r: 1.0 - cnt[c, group, 3] / max(1, cnt[c, group, 0]) for c, r in enumerate(rates)}
    rate = binary_search_goodput(lambda r: att[round(r, 10)], lo, hi, threshold, res)
    return {"goodput_rps": rate, "attainment": att, "counters": cnt, "rates": rates}


def preemption_summary(counters) -> dict:
    """fig:preemptions: per class (M, C, T, all) the number of
    preemptions, the time spent preempted (s) and the number of requests preempted at least once.
    `counters` is the device's int64 [4, 3] (or [cells, 4, 3], summed over cells) from
    Simulation.preemption_stats() -- classified on the device by the engine's own a1 classifier."""
    c = np.asarray(counters, dtype=np.int64)
    if c.ndim == 3:
        c = c.sum(axis=0)
    return {name: {"preemptions": int(c[g, 0]), "preempted_s": float(c[g, 1]) / 1e6,
                   "requests_preempted": int(c[g, 2])} for g, name in enumerate(GROUPS)}
