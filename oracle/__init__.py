"""TEST INFRASTRUCTURE ONLY -- the plain CPU oracle for TCM-Serve's scheduling step.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product (paper_2603_26498_b200) never imports it and shares
no code with it.  The arithmetic lives in tcm_oracle.c (plain C, gcc -O2
-ffp-contract=off); this file only marshals numpy arrays through ctypes.

Parity status: every function is pinned by tests/test_oracle_*.py
(simulate_growth, the NEXT-1 loop, by tests/test_oracle_next1.py)
except full random traces, whose schedules have no independent closed form ("parity
unpinned" beyond the invariants, reductions, hand-worked schedules and brute force).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

FCFS, TCM, EDF, NAIVE_AGING = 0, 1, 2, 3
HIST_BINS, GROUPS, NCNT = 496, 4, 6

# Paper constants and SPEC cost model in integer us (R9).
PAPER_S = (0.1, 0.05, 0.0)
PAPER_K = (0.05, 0.003, 0.00075)
PAPER_P = (3.5, 2.5, 1.1)
INF = 0xFFFFFFFF
SMART_THR = ((4096, INF), (0, INF), (0, 8192))   # R13 smart default: (thr_mc, thr_ct) per modality
NAIVE_THR = ((INF, INF), (0, INF), (0, 0))       # PAPER.md:393 naive text->M, image->C, video->T


class OrcModel(ctypes.Structure):
    _fields_ = [
        ("c0_us", ctypes.c_uint64), ("cp_us", ctypes.c_uint64), ("cd_us", ctypes.c_uint64),
        ("S", ctypes.c_double * 3), ("k", ctypes.c_double * 3), ("p", ctypes.c_double * 3),
        ("thr_mc", ctypes.c_uint32 * 3), ("thr_ct", ctypes.c_uint32 * 3),
        ("slo_num", ctypes.c_uint32), ("slo_den", ctypes.c_uint32),
    ]


class OrcReplica(ctypes.Structure):
    _fields_ = [
        ("policy", ctypes.c_uint32), ("chunk_budget", ctypes.c_uint32),
        ("kv_capacity", ctypes.c_uint64), ("alpha", ctypes.c_double),
        ("admit_skip", ctypes.c_uint32), ("pad", ctypes.c_uint32),
    ]


class OrcCounters(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "iterations", "decisions", "sum_pending", "max_pending", "admitted", "idle_jumps",
        "final_clock")]


ITER_DTYPE = np.dtype([
    ("clock_start", "<u8"), ("clock_end", "<u8"), ("kv_free_start", "<u8"),
    ("kv_free_admit", "<u8"), ("n_pending", "<u4"), ("n_dec", "<u4"), ("budget", "<u4"),
    ("tokens", "<u4"), ("n_admitted", "<u4"), ("n_first_tokens", "<u4"),
    ("n_partial_after", "<u4"), ("pad", "<u4"),
])


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "tcm_oracle.c")
    hdr = os.path.join(_HERE, "tcm_oracle.h")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(hdr)
    ):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-Wall",
                               "-Wextra", "-o", _SO, src, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        d, u64, i = ctypes.c_double, ctypes.c_uint64, ctypes.c_int
        L.orc_ln.restype = d; L.orc_ln.argtypes = [d]
        L.orc_exp.restype = d; L.orc_exp.argtypes = [d]
        L.orc_k1_const.restype = d
        L.orc_k1_const.argtypes = [d, d, d, ctypes.POINTER(i)]
        L.orc_priority.restype = d
        L.orc_priority.argtypes = [d, d, d, i, u64]
        L.orc_key_bits.restype = u64; L.orc_key_bits.argtypes = [d]
        L.orc_audit_monotone.restype = u64
        L.orc_audit_monotone.argtypes = [d, d, d, i, u64, u64]
        L.orc_classify.restype = i
        L.orc_classify.argtypes = [ctypes.c_void_p, ctypes.c_uint8, ctypes.c_uint32]
        L.orc_iso_ttft.restype = u64
        L.orc_iso_ttft.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        L.orc_iso_e2e.restype = u64
        L.orc_iso_e2e.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                  ctypes.c_uint32, ctypes.c_uint16]
        L.orc_simulate.restype = i
        L.orc_simulate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32] + \
            [ctypes.c_void_p] * 10 + [ctypes.c_void_p, u64, ctypes.c_void_p, u64]
        L.orc_simulate_growth.restype = i
        L.orc_simulate_growth.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32] + \
            [ctypes.c_void_p] * 14 + [u64]
        L.orc_decide.restype = ctypes.c_int
        L.orc_decide.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, u64, u64,
                                 ctypes.c_uint32] + [ctypes.c_void_p] * 9
        L.orc_ttft_bucket.restype = ctypes.c_uint32
        L.orc_ttft_bucket.argtypes = [u64]
        L.orc_aggregate.restype = None
        L.orc_aggregate.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32] + \
            [ctypes.c_void_p] * 9
        _lib = L
    return _lib


def model(c0_us=5000, cp_us=20, cd_us=500, S=PAPER_S, k=PAPER_K, p=PAPER_P, thresholds=SMART_THR,
          slo_num=5, slo_den=1) -> OrcModel:
    m = OrcModel()
    m.c0_us, m.cp_us, m.cd_us = c0_us, cp_us, cd_us
    for c in range(3):
        m.S[c], m.k[c], m.p[c] = S[c], k[c], p[c]
        m.thr_mc[c], m.thr_ct[c] = thresholds[c]
    m.slo_num, m.slo_den = slo_num, slo_den
    return m


def ln(v: float) -> float:
    return lib().orc_ln(v)


def exp(y: float) -> float:
    return lib().orc_exp(y)


def k1_const(alpha: float, k: float, p: float):
    z = ctypes.c_int(0)
    C = lib().orc_k1_const(alpha, k, p, ctypes.byref(z))
    return C, z.value


def priority(cls: int, w_us: int, alpha: float = 1.0, m: OrcModel | None = None) -> float:
    m = m or model()
    C, z = k1_const(alpha, m.k[cls], m.p[cls])
    return lib().orc_priority(m.S[cls], m.p[cls], C, z, int(w_us))


def audit_monotone(cls: int, w_lo: int, w_hi: int, alpha: float = 1.0, m=None) -> int | None:
    """First w in [w_lo, w_hi) where key(w+1) < key(w), or None (Lemma L1)."""
    m = m or model()
    C, z = k1_const(alpha, m.k[cls], m.p[cls])
    r = lib().orc_audit_monotone(m.S[cls], m.p[cls], C, z, int(w_lo), int(w_hi))
    return None if r == 0xFFFFFFFFFFFFFFFF else r


def key_bits(P: float) -> int:
    return lib().orc_key_bits(P)


def classify(modality: int, footprint: int, m: OrcModel | None = None) -> int:
    m = m or model()
    return lib().orc_classify(ctypes.byref(m), modality, footprint)


def iso_ttft(footprint, inline_us, chunk_budget=2048, m=None) -> int:
    m = m or model()
    return lib().orc_iso_ttft(ctypes.byref(m), chunk_budget, footprint, inline_us)


def iso_e2e(footprint, inline_us, out, chunk_budget=2048, m=None) -> int:
    m = m or model()
    return lib().orc_iso_e2e(ctypes.byref(m), chunk_budget, footprint, inline_us, out)


def ttft_bucket(t: int) -> int:
    return lib().orc_ttft_bucket(int(t))


@dataclass
class Result:
    admit_seq: np.ndarray
    first_token_us: np.ndarray
    done_us: np.ndarray
    cls: np.ndarray
    counters: dict
    iters: np.ndarray | None
    status: int


def simulate(arrival_us, footprint, inline_us, out_tokens, modality, policy=TCM, alpha=1.0,
             kv_capacity=131072, chunk_budget=2048, m: OrcModel | None = None,
             log: bool = False, max_iters: int = 0, admit_skip: bool = False) -> Result:
    """Run one replica through the oracle engine loop."""
    m = m or model()
    a = np.ascontiguousarray(arrival_us, dtype=np.uint64)
    f = np.ascontiguousarray(footprint, dtype=np.uint32)
    il = np.ascontiguousarray(inline_us, dtype=np.uint32)
    o = np.ascontiguousarray(out_tokens, dtype=np.uint16)
    md = np.ascontiguousarray(modality, dtype=np.uint8)
    n = len(a)
    seq = np.full(n, 0xFFFFFFFF, np.uint32)
    ft = np.zeros(n, np.uint64)
    dn = np.zeros(n, np.uint64)
    cl = np.zeros(n, np.uint8)
    cnt = OrcCounters()
    r = OrcReplica(policy, chunk_budget, kv_capacity, alpha, int(admit_skip), 0)
    cap = 0
    logbuf = None
    log_n = ctypes.c_uint64(0)
    if log:
        cap = 1 << 22
        logbuf = np.zeros(cap, dtype=ITER_DTYPE)
    st = lib().orc_simulate(
        ctypes.byref(m), ctypes.byref(r), n, a.ctypes.data, f.ctypes.data, il.ctypes.data,
        o.ctypes.data, md.ctypes.data, seq.ctypes.data, ft.ctypes.data, dn.ctypes.data,
        cl.ctypes.data, ctypes.byref(cnt), None if logbuf is None else logbuf.ctypes.data, cap,
        ctypes.byref(log_n), max_iters)
    counters = {name: getattr(cnt, name) for name, _ in OrcCounters._fields_}
    iters = None
    if log:
        assert log_n.value <= cap, "iteration log overflow"
        iters = logbuf[: log_n.value].copy()
    return Result(seq, ft, dn, cl, counters, iters, st)


@dataclass
class GrowthResult:
    admit_seq: np.ndarray
    first_token_us: np.ndarray
    done_us: np.ndarray
    preempt_count: np.ndarray
    preempted_us: np.ndarray
    cls: np.ndarray
    counters: dict
    status: int


def decide(arrival_us, footprint, inline_us, out_tokens, cls, rem, reserved, clock, kv_free, n_dec,
           policy=TCM, alpha=1.0, chunk_budget=2048, m: OrcModel | None = None, admit_skip=False):
    """One decision on an explicit state; every request is pending.
    Returns (chunk per request, admit rank per request or -1, tokens, inline, kv_free after, Bp)."""
    m = m or model()
    n = len(arrival_us)
    a = np.ascontiguousarray(arrival_us, dtype=np.uint64)
    f = np.ascontiguousarray(footprint, dtype=np.uint32)
    il = np.ascontiguousarray(inline_us, dtype=np.uint32)
    o = np.ascontiguousarray(out_tokens, dtype=np.uint16)
    cl = np.ascontiguousarray(cls, dtype=np.uint8)
    rem0 = np.ascontiguousarray(rem, dtype=np.uint32)
    rm = rem0.copy()
    rs = np.ascontiguousarray(reserved, dtype=np.uint8).copy()
    seq = np.full(n, 0xFFFFFFFF, dtype=np.uint32)
    res = np.zeros(4, dtype=np.uint64)
    r = OrcReplica(policy, chunk_budget, 1 << 40, alpha, int(admit_skip), 0)
    st = lib().orc_decide(ctypes.byref(m), ctypes.byref(r), n, int(clock), int(kv_free), int(n_dec),
                          a.ctypes.data, f.ctypes.data, il.ctypes.data, o.ctypes.data, cl.ctypes.data,
                          rm.ctypes.data, rs.ctypes.data, seq.ctypes.data, res.ctypes.data)
    if st != 0:
        raise ValueError("orc_decide: bad argument")
    adm = np.where(seq == 0xFFFFFFFF, -1, seq.astype(np.int64))
    return (rem0 - rm).astype(np.int64), adm, int(res[0]), int(res[1]), int(res[2]), int(res[3])


def simulate_growth(arrival_us, footprint, inline_us, out_tokens, modality, policy=TCM, alpha=1.0,
                    kv_capacity=131072, chunk_budget=2048, m: OrcModel | None = None,
                    max_iters: int = 0, admit_skip: bool = False) -> GrowthResult:
    """NEXT-1 engine loop: decode KV growth + preemption by recomputation (R28-R32)."""
    m = m or model()
    a = np.ascontiguousarray(arrival_us, dtype=np.uint64)
    f = np.ascontiguousarray(footprint, dtype=np.uint32)
    il = np.ascontiguousarray(inline_us, dtype=np.uint32)
    o = np.ascontiguousarray(out_tokens, dtype=np.uint16)
    md = np.ascontiguousarray(modality, dtype=np.uint8)
    n = len(a)
    seq = np.full(n, 0xFFFFFFFF, np.uint32)
    ft = np.zeros(n, np.uint64)
    dn = np.zeros(n, np.uint64)
    pc = np.zeros(n, np.uint32)
    pt = np.zeros(n, np.uint64)
    cl = np.zeros(n, np.uint8)
    cnt = OrcCounters()
    npre, nforced = ctypes.c_uint64(0), ctypes.c_uint64(0)
    r = OrcReplica(policy, chunk_budget, kv_capacity, alpha, int(admit_skip), 0)
    st = lib().orc_simulate_growth(
        ctypes.byref(m), ctypes.byref(r), n, a.ctypes.data, f.ctypes.data, il.ctypes.data,
        o.ctypes.data, md.ctypes.data, seq.ctypes.data, ft.ctypes.data, dn.ctypes.data,
        pc.ctypes.data, pt.ctypes.data, cl.ctypes.data, ctypes.byref(cnt), ctypes.byref(npre),
        ctypes.byref(nforced), max_iters)
    counters = {name: getattr(cnt, name) for name, _ in OrcCounters._fields_}
    counters["preemptions"] = npre.value
    counters["forced_preemptions"] = nforced.value
    return GrowthResult(seq, ft, dn, pc, pt, cl, counters, st)


def simulate_trace_growth(tr, r: int, policy=TCM, alpha=1.0, kv_capacity=131072, chunk_budget=2048,
                          m=None, max_iters=0, admit_skip=False) -> GrowthResult:
    a, b = int(tr.offset[r]), int(tr.offset[r + 1])
    return simulate_growth(tr.arrival_us[a:b], tr.footprint[a:b], tr.inline_us[a:b],
                           tr.out_tokens[a:b], tr.modality[a:b], policy, alpha, kv_capacity,
                           chunk_budget, m, max_iters, admit_skip)


def simulate_trace(tr, r: int, policy=TCM, alpha=1.0, kv_capacity=131072, chunk_budget=2048,
                   m=None, log=False, max_iters=0, admit_skip=False) -> Result:
    a, b = int(tr.offset[r]), int(tr.offset[r + 1])
    return simulate(tr.arrival_us[a:b], tr.footprint[a:b], tr.inline_us[a:b],
                    tr.out_tokens[a:b], tr.modality[a:b], policy, alpha, kv_capacity,
                    chunk_budget, m, log, max_iters, admit_skip)


def aggregate(tr_slice, res: Result, chunk_budget=2048, m=None, hist=None, cnt=None):
    """a6 aggregation of one replica's results into (hist[4][496], cnt[4][6]) int64 arrays."""
    m = m or model()
    if hist is None:
        hist = np.zeros((GROUPS, HIST_BINS), np.int64)
    if cnt is None:
        cnt = np.zeros((GROUPS, NCNT), np.int64)
    a = np.ascontiguousarray(tr_slice.arrival_us, dtype=np.uint64)
    lib().orc_aggregate(ctypes.byref(m), chunk_budget, len(a), a.ctypes.data,
                        np.ascontiguousarray(tr_slice.footprint, np.uint32).ctypes.data,
                        np.ascontiguousarray(tr_slice.inline_us, np.uint32).ctypes.data,
                        np.ascontiguousarray(tr_slice.out_tokens, np.uint16).ctypes.data,
                        np.ascontiguousarray(tr_slice.modality, np.uint8).ctypes.data,
                        np.ascontiguousarray(res.first_token_us, np.uint64).ctypes.data,
                        np.ascontiguousarray(res.done_us, np.uint64).ctypes.data,
                        hist.ctypes.data, cnt.ctypes.data)
    return hist, cnt
