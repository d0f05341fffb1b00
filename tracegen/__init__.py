"""Seeded synthetic trace generator (input module shared by the oracle tests and the CUDA path).

Holds none of the scheduling arithmetic: it only draws inputs (SURVEY.md 8(d) recipe,
DESIGN.md "Input recipe").  The host build (libtracegen.so, from tcm_tracegen.h) and the
device build (compiled into libtcm.so as tcm_generate_trace) are bit-identical.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libtracegen.so")

# Workload mixes (text, image, video): SPEC.md:207 (TO/ML/MH) and the north star's 70/25/5, 50/20/30.
MIXES = {
    "TO": (1.0, 0.0, 0.0),
    "ML": (0.90, 0.07, 0.03),
    "MH": (0.60, 0.25, 0.15),
    "70/25/5": (0.70, 0.25, 0.05),
    "50/20/30": (0.50, 0.20, 0.30),
    "80/20/0": (0.80, 0.20, 0.0),
    "80/0/20": (0.80, 0.0, 0.20),
    "40/40/20": (0.40, 0.40, 0.20),
}


class TgReplica(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("kv_capacity", ctypes.c_uint64),
        ("mean_gap_us", ctypes.c_double),
        ("mix_t1", ctypes.c_uint64),
        ("mix_t2", ctypes.c_uint64),
        ("n_requests", ctypes.c_uint32),
        ("flags", ctypes.c_uint32),
    ]


assert ctypes.sizeof(TgReplica) == 48

TG_REPLICA_DTYPE = np.dtype(
    [("seed", "<u8"), ("kv_capacity", "<u8"), ("mean_gap_us", "<f8"), ("mix_t1", "<u8"),
     ("mix_t2", "<u8"), ("n_requests", "<u4"), ("flags", "<u4")]
)
assert TG_REPLICA_DTYPE.itemsize == 48

FLAG_ALL_AT_ZERO = 1


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "tracegen_host.c")
    hdr = os.path.join(_HERE, "tcm_tracegen.h")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(hdr)
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-Wall",
             "-o", _SO, src, "-lm"]
        )
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        L.tcmgen_make_replica.restype = TgReplica
        L.tcmgen_make_replica.argtypes = [
            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double,
            ctypes.c_double, ctypes.c_double, ctypes.c_uint64, ctypes.c_uint32,
        ]
        L.tcmgen_fill.restype = ctypes.c_int
        L.tcmgen_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint32] + [ctypes.c_void_p] * 6
        _lib = L
    return _lib


def make_replica(base_seed: int, replica: int, n_requests: int, rate: float,
                 mix=(0.70, 0.25, 0.05), kv_capacity: int = 131072, flags: int = 0) -> np.void:
    r = lib().tcmgen_make_replica(base_seed, replica, n_requests, float(rate), float(mix[0]),
                                  float(mix[1]), kv_capacity, flags)
    arr = np.zeros(1, dtype=TG_REPLICA_DTYPE)
    ctypes.memmove(arr.ctypes.data, ctypes.byref(r), 48)
    return arr[0]


@dataclass
class Trace:
    """SoA trace in CSR form (SURVEY.md 8(a) layout): replica r owns [offset[r], offset[r+1])."""

    offset: np.ndarray          # u64 [R+1]
    arrival_us: np.ndarray      # u64 [N]
    footprint: np.ndarray       # u32 [N] prompt + media tokens (KV footprint)
    inline_us: np.ndarray       # u32 [N] preprocess + encode (R10)
    out_tokens: np.ndarray      # u16 [N]
    modality: np.ndarray        # u8  [N] 0 text, 1 image, 2 video
    gen: np.ndarray = field(default=None)  # TG_REPLICA_DTYPE [R] (how it was generated)

    @property
    def n_replicas(self) -> int:
        return len(self.offset) - 1

    @property
    def n_requests(self) -> int:
        return int(self.offset[-1])

    def replica(self, r: int) -> "Trace":
        a, b = int(self.offset[r]), int(self.offset[r + 1])
        return Trace(np.array([0, b - a], dtype=np.uint64), self.arrival_us[a:b],
                     self.footprint[a:b], self.inline_us[a:b], self.out_tokens[a:b],
                     self.modality[a:b], None if self.gen is None else self.gen[r:r + 1])


def alloc(offset: np.ndarray) -> Trace:
    n = int(offset[-1])
    return Trace(offset.astype(np.uint64), np.zeros(n, np.uint64), np.zeros(n, np.uint32),
                 np.zeros(n, np.uint32), np.zeros(n, np.uint16), np.zeros(n, np.uint8))


def generate(reps: np.ndarray) -> Trace:
    """Generate every replica described by a TG_REPLICA_DTYPE array (host, OpenMP)."""
    reps = np.ascontiguousarray(reps, dtype=TG_REPLICA_DTYPE)
    counts = reps["n_requests"].astype(np.uint64)
    offset = np.zeros(len(reps) + 1, dtype=np.uint64)
    np.cumsum(counts, out=offset[1:])
    t = alloc(offset)
    rc = lib().tcmgen_fill(reps.ctypes.data, len(reps), t.offset.ctypes.data,
                           t.arrival_us.ctypes.data, t.footprint.ctypes.data,
                           t.inline_us.ctypes.data, t.out_tokens.ctypes.data,
                           t.modality.ctypes.data)
    if rc != 0:
        raise RuntimeError("tcmgen_fill failed")
    t.gen = reps
    return t


def from_requests(reqs) -> Trace:
    """Hand-written trace for one replica: reqs = [(arrival_us, footprint, inline_us, out, modality)]."""
    n = len(reqs)
    t = alloc(np.array([0, n], dtype=np.uint64))
    for i, (a, f, inl, o, m) in enumerate(reqs):
        t.arrival_us[i] = a
        t.footprint[i] = f
        t.inline_us[i] = inl
        t.out_tokens[i] = o
        t.modality[i] = m
    return t


def concat(traces) -> Trace:
    """Stack single- or multi-replica traces into one CSR trace."""
    counts = []
    for tr in traces:
        counts.extend(np.diff(tr.offset).tolist())
    offset = np.zeros(len(counts) + 1, dtype=np.uint64)
    np.cumsum(np.array(counts, dtype=np.uint64), out=offset[1:])
    return Trace(offset, np.concatenate([t.arrival_us for t in traces]),
                 np.concatenate([t.footprint for t in traces]),
                 np.concatenate([t.inline_us for t in traces]),
                 np.concatenate([t.out_tokens for t in traces]),
                 np.concatenate([t.modality for t in traces]))
