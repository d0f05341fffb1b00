"""Thin ctypes binding of libtcm (include/tcm.h): same names, argument marshalling only.

Every step of the scheduling path runs in libtcm's CUDA kernels; this module only turns
torch tensors / numpy arrays into pointers.  There is no CPU fallback: if libtcm.so is
missing or no CUDA device is present, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TCM_LIB_PATH") or os.path.join(_HERE, "_build", "libtcm.so")

TCM_ABI_VERSION = 3
TCM_OK = 0
ERRORS = {-1: "TCM_E_ARG", -2: "TCM_E_STATE", -3: "TCM_E_CAPACITY", -4: "TCM_E_CUDA",
          -5: "TCM_E_OOM", -6: "TCM_E_REPLICA", -7: "TCM_E_VERSION"}
POLICY_FCFS, POLICY_TCM, POLICY_EDF, POLICY_NAIVE_AGING = 0, 1, 2, 3
ADMIT_SKIP = 1
KV_GROWTH = 2          # NEXT-1: decode KV growth + preemption by recomputation (R28-R32)
ENGINE_FUSED, ENGINE_STEPWISE = 0, 1
MEM_DEVICE, MEM_HOST = 0, 1
HIST_BINS, GROUPS, NCNT = 496, 4, 6
INF32 = 0xFFFFFFFF

EXPORTS = ("tcm_create", "tcm_load_trace", "tcm_reset", "tcm_step", "tcm_run", "tcm_run_async", "tcm_wait", "tcm_stats",
           "tcm_destroy",
           "tcm_last_error", "tcm_workspace_bytes", "tcm_generate_trace", "tcm_k1_eval",
           "tcm_k1_audit", "tcm_k1_filter_error", "tcm_replica_counters", "tcm_preemption_stats")


class TcmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class tcm_config(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_uint32), ("engine", ctypes.c_uint32),
        ("c0_us", ctypes.c_uint64), ("cp_us", ctypes.c_uint64), ("cd_us", ctypes.c_uint64),
        ("S", ctypes.c_double * 3), ("k", ctypes.c_double * 3), ("p", ctypes.c_double * 3),
        ("thr_mc", ctypes.c_uint32 * 3), ("thr_ct", ctypes.c_uint32 * 3),
        ("slo_num", ctypes.c_uint32), ("slo_den", ctypes.c_uint32),
        ("n_cells", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
    ]


class tcm_trace_view(ctypes.Structure):
    _fields_ = [
        ("mem", ctypes.c_uint32), ("n_replicas", ctypes.c_uint32), ("n_requests", ctypes.c_uint64),
        ("req_offset", ctypes.c_void_p), ("arrival_us", ctypes.c_void_p),
        ("footprint", ctypes.c_void_p), ("inline_us", ctypes.c_void_p),
        ("out_tokens", ctypes.c_void_p), ("modality", ctypes.c_void_p), ("params", ctypes.c_void_p),
    ]


class tcm_results_view(ctypes.Structure):
    _fields_ = [
        ("mem", ctypes.c_uint32), ("reserved", ctypes.c_uint32), ("admit_seq", ctypes.c_void_p),
        ("first_token_us", ctypes.c_void_p), ("done_us", ctypes.c_void_p),
        ("preempt_count", ctypes.c_void_p), ("preempted_us", ctypes.c_void_p),
    ]


class tcm_stats_host(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "iterations", "decisions", "ff_iterations", "idle_jumps", "sum_pending", "max_pending",
        "requests_done", "replicas_done", "replicas_active", "kernel_launches", "scanned_decisions")] + [
        ("first_bad_replica", ctypes.c_int32), ("first_bad_status", ctypes.c_int32),
        ("reset_ms", ctypes.c_double), ("engine_ms", ctypes.c_double), ("stamp_ms", ctypes.c_double),
        ("preemptions", ctypes.c_uint64), ("forced_preemptions", ctypes.c_uint64)]


# tcm_replica_params (32 B) as a numpy record so whole sweeps are built vectorised.
PARAMS_DTYPE = np.dtype([("policy", "<u4"), ("chunk_budget", "<u4"), ("kv_capacity", "<u8"),
                         ("aging_alpha", "<f8"), ("cell_id", "<u4"), ("flags", "<u4")])
assert PARAMS_DTYPE.itemsize == 32

_lib = None


def lib():
    """Load libtcm.so (raises if it has not been built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libtcm.so not built at {LIB_PATH}: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, st = ctypes.c_void_p, ctypes.c_int32
        L.tcm_create.restype = st
        L.tcm_create.argtypes = [ctypes.POINTER(tcm_config), vp, ctypes.POINTER(vp)]
        L.tcm_load_trace.restype = st
        L.tcm_load_trace.argtypes = [vp, ctypes.POINTER(tcm_trace_view), ctypes.POINTER(tcm_results_view)]
        L.tcm_reset.restype = st
        L.tcm_reset.argtypes = [vp]
        L.tcm_step.restype = st
        L.tcm_step.argtypes = [vp, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]
        L.tcm_run.restype = st
        L.tcm_run.argtypes = [vp]
        L.tcm_run_async.restype = st
        L.tcm_run_async.argtypes = [vp]
        L.tcm_wait.restype = st
        L.tcm_wait.argtypes = [vp, ctypes.c_int]
        L.tcm_stats.restype = st
        L.tcm_stats.argtypes = [vp, ctypes.POINTER(tcm_stats_host), vp, vp]
        L.tcm_replica_counters.restype = st
        L.tcm_replica_counters.argtypes = [vp, vp]
        L.tcm_preemption_stats.restype = st
        L.tcm_preemption_stats.argtypes = [vp, vp]
        L.tcm_destroy.restype = None
        L.tcm_destroy.argtypes = [vp]
        L.tcm_last_error.restype = ctypes.c_char_p
        L.tcm_last_error.argtypes = [vp]
        L.tcm_workspace_bytes.restype = ctypes.c_size_t
        L.tcm_workspace_bytes.argtypes = [ctypes.POINTER(tcm_config), ctypes.c_uint32, ctypes.c_uint64,
                                          ctypes.c_int]
        L.tcm_generate_trace.restype = st
        L.tcm_generate_trace.argtypes = [vp, ctypes.c_uint32] + [vp] * 7
        L.tcm_k1_eval.restype = st
        L.tcm_k1_eval.argtypes = [ctypes.POINTER(tcm_config), vp, vp, vp, vp, ctypes.c_uint64, vp]
        L.tcm_k1_audit.restype = st
        L.tcm_k1_audit.argtypes = [ctypes.POINTER(tcm_config), ctypes.c_uint32, ctypes.c_double,
                                   ctypes.c_uint64, ctypes.c_uint64, vp, vp]
        L.tcm_k1_filter_error.restype = st
        L.tcm_k1_filter_error.argtypes = [ctypes.POINTER(tcm_config), ctypes.c_uint32, ctypes.c_double,
                                          ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.POINTER(ctypes.c_double), vp]
        _lib = L
    return _lib


def _check(code, ctx=None):
    if code != TCM_OK:
        msg = lib().tcm_last_error(ctx)
        raise TcmError(code, msg.decode() if msg else "")


def config(engine=ENGINE_FUSED, c0_us=5000, cp_us=20, cd_us=500, S=(0.1, 0.05, 0.0),
           k=(0.05, 0.003, 0.00075), p=(3.5, 2.5, 1.1),
           thresholds=((4096, INF32), (0, INF32), (0, 8192)), slo_num=5, slo_den=1,
           n_cells=1) -> tcm_config:
    """tcm_config with the paper's constants, SPEC cost model and
    the smart-classifier thresholds of reading R13."""
    c = tcm_config()
    c.abi_version = TCM_ABI_VERSION
    c.engine = engine
    c.c0_us, c.cp_us, c.cd_us = c0_us, cp_us, cd_us
    for i in range(3):
        c.S[i], c.k[i], c.p[i] = S[i], k[i], p[i]
        c.thr_mc[i], c.thr_ct[i] = thresholds[i]
    c.slo_num, c.slo_den, c.n_cells, c.reserved = slo_num, slo_den, n_cells, 0
    return c


def make_params(n, policy=POLICY_TCM, chunk_budget=2048, kv_capacity=131072, aging_alpha=1.0,
                cell_id=0) -> np.ndarray:
    a = np.zeros(n, dtype=PARAMS_DTYPE)
    a["policy"], a["chunk_budget"], a["kv_capacity"] = policy, chunk_budget, kv_capacity
    a["aging_alpha"], a["cell_id"] = aging_alpha, cell_id
    return a


def _ptr(x):
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


def tcm_create(cfg: tcm_config, stream=None):
    ctx = ctypes.c_void_p()
    s = None if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    _check(lib().tcm_create(ctypes.byref(cfg), s, ctypes.byref(ctx)))
    return ctx


def tcm_load_trace(ctx, trace: dict, results: dict | None, mem=MEM_DEVICE):
    """trace: dict of arrays (torch device tensors for MEM_DEVICE, numpy for MEM_HOST) with keys
    req_offset, arrival_us, footprint, inline_us, out_tokens, modality, params."""
    tv = tcm_trace_view()
    tv.mem = mem
    tv.n_replicas = len(trace["req_offset"]) - 1
    tv.n_requests = len(trace["arrival_us"])
    for k in ("req_offset", "arrival_us", "footprint", "inline_us", "out_tokens", "modality", "params"):
        setattr(tv, k, _ptr(trace[k]))
    rv = tcm_results_view()
    rv.mem = mem
    if results:
        rv.admit_seq = _ptr(results.get("admit_seq"))
        rv.first_token_us = _ptr(results.get("first_token_us"))
        rv.done_us = _ptr(results.get("done_us"))
        rv.preempt_count = _ptr(results.get("preempt_count"))
        rv.preempted_us = _ptr(results.get("preempted_us"))
    _check(lib().tcm_load_trace(ctx, ctypes.byref(tv), ctypes.byref(rv)), ctx)


def tcm_reset(ctx):
    _check(lib().tcm_reset(ctx), ctx)


def tcm_step(ctx, max_iterations: int) -> int:
    active = ctypes.c_uint32(0)
    _check(lib().tcm_step(ctx, max_iterations, ctypes.byref(active)), ctx)
    return active.value


def tcm_run(ctx):
    _check(lib().tcm_run(ctx), ctx)


WAIT_ENGINE, WAIT_ALL = 0, 1


def tcm_run_async(ctx):
    _check(lib().tcm_run_async(ctx), ctx)


def tcm_wait(ctx, what: int = WAIT_ALL):
    _check(lib().tcm_wait(ctx, what), ctx)


def tcm_stats(ctx, dev_hist=None, dev_cnt=None) -> dict:
    s = tcm_stats_host()
    _check(lib().tcm_stats(ctx, ctypes.byref(s), _ptr(dev_hist), _ptr(dev_cnt)), ctx)
    return {n: getattr(s, n) for n, _ in tcm_stats_host._fields_}


REPLICA_COUNTERS = ("iterations", "decisions", "sum_pending", "scanned_decisions", "requests_done", "preemptions")


def tcm_replica_counters(ctx, dev_out):
    """dev_out: device uint64 tensor [R, 6] (REPLICA_COUNTERS order)."""
    _check(lib().tcm_replica_counters(ctx, _ptr(dev_out)), ctx)


PREEMPT_COUNTERS = ("preemptions", "preempted_us", "requests_preempted")


def tcm_preemption_stats(ctx, dev_out):
    """dev_out: device int64 tensor [n_cells, 4, 3] (groups M, C, T, all; PREEMPT_COUNTERS order)."""
    _check(lib().tcm_preemption_stats(ctx, _ptr(dev_out)), ctx)


def tcm_destroy(ctx):
    lib().tcm_destroy(ctx)


def tcm_last_error(ctx=None) -> str:
    return (lib().tcm_last_error(ctx) or b"").decode()


def tcm_workspace_bytes(cfg, n_replicas, n_requests, host_mirror=False) -> int:
    return lib().tcm_workspace_bytes(ctypes.byref(cfg), n_replicas, n_requests, int(host_mirror))


def tcm_generate_trace(reps_dev, req_offset_dev, out: dict, stream=None):
    """reps_dev: device uint8 tensor holding tcm_gen_replica records (48 B each)."""
    s = None if stream is None else stream.cuda_stream
    R = reps_dev.numel() // 48
    _check(lib().tcm_generate_trace(_ptr(reps_dev), R, _ptr(req_offset_dev), _ptr(out["arrival_us"]),
                                    _ptr(out["footprint"]), _ptr(out["inline_us"]),
                                    _ptr(out["out_tokens"]), _ptr(out["modality"]), s))


def tcm_k1_eval(cfg, cls_dev, w_dev, alpha_dev, out_dev, stream=None):
    s = None if stream is None else stream.cuda_stream
    _check(lib().tcm_k1_eval(ctypes.byref(cfg), _ptr(cls_dev), _ptr(w_dev), _ptr(alpha_dev),
                             _ptr(out_dev), out_dev.numel(), s))


def tcm_k1_audit(cfg, cls, alpha, w_lo, w_hi, first_dev, stream=None):
    s = None if stream is None else stream.cuda_stream
    _check(lib().tcm_k1_audit(ctypes.byref(cfg), cls, alpha, w_lo, w_hi, _ptr(first_dev), s))


def tcm_k1_filter_error(cfg, cls, alpha, w_lo, w_hi, step=1, stream=None) -> float:
    s = None if stream is None else stream.cuda_stream
    out = ctypes.c_double(0.0)
    _check(lib().tcm_k1_filter_error(ctypes.byref(cfg), cls, alpha, w_lo, w_hi, step, ctypes.byref(out), s))
    return out.value


# --------------------------------------------------------------------------------------
# Convenience layer over the same calls (torch for device memory and streams only).
# --------------------------------------------------------------------------------------
_TORCH_DT = None


def _dtypes():
    import torch
    return {"req_offset": torch.uint64, "arrival_us": torch.uint64, "footprint": torch.uint32,
            "inline_us": torch.uint32, "out_tokens": torch.uint16, "modality": torch.uint8}


def to_device(trace, params: np.ndarray, device="cuda") -> dict:
    """Copy a tracegen.Trace (numpy SoA) and a PARAMS_DTYPE array to device tensors."""
    import torch
    d = {}
    for k, dt in _dtypes().items():
        arr = trace.offset if k == "req_offset" else getattr(trace, k)
        d[k] = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
        assert d[k].dtype == dt
    d["params"] = torch.from_numpy(np.ascontiguousarray(params).view(np.uint8)).to(device)
    return d


def to_device_params(params: np.ndarray, device="cuda"):
    """PARAMS_DTYPE records -> device byte tensor (tcm_replica_params[R])."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(params, dtype=PARAMS_DTYPE).view(np.uint8)).to(device)


def alloc_results(n: int, device="cuda", preemption: bool = False) -> dict:
    import torch
    res = {"admit_seq": torch.empty(n, dtype=torch.uint32, device=device),
           "first_token_us": torch.empty(n, dtype=torch.uint64, device=device),
           "done_us": torch.empty(n, dtype=torch.uint64, device=device)}
    if preemption:     # NEXT-1 outputs (stepwise engine with KV_GROWTH replicas)
        res["preempt_count"] = torch.empty(n, dtype=torch.uint32, device=device)
        res["preempted_us"] = torch.empty(n, dtype=torch.uint64, device=device)
    return res


def generate_device(reps: np.ndarray, device="cuda", stream=None) -> dict:
    """Generate traces on the device (tcm_generate_trace) from tracegen replica records."""
    import torch
    counts = reps["n_requests"].astype(np.uint64)
    off = np.zeros(len(reps) + 1, np.uint64)
    np.cumsum(counts, out=off[1:])
    N = int(off[-1])
    out = {"req_offset": torch.from_numpy(off).to(device),
           "arrival_us": torch.empty(N, dtype=torch.uint64, device=device),
           "footprint": torch.empty(N, dtype=torch.uint32, device=device),
           "inline_us": torch.empty(N, dtype=torch.uint32, device=device),
           "out_tokens": torch.empty(N, dtype=torch.uint16, device=device),
           "modality": torch.empty(N, dtype=torch.uint8, device=device)}
    reps_dev = torch.from_numpy(np.ascontiguousarray(reps).view(np.uint8)).to(device)
    tcm_generate_trace(reps_dev, out["req_offset"], out, stream)
    return out


@dataclass
class Simulation:
    """One context: load a trace, run it, read results and the a6 aggregation."""
    cfg: tcm_config
    stream: object = None

    def __post_init__(self):
        self.ctx = tcm_create(self.cfg, self.stream)

    def load(self, trace: dict, results: dict | None = None, mem=MEM_DEVICE):
        # the library borrows every buffer until destroy / the next load (include/tcm.h):
        # keep them alive here so torch's allocator cannot recycle them underneath it
        self._borrowed = (trace, results)
        tcm_load_trace(self.ctx, trace, results, mem)

    def run(self):
        tcm_run(self.ctx)

    def run_async(self):
        tcm_run_async(self.ctx)

    def wait(self, what: int = WAIT_ALL):
        tcm_wait(self.ctx, what)

    def reset(self):
        tcm_reset(self.ctx)

    def step(self, max_iterations: int) -> int:
        return tcm_step(self.ctx, max_iterations)

    def stats(self) -> dict:
        return tcm_stats(self.ctx)

    def aggregate(self, device="cuda"):
        import torch
        import contextlib
        n = self.cfg.n_cells
        # tcm_stats overwrites both buffers on the context's stream; allocate them on that stream
        # so torch's allocator orders any reuse of their memory after the library's writes
        on = torch.cuda.stream(self.stream) if isinstance(self.stream, torch.cuda.Stream) else contextlib.nullcontext()
        with on:
            hist = torch.empty((n, GROUPS, HIST_BINS), dtype=torch.int64, device=device)
            cnt = torch.empty((n, GROUPS, NCNT), dtype=torch.int64, device=device)
        st = tcm_stats(self.ctx, hist, cnt)
        return hist, cnt, st

    def replica_counters(self, n_replicas: int, device="cuda") -> np.ndarray:
        """Per-replica counters as a structured numpy array (REPLICA_COUNTERS fields)."""
        import torch
        out = torch.empty((n_replicas, len(REPLICA_COUNTERS)), dtype=torch.uint64, device=device)
        tcm_replica_counters(self.ctx, out)
        a = out.cpu().numpy()
        return {k: a[:, i] for i, k in enumerate(REPLICA_COUNTERS)}

    def preemption_stats(self, device="cuda"):
        """fig:preemptions counters per (cell, group) from the device (int64 [n_cells, 4, 3])."""
        import torch
        import contextlib
        on = torch.cuda.stream(self.stream) if isinstance(self.stream, torch.cuda.Stream) else contextlib.nullcontext()
        with on:
            out = torch.empty((self.cfg.n_cells, GROUPS, len(PREEMPT_COUNTERS)), dtype=torch.int64, device=device)
        tcm_preemption_stats(self.ctx, out)
        return out

    def close(self):
        if self.ctx:
            tcm_destroy(self.ctx)
            self.ctx = None
        self._borrowed = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
