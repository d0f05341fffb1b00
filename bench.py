#!/usr/bin/env python3
"""Benchmark: TCM-Serve's per-iteration scheduling step as a trace-driven simulation on B200.

Metric (BASELINE.json): scheduling decisions/s and simulated requests/s at 1/2/4/8 B200, with
the HBM-roofline fraction.  Workload at N GPUs: the C4 memory-pressure sweep (video-heavy
50/20/30 mix, KV {128k,64k,32k,16k} x lambda {0.5,1,2,4} x {FCFS,TCM}), 65,536 replicas x
10,000 requests PER GPU (weak scaling: replicas are independent; rank k simulates global
replicas k, k+N, ...).  One step = reset + tcm_run (rows a1-a5 to completion for every
replica) + a6 aggregation (tcm_stats) + NCCL all-reduce of the int64 histograms (N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tcm|reference]

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle (the reference arm for
this tier) on a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0           # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)

# Algorithmic bytes of the path per simulated request: the trace SoA read once
# (arrival 8 + footprint 4 + inline 4 + out 2 + modality 1 = 19 B), the results written once
# (admit_seq 4 + first_token 8 + done 8 = 20 B) and the decode-calendar update (~16 B); per replica
# the 128 B state read + written.  k_fused's own workspace traffic (class records, event log, finish
# iterations: DESIGN.md 7) is implementation overhead and is reported apart, not counted.
ALG_BYTES_PER_REQ = 19 + 20 + 16
ALG_BYTES_PER_REPLICA = 256
FUSED_WS_BYTES_PER_REQ = 32 + 16 + 8 + 8     # record read + event log + finish iteration + record write
STEP_BYTES_PER_PENDING = 9                 # stepwise: arrival (8) + state byte (1) per pending key
STEP_BYTES_PER_DECISION = 256              # replica state r+w

# One metric string per workload, identical on both arms (the driver divides the two lines).
METRIC = {w: f"simulated requests/sec ({w.upper()} sweep)" for w in ("c3", "c4", "c5")}
METRIC["c4"] = "simulated requests/sec (C4 memory-pressure sweep)"
METRIC["c1"] = "simulated requests/sec (C1 single trace)"


def peak_hbm():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args):
    """`bench.py --gpus N` (N > 1) run without a launcher re-executes itself under torchrun with N
    ranks (one process per GPU, rendezvous on 127.0.0.1).  Returns the exit code, or None when this
    process is already a rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")              # communicator-init lines (rank count, transport)
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/tmp/tcm_bench_nccl.%h.%p.log")   # keep stdout to the JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    log("spawning:", " ".join(cmd))
    return subprocess.call(cmd, env=env)


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    if world > 1:
        import torch.distributed as dist
        if args.impl == "tcm":
            import torch
            ngpu = torch.cuda.device_count()
            if world <= ngpu:                # one process per GPU, NCCL over NVLink
                torch.cuda.set_device(local)
                dist.init_process_group(backend="nccl", device_id=torch.device("cuda", local))
                args.collective = "nccl"
            else:                            # more ranks than GPUs (a functional run on a smaller box):
                local = local % ngpu         # ranks share GPUs; NCCL refuses two ranks on one device,
                torch.cuda.set_device(local) # so the int64 all-reduce goes through gloo (CUDA tensors)
                dist.init_process_group(backend="gloo")
                args.collective = f"gloo ({world} ranks sharing {ngpu} GPU(s): functional, not a scaling point)"
        else:
            dist.init_process_group(backend="gloo")
        assert dist.get_world_size() == args.gpus
    return rank, world, local


def nccl_evidence():
    """NCCL version and the communicator-init lines NCCL_DEBUG=INFO wrote (rank 0's view)."""
    import glob
    out = {}
    try:
        import torch
        out["version"] = ".".join(str(v) for v in torch.cuda.nccl.version())
    except Exception:
        pass
    lines = []
    for f in sorted(glob.glob("/tmp/tcm_bench_nccl.*.log")):
        try:
            lines += [ln.strip() for ln in open(f) if "Init COMPLETE" in ln or "nranks" in ln][:4]
        except OSError:
            pass
    if lines:
        out["init_lines"] = lines[:16]
    return out


# ----------------------------------------------------------------------------------- oracle
def _oracle_job(job):
    import oracle as O
    import tracegen as T
    gen, pol, kv, alpha, budget, n = job
    rep = np.array([gen], dtype=T.TG_REPLICA_DTYPE)
    rep["n_requests"] = n
    tr = T.generate(rep)
    t0 = time.perf_counter()
    r = O.simulate_trace(tr, 0, policy=pol, alpha=alpha, kv_capacity=kv, chunk_budget=budget)
    dt = time.perf_counter() - t0
    assert r.status == 0
    return dt, n, r.counters["decisions"]


def cpu_model():
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def sample_ids(sweep, n_sample):
    """A deterministic sample spread over the sweep: the same number of replicas from every cell
    (the k-th sampled replica of a cell is its (k + 1/2) * (cell size / per-cell sample)-th one)."""
    cells = np.asarray(sweep.params["cell_id"])
    nc = int(cells.max()) + 1
    per = max(1, n_sample // nc)
    pick = range(nc) if nc <= n_sample else [int(c) for c in np.linspace(0, nc - 1, n_sample)]
    out = []
    for c in pick:
        idx = np.nonzero(cells == c)[0]
        step = max(1, len(idx) // per)
        out += [int(i) for i in idx[step // 2::step][:per]]
    return sorted(out)[:n_sample] if len(out) >= n_sample else sorted(out)


def oracle_sample(sweep, n_trunc=0, n_sample=64, cores=None):
    """Time the oracle (as it stands) on a bounded sample of the sweep: n_sample replicas spread
    over every cell (sample_ids), each truncated to its first n_trunc requests (0 = full length),
    one single-threaded oracle process per replica on `cores` host cores (all by default).
    Returns the all-core wall time and the sum of the per-replica (1-core) times."""
    import multiprocessing as mp
    idx = sample_ids(sweep, n_sample)
    jobs = [(sweep.gen[i], int(sweep.params[i]["policy"]), int(sweep.params[i]["kv_capacity"]),
             float(sweep.params[i]["aging_alpha"]), int(sweep.params[i]["chunk_budget"]),
             n_trunc or int(sweep.gen[i]["n_requests"])) for i in idx]
    cores = min(len(jobs), cores or os.cpu_count() or 1)
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:     # never fork a CUDA process
        res = pool.map(_oracle_job, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    nreq = sum(r[1] for r in res)
    ndec = sum(r[2] for r in res)
    cpu_s = sum(r[0] for r in res)
    return {"wall_s": wall, "requests": nreq, "decisions": ndec, "cores": cores, "replicas": len(jobs),
            "n_trunc": n_trunc, "one_core_s": cpu_s, "max_replica_s": max(r[0] for r in res)}


def cpu_baseline_line(s, workload):
    length = f"first {s['n_trunc']} requests each" if s["n_trunc"] else "full length"
    return {"value": s["requests"] / s["wall_s"], "unit": "requests/s", "cores": s["cores"], "kind": "oracle",
            "decisions_per_s": s["decisions"] / s["wall_s"],
            "one_core_value": s["requests"] / s["one_core_s"],
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "sample": f"{s['replicas']} {workload.upper()} replicas spread over every cell (every "
                      f"R/{s['replicas']}-th replica), {length}, one single-threaded oracle process per replica on "
                      f"{s['cores']} host cores: {s['wall_s']:.1f} s wall (all-core value), "
                      f"{s['one_core_s']:.1f} s summed per-replica time (one_core_value)"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on the box's host cores (rank 0 only)."""
    if rank != 0:
        return
    sw = make_sweep(args, 0, 1)
    n_sample = min(32, sw.n_replicas)
    for _ in range(args.warmup):
        oracle_sample(sw, n_trunc=args.ref_requests, n_sample=n_sample)
    tot_req = tot_dec = 0
    tot_wall = tot_one = 0.0
    s = None
    for _ in range(args.steps):
        s = oracle_sample(sw, n_trunc=args.ref_requests, n_sample=n_sample)
        tot_req += s["requests"]
        tot_dec += s["decisions"]
        tot_wall += s["wall_s"]
        tot_one += s["one_core_s"]
    v = tot_req / tot_wall
    cb = cpu_baseline_line(dict(s, requests=tot_req, decisions=tot_dec, wall_s=tot_wall, one_core_s=tot_one),
                           args.workload)
    line = {
        "impl": "reference", "metric": METRIC[args.workload], "value": v,
        "unit": "requests/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_wall / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic",
        "decisions_per_s": tot_dec / tot_wall,
        "config": {"workload": f"{workload_name(args, sw)} (bounded oracle sample: {n_sample} replicas, first "
                               f"{args.ref_requests} requests each)",
                   "replicas": n_sample, "requests_per_replica": args.ref_requests},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_sweep(args, rank, world):
    from paper_2603_26498_b200 import workloads as W
    if args.workload == "c5":
        # C5 (BASELINE.json configs[4]): 1M replicas on 8 GPUs = 131,072 per GPU (weak scaling)
        return W.c5(rank, world, replicas=args.replicas * world, n_requests=args.requests)
    if args.workload == "c3":
        # C3 (configs[2]): 4,096 replicas x 10k, lambda x alpha sweep, per GPU
        return W.c3(rank, world, replicas=args.replicas * world, n_requests=args.requests)
    if args.workload == "c1":
        # C1 (configs[0]): one replica x 1,000 requests (TCM), a single serial engine per GPU; rank k
        # simulates seed 1 + k so that ranks never count the same replica twice
        return W.c1(seed=1 + rank)
    return W.c4(rank, world, replicas_per_gpu=args.replicas, n_requests=args.requests)


def workload_name(args, sw):
    R = sw.n_replicas
    if args.workload == "c3":
        return (f"C3 sweep: {R} replicas x {args.requests} requests per GPU (16 lambda x 16 alpha x seeds, 70/25/5, "
                "TCM), fused engine")
    if args.workload == "c1":
        return "C1: 1 replica x 1,000 requests per GPU (70/25/5, 2 req/s, TCM), fused engine: one serial engine"
    if args.workload == "c5":
        return (f"C5 full policy sweep: {R} replicas x {args.requests} requests per GPU (16 lambda x 8 mixes x 16 "
                f"alpha x 8 chunk budgets = {sw.n_cells} cells x seeds; 1M replicas at 8 GPUs), fused engine, "
                "per-request results kept in the library workspace")
    return (f"C4 memory-pressure sweep: {args.replicas} replicas x {args.requests} requests per GPU "
            "(50/20/30 mix, KV 128k..16k x lambda 0.5..4 x FCFS/TCM), fused engine")


# ------------------------------------------------------------------------------------ GPU
def run_tcm(args, rank, world, local):
    import torch
    from paper_2603_26498_b200 import _build, tcm
    from paper_2603_26498_b200 import workloads as W

    _build.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

    sw = make_sweep(args, rank, world)
    R, N = sw.n_replicas, sw.n_requests
    log(f"rank {rank}: {args.workload.upper()} shard {R} replicas, {N} requests; generating on device")
    with torch.cuda.stream(stream):
        trace = tcm.generate_device(sw.gen, device=dev, stream=stream)
        trace["params"] = torch.from_numpy(sw.params.view(np.uint8)).to(dev)
        results = tcm.alloc_results(N, device=dev) if args.workload == "c4" else None
    stream.synchronize()
    cfg = tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells)
    sim = tcm.Simulation(cfg, stream)
    sim.load(trace, results)
    with torch.cuda.stream(stream):        # tcm_stats overwrites them on the library's stream
        hist = torch.empty((sw.n_cells, tcm.GROUPS, tcm.HIST_BINS), dtype=torch.int64, device=dev)
        cnt = torch.empty((sw.n_cells, tcm.GROUPS, tcm.NCNT), dtype=torch.int64, device=dev)

    def one_step():
        sim.reset()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.run()
        e1.record(stream)
        st = tcm.tcm_stats(sim.ctx, hist, cnt)
        if dist is not None:
            with torch.cuda.stream(stream):
                W.allreduce_aggregate(hist, cnt)      # int64 SUM over NVLink (NCCL)
        kms.append((st["reset_ms"], st["engine_ms"], st["stamp_ms"]))
        return e0, e1

    kms = []     # per step: library-recorded device ms of (reset + prologue, k_fused, k_fstamp)

    for _ in range(args.warmup):
        one_step()
    stream.synchronize()
    log("warm-up done")
    st0 = sim.stats()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local)
    sampler.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    kern = []
    kms.clear()
    for _ in range(args.steps):
        kern.append(one_step())
    t_end.record(stream)
    stream.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    ms = t_start.elapsed_time(t_end)
    run_ms = [a.elapsed_time(b) for a, b in kern]
    st1 = sim.stats()
    decisions = st1["decisions"] - 0  # counters reset each step: st1 holds the last step
    launches_per_step = (st1["kernel_launches"] - st0["kernel_launches"]) / args.steps

    # max over ranks of the device time; totals over ranks
    tot = torch.tensor([float(N * args.steps), float(st1["decisions"] * args.steps),
                        float(st1["iterations"] * args.steps), float(st1["scanned_decisions"] * args.steps)],
                       dtype=torch.float64, device=dev)
    mx = torch.tensor([ms, max(run_ms)], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(tot)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    ms_max = float(mx[0])
    req_s = float(tot[0]) / (ms_max / 1e3)
    dec_s = float(tot[1]) / (ms_max / 1e3)

    scan_s = float(tot[3]) / (ms_max / 1e3)
    # roofline of the dominant kernel (k_fused): SURVEY.md 8(d)'s algorithmic bytes per launch / its
    # launch time, from CUDA events the library records around the launch on this stream
    peak, peak_kind = peak_hbm()
    fused_ms = float(np.mean([k[1] for k in kms]))
    alg_bytes = N * ALG_BYTES_PER_REQ + R * ALG_BYTES_PER_REPLICA
    achieved = alg_bytes / (fused_ms / 1e3) / 1e9
    traffic = issue = None
    prof = os.path.join(ROOT, "profiles", "fused_dram_bytes.json")
    if os.path.exists(prof) and args.workload == "c4":
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_request")
            traffic = traffic * N if traffic else None
        except Exception:
            traffic = None
    # issue-rate roof of the same kernel (it is latency/divergence-bound, not HBM-bound): executed
    # warp instructions of one launch (ncu, committed profile) / (148 SMs x 4 schedulers x SM clock)
    prof = os.path.join(ROOT, "profiles", "fused_issue.json")
    if os.path.exists(prof) and args.workload == "c4":
        try:
            pi = json.load(open(prof))
            slots = 148 * 4 * pi["sm_clock_hz"] * (fused_ms / 1e3)
            issue = {"inst_executed_per_launch": pi["inst_executed"], "issue_slots_per_launch": slots,
                     "frac": pi["inst_executed"] / slots,
                     "thread_inst_per_inst": pi.get("thread_inst_per_inst"), "source": pi.get("source")}
        except Exception:
            issue = None

    wl = workload_name(args, sw)
    out = {
        "metric": METRIC[args.workload],
        "value": req_s, "unit": "requests/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic",
        "decisions_per_s": dec_s,
        "scanned_decisions_per_s": scan_s,
        "config": {"workload": wl, "n_cells": sw.n_cells,
                   "replicas_per_gpu": args.replicas, "requests_per_replica": args.requests,
                   "requests_per_step": int(tot[0] / args.steps), "parallelism": f"replicas sharded x{world}", "collective": getattr(args, "collective", "none (1 rank)"),
                   "l2": "inputs larger than L2 (trace %.1f GB per GPU)" % (N * 19 / 1e9)},
        "roofline": {"kernel": "k_fused", "bound": "hbm", "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "launch_ms": fused_ms, "alg_bytes_per_launch": alg_bytes,
                     "alg_bytes_per_request": ALG_BYTES_PER_REQ,
                     "workspace_bytes_per_launch": N * FUSED_WS_BYTES_PER_REQ,
                     "issue": issue,
                     "note": "SURVEY.md 8(d) algorithmic bytes (trace 19 + results 20 + calendar 16 B per request); "
                             "the kernel is bound by per-replica dependent chains and SIMT divergence, so the issue "
                             "roof is reported alongside (DESIGN.md 7)"},
        "kernel_ms_per_step": {"reset_and_prologue": float(np.mean([k[0] for k in kms])), "k_fused": fused_ms,
                               "k_fstamp": float(np.mean([k[2] for k in kms]))},
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clocks,
        "work": {"iterations_per_step": st1["iterations"], "decisions_per_step": st1["decisions"],
                 "sum_pending_per_step": st1["sum_pending"], "ff_iterations": st1["ff_iterations"],
                 "run_ms": run_ms},
    }

    log(f"timed: {ms:.1f} ms for {args.steps} steps")
    # stepwise (paper-literal) per-step kernel on C2': its own HBM roofline
    if not args.skip_step and rank == 0:
        st_res = bench_stepwise(args, dev, stream)
        out["roofline_step"] = st_res.pop("C2'")
        out["step_kernels"] = st_res

    if not args.skip_next1 and rank == 0:          # fig:preemptions with all three policies (stepwise)
        out["next1_policies"] = bench_next1(args, dev, stream)
        log("next1 (stepwise, FCFS/EDF/TCM) done")

    # end-to-end through the C ABI with HOST buffers (H2D + run + D2H inside the timed region)
    log("stepwise done")
    e2e_skip = None
    if not args.skip_e2e:
        # pinned host memory of the e2e leg on this node: the trace once and two contexts' results, per rank
        per_rank = sum(trace[k].numel() * trace[k].element_size() for k in trace if k != "params") + 2 * 20 * N
        local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        avail = host_mem_available()
        bad = 1 if (avail is not None and local_ranks * per_rank > 0.85 * avail) else 0
        if world > 1:                                  # every rank takes the same decision
            flag = torch.tensor([bad], dtype=torch.int64, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            bad = int(flag[0])
        if bad:
            e2e_skip = (f"not run: {local_ranks} ranks x {per_rank / 1e9:.1f} GB of pinned host memory exceed 85 % of "
                        f"this node's available {avail / 1e9:.0f} GB")
    if not args.skip_e2e and e2e_skip is None:
        # free the device-resident run first: the two e2e contexts need ~74 GB each
        host = host_copy(trace)
        # a sample of the device-resident run's results: the e2e leg's outputs are checked against it
        pick = torch.arange(0, N, 997, device=dev)
        def take(x):       # torch has no index kernels for unsigned dtypes: gather through a signed view
            sig = {torch.uint32: (torch.int32, np.uint32), torch.uint64: (torch.int64, np.uint64)}.get(x.dtype)
            return x[pick].cpu().numpy() if sig is None else x.view(sig[0])[pick].cpu().numpy().view(sig[1])
        ref = {k: take(results[k]) for k in ("admit_seq", "first_token_us", "done_us")}
        sim.close()
        del trace, results
        torch.cuda.empty_cache()
        out["e2e"] = bench_e2e(args, sw, host, dev, dist, world, (pick.cpu().numpy(), ref))
        del host
    elif e2e_skip is not None:
        out["e2e"] = {"value": None, "unit": "requests/s", "skipped": e2e_skip}
    log("e2e done")

    if not args.skip_next1 and args.workload == "c4" and rank == 0:
        # NEXT-1 at the C4 size (65,536 x 10,000) on the fused engine (k_fgrow), after the
        # device-resident C4 run is freed
        sim.close()
        trace = results = None
        torch.cuda.empty_cache()
        out["next1"] = bench_next1(args, dev, stream, engine=tcm.ENGINE_FUSED, replicas=args.replicas,
                                   requests=args.requests, policies=(tcm.POLICY_FCFS, tcm.POLICY_TCM))
        log("next1 (fused, C4 size) done")

    if rank == 0 and world == 1 and not args.skip_cpu:      # the oracle baseline: rank 0 at N=1 only
        s = oracle_sample(sw, n_trunc=0 if args.cpu_full else args.ref_requests,
                          n_sample=min(64, sw.n_replicas))
        out["cpu_baseline"] = cpu_baseline_line(s, args.workload)
        prof = os.path.join(ROOT, "profiles", f"cpu_baseline_full_{args.workload}.json")
        if not args.cpu_full and os.path.exists(prof):
            try:     # the full-length sample, measured once on this box type (bench.py --cpu-full)
                out["cpu_baseline_full_length"] = json.load(open(prof))
            except Exception:
                pass
    if world > 1 and rank == 0:
        out["nccl"] = nccl_evidence()
    sim.close()
    if rank == 0:
        print(json.dumps(out), flush=True)


def _stage_c2(replicas, pending, engine, dev, stream):
    import torch
    from paper_2603_26498_b200 import tcm
    from paper_2603_26498_b200 import workloads as W
    sw = W.c2prime(replicas=replicas, pending=pending)
    with torch.cuda.stream(stream):
        tr = tcm.generate_device(sw.gen, device=dev, stream=stream)
        first = tr["req_offset"][:-1].to(torch.int64)
        tr["inline_us"].view(torch.int32)[first] = 60_000_000     # 60 s of encode time
        tr["modality"][first] = 1
        tr["footprint"].view(torch.int32)[first] = 800
        tr["params"] = torch.from_numpy(sw.params.view(np.uint8)).to(dev)
    stream.synchronize()
    sim = tcm.Simulation(tcm.config(engine=engine), stream)
    sim.load(tr, None)
    return sim


def time_steps(sim, stream, iters, reps):
    """Device time of single steady-state engine iterations 3..iters+2 (iteration 1 runs request 0
    alone, iteration 2 also ingests every other request: its classify bytes are not in the
    9 B-per-pending figure, so it is not timed).
    Returns (kernel ms, call ms, pending): the kernel time is the library's own CUDA-event
    measurement around its k_step / k_fused launch on its stream (tcm_stats_host.engine_ms);
    the call time brackets the whole tcm_step call (budget kernel, memsets, active-count read)."""
    import torch
    times, calls, pend = [], [], []
    for rep in range(reps):
        sim.reset()
        sim.step(1)          # iteration 1: request 0 alone (its 60 s encode moves the clock past every arrival)
        sim.step(1)          # iteration 2: ingests + classifies the other requests (a1), then decides
        for _ in range(iters):
            s0 = sim.stats()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sim.step(1)
            e1.record(stream)
            stream.synchronize()
            s1 = sim.stats()
            if rep > 0:            # first repetition is warm-up
                calls.append(e0.elapsed_time(e1))
                times.append(s1["engine_ms"] - s0["engine_ms"])
                pend.append(s1["sum_pending"] - s0["sum_pending"])
    return float(np.median(times)), float(np.median(calls)), float(np.median(pend))


def bench_stepwise(args, dev, stream):
    """Paper-literal per-step kernel (k_step: a1-a5, every pending request re-keyed) on C2'
     and on a larger-window variant; the fused engine's time for the same
    iteration alongside."""
    from paper_2603_26498_b200 import tcm
    peak, peak_kind = peak_hbm()
    out = {}
    for name, R, P in (("C2'", args.step_replicas, args.step_pending), ("C2'-wide", args.step_replicas // 4, args.step_pending * 4)):
        sim = _stage_c2(R, P, tcm.ENGINE_STEPWISE, dev, stream)
        ms, call_ms, keys = time_steps(sim, stream, args.step_iters, args.step_reps)
        sim.close()
        fsim = _stage_c2(R, P, tcm.ENGINE_FUSED, dev, stream)
        fms, _, _ = time_steps(fsim, stream, args.step_iters, 2)
        fsim.close()
        bytes_per = keys * STEP_BYTES_PER_PENDING + R * STEP_BYTES_PER_DECISION
        achieved = bytes_per / (ms / 1e3) / 1e9
        out[name] = {"kernel": "k_step", "workload": f"{name}: {R} replicas x {P} pending, one iteration (a1-a5)",
                     "bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "ms_per_step": ms, "call_ms_per_step": call_ms, "keys_per_step": keys,
                     "keys_per_s": keys / (ms / 1e3), "decisions_per_s": R / (ms / 1e3),
                     "fused_engine_ms_per_step": fms}
    prof = os.path.join(ROOT, "profiles", "step_dram_bytes.json")
    if os.path.exists(prof):
        try:
            out["C2'"]["traffic"] = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            pass
    # C2: one queue with 100k pending requests, per-step latency (BASELINE.json configs[1]; SURVEY.md
    # 8(d): median of >= 1,000 repetitions, warm and L2-flushed)
    lat = {"reps": args.c2_reps}
    for eng, nm in ((tcm.ENGINE_STEPWISE, "stepwise"), (tcm.ENGINE_FUSED, "fused")):
        sim = _stage_c2(1, 100_000, eng, dev, stream)
        for flush in (False, True):
            # kernel time: eager calls (the library's events around its k_step / k_fused launch);
            # call time: the replayed CUDA graph of tcm_step(1), as a user's loop of single steps runs
            os.environ["TCM_GRAPHS"] = "0"
            r = c2_latency(sim, stream, args.c2_reps, flush, dev)
            os.environ["TCM_GRAPHS"] = "1"
            g = c2_latency(sim, stream, args.c2_reps, flush, dev)
            sfx = "_flushed" if flush else ""
            lat[nm + "_us" + sfx] = r["kernel_us"]
            lat[nm + "_p90_us" + sfx] = r["kernel_p90_us"]
            lat[nm + "_call_us" + sfx] = g["call_us"]
            lat[nm + "_graph_us" + sfx] = g["kernel_us"]
            lat[nm + "_call_us_eager" + sfx] = r["call_us"]
            lat["pending"] = r["pending"]
        os.environ.pop("TCM_GRAPHS", None)
        sim.close()
    out["C2_latency"] = lat
    return out


def c2_latency(sim, stream, reps, flush, dev):
    """Median device time of one decision on C2 (one queue, 100k pending): iteration 3 of a fresh
    reset, repeated `reps` times; with flush, a 512 MB write (> the 126 MB L2) runs on the stream
    right before the step.  Kernel time from the library's CUDA events around its launch; call time
    brackets the whole tcm_step(1) call."""
    import torch
    buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if flush else None
    ks, cs, pend = [], [], 0
    for rep in range(reps + 3):
        sim.reset()
        sim.step(1)
        sim.step(1)
        if flush:
            with torch.cuda.stream(stream):
                buf.fill_(rep & 0xFF)
        s0 = sim.stats()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.step(1)
        e1.record(stream)
        stream.synchronize()
        s1 = sim.stats()
        if rep >= 3:                               # three warm-up repetitions
            ks.append(s1["engine_ms"] - s0["engine_ms"])
            cs.append(e0.elapsed_time(e1))
            pend = s1["sum_pending"] - s0["sum_pending"]
    return {"kernel_us": float(np.median(ks)) * 1e3, "call_us": float(np.median(cs)) * 1e3,
            "kernel_p90_us": float(np.percentile(ks, 90)) * 1e3, "pending": pend}


def bench_next1(args, dev, stream, engine=None, replicas=None, requests=None, policies=None, reps=2):
    """NEXT-1 (decode KV growth + preemption by recomputation, R28-R32): the C4 grid with
    tcm.KV_GROWTH; simulated requests/s, preemptions and, per policy, the class of the victims and
    the time spent preempted (fig:preemptions).  Default: the stepwise engine at
    a reduced size with FCFS, EDF (R34 inversion preemption) and TCM cells; engine=FUSED runs k_fgrow
    (FCFS and TCM: EDF is not class-monotone)."""
    import torch
    from paper_2603_26498_b200 import tcm
    from paper_2603_26498_b200 import workloads as W
    engine = tcm.ENGINE_STEPWISE if engine is None else engine
    replicas = replicas or args.next1_replicas
    requests = requests or args.next1_requests
    policies = policies or (tcm.POLICY_FCFS, tcm.POLICY_TCM, tcm.POLICY_EDF)
    sw = W.c4_growth(replicas_per_gpu=replicas, n_requests=requests, policies=policies)
    with torch.cuda.stream(stream):
        tr = tcm.generate_device(sw.gen, device=dev, stream=stream)
        tr["params"] = torch.from_numpy(sw.params.view(np.uint8)).to(dev)
        res = tcm.alloc_results(sw.n_requests, device=dev, preemption=True)
    stream.synchronize()
    sim = tcm.Simulation(tcm.config(engine=engine, n_cells=sw.n_cells), stream)
    sim.load(tr, res)
    times = []
    for rep in range(reps):                    # the first run is warm-up
        sim.reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.run()
        e1.record(stream)
        stream.synchronize()
        times.append(e0.elapsed_time(e1))
    st = sim.stats()
    ms = times[-1]
    # per policy and class (the engine's a1 classifier, on the device): fig:preemptions
    from paper_2603_26498_b200 import metrics as M
    pst = sim.preemption_stats(device=dev).cpu().numpy()          # [cells][M, C, T, all][3]
    cell_pol = np.array([c["policy"] for c in sw.cells])
    by = {}
    for name, p in (("FCFS", tcm.POLICY_FCFS), ("EDF", tcm.POLICY_EDF), ("TCM", tcm.POLICY_TCM)):
        if p not in policies:
            continue
        summ = M.preemption_summary(pst[cell_pol == p])
        by[name] = {"preemptions": summ["all"]["preemptions"], "motorcycle_preemptions": summ["M"]["preemptions"],
                    "requests_preempted": summ["all"]["requests_preempted"],
                    "preempted_s": {g: round(summ[g]["preempted_s"], 3) for g in ("M", "C", "T")}}
    sim.close()
    names = "/".join({tcm.POLICY_FCFS: "FCFS", tcm.POLICY_TCM: "TCM", tcm.POLICY_EDF: "EDF"}[p] for p in policies)
    eng = "fused engine (k_fgrow)" if engine == tcm.ENGINE_FUSED else "stepwise engine"
    return {"workload": f"C4-growth: {sw.n_replicas} replicas x {requests} requests (C4 grid x {names}, "
                        f"KV growth + preemption by recomputation), {eng}",
            "value": sw.n_requests / (ms / 1e3), "unit": "requests/s", "ms": ms,
            "decisions_per_s": st["decisions"] / (ms / 1e3), "iterations": st["iterations"],
            "scanned_decisions": st["scanned_decisions"],
            "preemptions": st["preemptions"], "forced_preemptions": st["forced_preemptions"],
            "by_policy": by}


def host_copy(trace):
    """Pinned host copies of the device trace (the e2e leg's inputs), copied straight into pinned memory."""
    import torch
    out = {}
    for k in ("req_offset", "arrival_us", "footprint", "inline_us", "out_tokens", "modality", "params"):
        x = trace[k]
        out[k] = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        out[k].copy_(x)
    return out


def host_mem_available():
    """MemAvailable of this node in bytes (Linux), or None."""
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def bench_e2e(args, sw, host, dev, dist, world, check):
    """Same metric through the C ABI with HOST (pinned) buffers: every step copies its trace in
    (tcm_load_trace), runs (tcm_run, which copies the per-request results back) and reads the a6
    counters (tcm_stats).  Two contexts on two streams, each driven by its own host thread and
    writing its own pinned result buffers, take alternate steps, so one step's host<->device copies
    overlap the other step's kernels (a user streaming sweeps through the API does the same); the
    timed region covers every step's copies.  Afterwards both contexts' host results are compared
    with the device-resident run on a sample (`check`)."""
    import threading
    import torch
    from paper_2603_26498_b200 import tcm
    N = sw.n_requests
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    per_ctx = max(4, min(args.steps, 8) // 2)
    lanes = []
    for _ in range(2):
        res = {"admit_seq": torch.empty(N, dtype=torch.uint32).pin_memory(),
               "first_token_us": torch.empty(N, dtype=torch.uint64).pin_memory(),
               "done_us": torch.empty(N, dtype=torch.uint64).pin_memory()}
        st = torch.cuda.Stream(device=dev)
        sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells), st)
        lanes.append((sim, res, st))
    d2h = sum(v.numel() * v.element_size() for v in lanes[0][1].values())

    def step(lane):
        sim, res, st = lane
        sim.load(host, res, mem=tcm.MEM_HOST)     # H2D inside the timed region
        sim.run()                                 # results copied back (D2H) before returning
        with torch.cuda.stream(st):
            hist, cnt, _ = sim.aggregate(device=dev)
        return cnt

    for lane in lanes:                            # warm-up (allocates each context's workspace)
        step(lane)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    loaded = threading.Event()
    gpu = threading.Lock()                        # one context's engine kernels at a time
    errors = []

    def worker(k):
        try:
            torch.cuda.set_device(dev)
            if k == 1:
                loaded.wait()                     # stagger: context 1 starts once context 0 has its inputs
            for i in range(per_ctx):
                sim, res, st = lanes[k]
                sim.load(host, res, mem=tcm.MEM_HOST)
                if k == 0 and i == 0:
                    loaded.set()
                # tcm_run_async: the engine's and the a6 aggregation's kernels run alone on the GPU (the lock);
                # this context's result copy-back and next trace upload overlap the other context's kernels
                with gpu:
                    sim.run_async()
                    with torch.cuda.stream(st):
                        sim.aggregate(device=dev)   # a6 right after the engine; the copy-back is on its own stream
                sim.wait(tcm.WAIT_ALL)
        except Exception as e:                    # surfaced below
            errors.append(e)
            loaded.set()

    t0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    if errors:
        raise errors[0]
    mx = torch.tensor([wall], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    pick, ref = check
    checked = 0
    for sim, res, _ in lanes:
        for k, v in ref.items():
            got = res[k].numpy()[pick]
            if not np.array_equal(got, v):
                raise RuntimeError(f"e2e: host results ({k}) differ from the device-resident run")
            checked += len(pick)
        sim.close()
    steps = 2 * per_ctx
    total_req = N * world * steps
    return {"value": total_req / float(mx[0]), "unit": "requests/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps, "results_checked": checked,
            "note": "HOST pinned buffers through tcm_load_trace/tcm_run_async+tcm_wait/tcm_stats every step; two "
                    "contexts on two streams (own result buffers each) take alternate steps: one context's engine "
                    "kernels run alone while the other uploads its trace and copies its results back; host wall "
                    "clock, max over ranks; both contexts' results equal the device run on every 997th request"}


def log(*a):
    print(f"[bench {time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)


def main():
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("BENCH_HANG_DUMP_S", "1500")), exit=False)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["tcm", "reference"], default="tcm")
    ap.add_argument("--workload", choices=["c4", "c5", "c3", "c1"], default="c4")
    ap.add_argument("--replicas", type=int, default=None, help="replicas per GPU (C4 65,536; C5 131,072)")
    ap.add_argument("--requests", type=int, default=10_000)
    ap.add_argument("--ref-requests", type=int, default=2000, help="oracle sample: requests per replica")
    ap.add_argument("--step-replicas", type=int, default=65536)
    ap.add_argument("--step-pending", type=int, default=1024)
    ap.add_argument("--step-iters", type=int, default=4)
    ap.add_argument("--step-reps", type=int, default=3)
    ap.add_argument("--skip-step", action="store_true")
    ap.add_argument("--skip-next1", action="store_true")
    ap.add_argument("--next1-replicas", type=int, default=1536)
    ap.add_argument("--next1-requests", type=int, default=1000)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cpu-full", action="store_true",
                    help="cpu_baseline on full-length replicas (64 x 10k requests: minutes of host time)")
    ap.add_argument("--c2-reps", type=int, default=1000, help="C2 per-step latency: repetitions (median)")
    args = ap.parse_args()
    if args.replicas is None:
        args.replicas = {"c5": 131072, "c3": 4096, "c1": 1}.get(args.workload, 65536)
    if args.workload == "c1":
        args.requests = 1000
    if args.workload != "c4":
        # the C4-specific legs (e2e, stepwise C2', NEXT-1) run with the default workload only
        args.skip_e2e = args.skip_step = args.skip_next1 = True
    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)
    rank, world, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_tcm(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
