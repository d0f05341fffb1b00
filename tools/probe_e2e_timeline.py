"""Timeline of the e2e leg's two-context pipeline (development tool): per context and step, host
timestamps around tcm_load_trace, tcm_run (kernels + D2H) and tcm_stats, as bench.py's e2e runs them."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2603_26498_b200 import tcm, workloads as W

R = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
per_ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda:0")
sw = W.c4(replicas_per_gpu=R)
tr = tcm.generate_device(sw.gen)
tr["params"] = torch.from_numpy(sw.params.view(np.uint8)).to(dev)
host = bench.host_copy(tr)
del tr
torch.cuda.empty_cache()
N = sw.n_requests
lanes = []
for _ in range(2):
    res = {"admit_seq": torch.empty(N, dtype=torch.uint32).pin_memory(),
           "first_token_us": torch.empty(N, dtype=torch.uint64).pin_memory(),
           "done_us": torch.empty(N, dtype=torch.uint64).pin_memory()}
    st = torch.cuda.Stream(device=dev)
    sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells), st)
    sim.load(host, res, mem=tcm.MEM_HOST); sim.run()          # warm-up: allocations
    lanes.append((sim, res, st))
torch.cuda.synchronize()
T0 = time.perf_counter()
ev = []
loaded = threading.Event()
gpu = threading.Lock()
ASYNC = os.environ.get("E2E_ASYNC", "1") != "0"

def worker(k):
    torch.cuda.set_device(dev)
    if k == 1:
        loaded.wait()
    sim, res, st = lanes[k]
    for i in range(per_ctx):
        a = time.perf_counter(); sim.load(host, res, mem=tcm.MEM_HOST); b = time.perf_counter()
        if k == 0 and i == 0:
            loaded.set()
        if ASYNC:
            with gpu:
                sim.run_async()
                with torch.cuda.stream(st):
                    sim.aggregate(device=dev)
            c = time.perf_counter()
            sim.wait(tcm.WAIT_ALL)
        else:
            sim.run()
            c = time.perf_counter()
            with torch.cuda.stream(st):
                sim.aggregate(device=dev)
        d = time.perf_counter()
        ev.append((k, i, a - T0, b - T0, c - T0, d - T0))

th = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
for t in th: t.start()
for t in th: t.join()
torch.cuda.synchronize()
wall = time.perf_counter() - T0
for e in sorted(ev, key=lambda e: e[2]):
    print(f"ctx {e[0]} step {e[1]}: load {e[2]:.3f}-{e[3]:.3f}  run {e[3]:.3f}-{e[4]:.3f}  stats {e[4]:.3f}-{e[5]:.3f}")
print(f"wall {wall:.3f} s for {2 * per_ctx} steps: {2 * per_ctx * N / wall:.3e} req/s", flush=True)
