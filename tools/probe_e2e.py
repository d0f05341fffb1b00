"""Phase times of the e2e leg (development tool): one context, HOST buffers, C4 workload -- host wall
time of tcm_load_trace (H2D + validation + class pack), tcm_run (kernels + D2H of the results) and
tcm_stats, plus the raw pinned-copy bandwidth both ways."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2603_26498_b200 import tcm, workloads as W

R = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
dev = torch.device("cuda:0")
sw = W.c4(replicas_per_gpu=R)
tr = tcm.generate_device(sw.gen)
tr["params"] = torch.from_numpy(sw.params.view(np.uint8)).to(dev)
host = bench.host_copy(tr)
N = sw.n_requests
res = {"admit_seq": torch.empty(N, dtype=torch.uint32).pin_memory(),
       "first_token_us": torch.empty(N, dtype=torch.uint64).pin_memory(),
       "done_us": torch.empty(N, dtype=torch.uint64).pin_memory()}
st = torch.cuda.Stream(device=dev)
sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells), st)
for rep in range(3):
    t0 = time.perf_counter(); sim.load(host, res, mem=tcm.MEM_HOST); st.synchronize(); t1 = time.perf_counter()
    sim.run(); st.synchronize(); t2 = time.perf_counter()
    with torch.cuda.stream(st):
        sim.aggregate(device=dev)
    st.synchronize(); t3 = time.perf_counter()
    s = sim.stats()
    print(f"rep {rep}: load {t1 - t0:.3f} s, run {t2 - t1:.3f} s (engine {s['engine_ms']:.0f} ms, stamp {s.get('stamp_ms', 0):.0f} ms, "
          f"reset {s.get('reset_ms', 0):.0f} ms), stats {t3 - t2:.3f} s", flush=True)
h2d = sum(v.numel() * v.element_size() for v in host.values())
d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
hbuf = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
for name, fn in (("H2D", lambda: d.copy_(hbuf, non_blocking=True)), ("D2H", lambda: hbuf.copy_(d, non_blocking=True))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(4): fn()
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{name} pinned copy: {4 / dt:.1f} GiB/s", flush=True)
print(f"bytes per step: H2D {h2d / 1e9:.2f} GB, D2H {sum(v.numel() * v.element_size() for v in res.values()) / 1e9:.2f} GB")
