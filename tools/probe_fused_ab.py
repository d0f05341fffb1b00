"""Time k_fused on the C4 bench workload with the libtcm at TCM_LIB_PATH and print a digest of the
results, for A/B of build variants (development tool)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_26498_b200 import tcm, workloads as W

R = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
order = sys.argv[2] if len(sys.argv) > 2 else "cell"
sw = W.c4(replicas_per_gpu=R)
cells = sw.params["cell_id"].astype(np.int64)
if order != "cell":                 # permutations of the replica -> lane assignment (results are invariant)
    nc = sw.n_cells
    per = R // nc
    idx = np.arange(R).reshape(nc, per)                      # cell-major
    if order == "mix2":             # a warp = 16 FCFS replicas + 16 TCM replicas of the same (lambda, KV)
        f, t = idx[:16], idx[16:]
        perm = np.stack([f.reshape(16, per // 16, 16), t.reshape(16, per // 16, 16)], axis=2).reshape(-1)
    elif order == "mixall":         # a warp = one replica of every cell (round 1's cyclic layout)
        perm = idx.T.reshape(-1)
    elif order == "rev":            # TCM cells first
        perm = np.concatenate([idx[16:].reshape(-1), idx[:16].reshape(-1)])
    sw.gen = sw.gen[perm]
    sw.params = sw.params[perm]
dev = tcm.generate_device(sw.gen)
dev["params"] = tcm.to_device_params(sw.params)
sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells))
res = tcm.alloc_results(sw.n_requests)
ts = []
for rep in range(3):
    sim.load(dev, res)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); sim.run(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
st = sim.stats()
h = hashlib.sha256()
for k in ("admit_seq", "first_token_us", "done_us"):
    x = res[k]
    x = x.view(torch.int64 if x.element_size() == 8 else torch.int32).to(torch.int64)
    w = (torch.arange(x.numel(), device=x.device, dtype=torch.int64) % 65521) + 1
    h.update(str(int(x.sum())).encode() + b"/" + str(int((x * w).sum())).encode())
for k in ("iterations", "decisions", "sum_pending", "requests_done"):
    h.update(str(st[k]).encode())
name = os.path.basename(os.environ.get("TCM_LIB_PATH", "libtcm.so"))
print(f"{name} [{order}]: run ms {['%.1f' % t for t in ts]} engine_ms {st.get('engine_ms', 0):.1f} scanned {st['scanned_decisions']} "
      f"decisions {st['decisions']} digest {h.hexdigest()[:16]}", flush=True)
