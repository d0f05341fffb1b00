"""Quick timing probe of the fused engine on device-generated sweeps (development tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tracegen as T
from paper_2603_26498_b200 import tcm

def sweep_c3(R=4096, n=10000):
    rates = np.arange(1, 17) * 0.25
    alphas = [0.0] + [2.0 ** e for e in range(-7, 8)]
    reps = []; params = tcm.make_params(R)
    for r in range(R):
        cell = r // 16
        lam = rates[cell // 16]; al = alphas[cell % 16]
        reps.append(T.make_replica(2026, r, n, lam, (0.7, 0.25, 0.05), 131072))
        params[r]["aging_alpha"] = al; params[r]["cell_id"] = cell
    return np.array(reps), params

def sweep_c4(R=65536, n=10000):
    kvs = [131072, 65536, 32768, 16384]; lams = [0.5, 1, 2, 4]
    reps = []; params = tcm.make_params(R)
    for r in range(R):
        cell = r % 32
        kv = kvs[cell % 4]; lam = lams[(cell // 4) % 4]; pol = (cell // 16) % 2
        reps.append(T.make_replica(4044, r, n, lam, (0.5, 0.2, 0.3), kv))
        params[r]["kv_capacity"] = kv; params[r]["policy"] = pol; params[r]["cell_id"] = cell
    return np.array(reps), params

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
R = int(sys.argv[2]) if len(sys.argv) > 2 else (4096 if which == "c3" else 65536)
reps, params = (sweep_c3 if which == "c3" else sweep_c4)(R)
t0 = time.time()
dev = tcm.generate_device(reps)
torch.cuda.synchronize(); print("gen s", time.time() - t0, flush=True)
dev["params"] = torch.from_numpy(params.view(np.uint8)).cuda()
ncell = int(params["cell_id"].max()) + 1
for engine in (tcm.ENGINE_FUSED,):
    sim = tcm.Simulation(tcm.config(engine=engine, n_cells=ncell))
    for rep in range(2):
        sim.load(dev, None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); t0 = time.time()
        sim.run()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        st = sim.stats()
        N = int(reps["n_requests"].sum())
        print(f"{which} R={R} engine={engine} run {ms:.1f} ms wall {time.time()-t0:.2f}s  req/s {N/ms*1e3:.3e}  dec/s {st['decisions']/ms*1e3:.3e}", st, flush=True)
    hist, cnt, _ = sim.aggregate()
    c = cnt.cpu().numpy()
    print("mean TTFT (s) per cell [M,C,T,all] first cells:", (c[:8, :, 1] / np.maximum(c[:8, :, 0], 1) / 1e6).round(3).tolist())
