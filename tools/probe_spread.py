"""Does spreading the heavy C4 cells over more warps (fewer replicas per warp, empty dummy replicas
in the other lanes) shorten the fused engine's run?  (development tool)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tracegen as T
from paper_2603_26498_b200 import tcm, workloads as W


def timed(gen, params, ncell=32, reps=2):
    dev = tcm.generate_device(gen)
    dev["params"] = tcm.to_device_params(params)
    sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=ncell))
    best = None
    for _ in range(reps):
        sim.load(dev, None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); sim.run(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    st = sim.stats()
    sim.close()
    return best, st


sw = W.c4(replicas_per_gpu=65536)
cells = sw.params["cell_id"]
ms, st = timed(sw.gen, sw.params)
print(f"baseline: {ms:.1f} ms", flush=True)
per = {}
for c in range(sw.n_cells):
    idx = np.nonzero(cells == c)[0][:256]
    per[c], _ = timed(sw.gen[idx], sw.params[idx])
order = sorted(per, key=lambda c: -per[c])
print("cell ms (256 replicas):", [(c, round(per[c], 1)) for c in order], flush=True)
dummy = T.make_replica(1, 0, 0, 1.0, (1.0, 0.0, 0.0), 131072)
for nheavy in (4, 8, 12):
    heavy = set(order[:nheavy])
    for lanes in (16, 8):
        gens, pars = [], []
        for c in range(sw.n_cells):
            idx = np.nonzero(cells == c)[0]
            if c in heavy:
                n = len(idx) * 32 // lanes
                g = np.zeros(n, dtype=sw.gen.dtype); g[:] = dummy
                p = tcm.make_params(n); p["cell_id"] = c
                pos = np.array([(k // lanes) * 32 + (k % lanes) for k in range(len(idx))])
                g[pos] = sw.gen[idx]; p[pos] = sw.params[idx]
            else:
                g, p = sw.gen[idx], sw.params[idx]
            gens.append(g); pars.append(p)
        ms, st = timed(np.concatenate(gens), np.concatenate(pars))
        print(f"heavy cells {nheavy} at {lanes} replicas/warp: {ms:.1f} ms", flush=True)
