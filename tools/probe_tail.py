"""Where does the fused engine's C4 time go?  Per-cell timings, and the heaviest cell packed
32, 8 or 1 replicas per warp (empty dummy replicas fill the other lanes) (development tool)."""
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


sw = W.c4(replicas_per_gpu=int(sys.argv[1]) if len(sys.argv) > 1 else 65536)
R = sw.n_replicas
only = int(sys.argv[2]) if len(sys.argv) > 2 else -1     # skip straight to this cell's experiments
ms, st = timed(sw.gen, sw.params) if only < 0 else (0.0, {"decisions": 0, "scanned_decisions": 0})
print(f"full R={R}: {ms:.1f} ms decisions {st['decisions']:.3e} scanned {st['scanned_decisions']:.3e}", flush=True)
cells = sw.params["cell_id"]
per = []
for c in (range(sw.n_cells) if only < 0 else [only]):
    idx = np.nonzero(cells == c)[0]
    ms, st = timed(sw.gen[idx], sw.params[idx])
    d = sw.cells[c]
    per.append((ms, c))
    print(f"cell {c:2d} pol={d['policy']} lam={d['rate']} kv={d['kv']}: {ms:8.1f} ms  dec/rep {st['decisions']/len(idx):.3e}"
          f" scanned/rep {st['scanned_decisions']/len(idx):.3e}", flush=True)
per.sort(reverse=True)
c = per[0][1]
idx = np.nonzero(cells == c)[0]
for lanes in (32, 8, 1):
    gen = np.zeros(len(idx) * 32 // lanes, dtype=sw.gen.dtype)
    params = tcm.make_params(len(gen))
    dummy = T.make_replica(1, 0, 0, 1.0, (1.0, 0.0, 0.0), 131072)
    gen[:] = dummy
    pos = np.array([(k // lanes) * 32 + (k % lanes) for k in range(len(idx))])
    gen[pos] = sw.gen[idx]
    params[pos] = sw.params[idx]
    params["cell_id"] = 0
    ms, st = timed(gen, params, ncell=1)
    print(f"heaviest cell {c}, {lanes} replicas per warp ({len(gen)} slots): {ms:.1f} ms", flush=True)
for k in (1, 32):
    ms, st = timed(sw.gen[idx[:k]], sw.params[idx[:k]])
    print(f"heaviest cell {c}, first {k} replicas alone: {ms:.1f} ms", flush=True)
