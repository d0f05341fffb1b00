"""Timing probe of the stepwise engine's per-iteration kernel on C2' and C2 (development tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_26498_b200 import tcm, workloads as W

def stage(R, pending, engine):
    sw = W.c2prime(replicas=R, pending=pending)
    tr = tcm.generate_device(sw.gen)
    first = tr["req_offset"][:-1].to(torch.int64)
    tr["inline_us"].view(torch.int32)[first] = 60_000_000
    tr["modality"][first] = 1
    tr["footprint"].view(torch.int32)[first] = 800
    tr["params"] = torch.from_numpy(sw.params.view(np.uint8)).cuda()
    sim = tcm.Simulation(tcm.config(engine=engine))
    res = tcm.alloc_results(sw.n_requests)
    sim.load(tr, res)
    return sim, res

CONFIGS = [(65536, 1024), (16384, 4096), (4096, 16384), (1, 100000)]
ENGINES = (tcm.ENGINE_STEPWISE, tcm.ENGINE_FUSED)
if len(sys.argv) > 2:
    CONFIGS = [(int(sys.argv[1]), int(sys.argv[2]))]
    ENGINES = (tcm.ENGINE_STEPWISE,)
for R, pend in CONFIGS:
    for engine in ENGINES:
        sim, res = stage(R, pend, engine)
        sim.step(1)
        ts = []
        for it in range(6):
            s0 = sim.stats()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); sim.step(1); e1.record(); torch.cuda.synchronize()
            s1 = sim.stats()
            ts.append((s1["engine_ms"] - s0["engine_ms"], s1["sum_pending"] - s0["sum_pending"], s1["decisions"] - s0["decisions"], e0.elapsed_time(e1)))
        ms = np.mean([t[0] for t in ts[1:]]); cms = np.mean([t[3] for t in ts[1:]]); keys = np.mean([t[1] for t in ts[1:]])
        gbs = keys * 9 / (ms / 1e3) / 1e9
        print(f"R={R} pending={pend} engine={'stepwise' if engine else 'fused'} kernel ms/iter={ms:.4f} (call {cms:.4f}) keys/iter={keys:.0f} eqv GB/s={gbs:.1f} ({gbs/6540.8*100:.1f}% HBM)", [round(t[0], 3) for t in ts], flush=True)
        # compare engines' results after 7 iterations
        if len(ENGINES) == 1:
            pass
        elif engine == tcm.ENGINE_STEPWISE:
            ref = {k: v.clone() for k, v in res.items()}
        else:
            same = all(torch.equal(ref[k], res[k]) for k in ref)
            print("  engines identical after 7 iterations:", same, flush=True)
        sim.close()
