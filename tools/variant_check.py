"""Parity quick-check of a libtcm variant (TCM_LIB_PATH): C2 single queue vs oracle, C2' stepwise vs fused."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, tracegen as T
from paper_2603_26498_b200 import tcm, workloads as W

def stage(R, pend, engine):
    sw = W.c2prime(replicas=R, pending=pend)
    tr = T.generate(sw.gen)
    W.stage_c2prime(tr)
    dev = tcm.to_device(tr, sw.params)
    res = tcm.alloc_results(tr.n_requests)
    sim = tcm.Simulation(tcm.config(engine=engine))
    sim.load(dev, res)
    return tr, sim, res

tag = os.environ.get("TCM_LIB_PATH", "default")
tr, sim, res = stage(1, 100_000, tcm.ENGINE_STEPWISE)
for _ in range(6): sim.step(1)
o = O.simulate_trace(tr, 0, policy=O.TCM, max_iters=6)
bad = int((res["admit_seq"].cpu().numpy() != o.admit_seq).sum())
sim.close()
outs = []
for e in (tcm.ENGINE_FUSED, tcm.ENGINE_STEPWISE):
    tr, sim, res = stage(4096, 1024, e)
    for _ in range(4): sim.step(1)
    outs.append(res["admit_seq"].cpu().numpy()); sim.close()
bad2 = int((outs[0] != outs[1]).sum())
print(f"{tag}: C2 admit mismatches {bad}; C2' 4096x1024 stepwise-vs-fused mismatches {bad2}", flush=True)
