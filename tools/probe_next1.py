"""Timing probe of the NEXT-1 (KV growth + preemption) C4 sweep (development tool).
usage: python tools/probe_next1.py replicas requests [fused|stepwise]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2603_26498_b200 import tcm, workloads as W

R, n = int(sys.argv[1]), int(sys.argv[2])
eng = tcm.ENGINE_FUSED if (len(sys.argv) > 3 and sys.argv[3] == "fused") else tcm.ENGINE_STEPWISE
pols = (tcm.POLICY_FCFS, tcm.POLICY_TCM) if eng == tcm.ENGINE_FUSED else (tcm.POLICY_FCFS, tcm.POLICY_TCM, tcm.POLICY_EDF)
for growth in (True, False):
    sw = W.c4_growth(replicas_per_gpu=R, n_requests=n, policies=pols)
    if not growth:
        sw.params["flags"] = 0
    tr = tcm.generate_device(sw.gen)
    tr["params"] = torch.from_numpy(sw.params.view(np.uint8)).cuda()
    res = tcm.alloc_results(sw.n_requests, preemption=True)
    sim = tcm.Simulation(tcm.config(engine=eng, n_cells=sw.n_cells))
    sim.load(tr, res)
    for rep in range(2):
        sim.reset()
        torch.cuda.synchronize()
        t0 = time.time()
        sim.run()
        torch.cuda.synchronize()
        dt = time.time() - t0
    st = sim.stats()
    pc = res["preempt_count"].cpu().numpy()
    print(f"{'fused' if eng == tcm.ENGINE_FUSED else 'stepwise'} growth={growth} R={R} n={n}: {dt*1e3:.1f} ms, {sw.n_requests/dt:.3e} req/s, "
          f"decisions {st['decisions']:.3e} ({st['decisions']/dt:.3e}/s), iterations {st['iterations']}, "
          f"launches {st['kernel_launches']}, preemptions {st['preemptions']} forced {st['forced_preemptions']}, "
          f"requests preempted {(pc > 0).sum()}, engine_ms {st['engine_ms']:.1f}", flush=True)
    sim.close()
