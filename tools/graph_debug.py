import os, sys
sys.path.insert(0, os.getcwd())
os.environ["TCM_GRAPH_DEBUG"] = "1"
import numpy as np, tracegen as T
from paper_2603_26498_b200 import tcm
from tests.test_gpu_next1 import growth_sweep
tr, params = growth_sweep(96, 500, 71)
for eng in (tcm.ENGINE_STEPWISE, tcm.ENGINE_FUSED):
    sim = tcm.Simulation(tcm.config(engine=eng))
    dev = tcm.to_device(tr, params)
    res = tcm.alloc_results(tr.n_requests, preemption=True)
    sim.load(dev, res)
    k = 0
    while sim.step(7) > 0:
        k += 1
    print("engine", eng, "steps", k, sim.stats()["requests_done"], flush=True)
    sim.close()
