"""One k_fused launch over the bench's C4 workload, for ncu application replay (development tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_26498_b200 import tcm, workloads as W

R = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
sw = W.c4(replicas_per_gpu=R)
dev = tcm.generate_device(sw.gen)
dev["params"] = tcm.to_device_params(sw.params)
sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells))
res = tcm.alloc_results(sw.n_requests)
sim.load(dev, res)
sim.run()
torch.cuda.synchronize()
print(sim.stats())
