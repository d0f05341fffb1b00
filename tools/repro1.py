import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2603_26498_b200 import tcm, workloads as W
sw = W.c4(replicas_per_gpu=int(sys.argv[2]) if len(sys.argv) > 2 else 2048)
idx = np.nonzero(sw.params["cell_id"] == 17)[0][:int(sys.argv[1])]
dev = tcm.generate_device(sw.gen[idx])
dev["params"] = tcm.to_device_params(sw.params[idx])
sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=32))
sim.load(dev, None)
sim.run(); torch.cuda.synchronize()
print(sim.stats())
