import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, tracegen as T
from paper_2603_26498_b200 import tcm
reps = np.array([T.make_replica(77, r, 300, 2.0, (0.5, 0.2, 0.3), 32768) for r in range(3)])
tr = T.generate(reps)
params = tcm.make_params(3, kv_capacity=32768)
params["cell_id"] = [0, 1, 0]
cfg = tcm.config(n_cells=2)
sim = tcm.Simulation(cfg)
dev = tcm.to_device(tr, params); res = tcm.alloc_results(tr.n_requests)
sim.load(dev, res); sim.run()
out = {k: v.cpu().numpy() for k, v in res.items()}
hist, cnt, _ = sim.aggregate()
hist = hist.cpu().numpy(); cnt = cnt.cpu().numpy()
H = np.zeros((2, 4, 496), np.int64); C = np.zeros((2, 4, 6), np.int64)
for r in range(3):
    a, b = int(tr.offset[r]), int(tr.offset[r+1])
    rr = O.Result(out["admit_seq"][a:b], out["first_token_us"][a:b], out["done_us"][a:b], None, {}, None, 0)
    O.aggregate(tr.replica(r), rr, chunk_budget=2048, hist=H[params["cell_id"][r]], cnt=C[params["cell_id"][r]])
print("cnt gpu", cnt.tolist()); print("cnt orc", C.tolist())
print("hist sums gpu", hist.sum(-1).tolist(), "orc", H.sum(-1).tolist())
d = np.argwhere(hist != H)[:10]
for c, g, bb in d: print(c, g, bb, hist[c, g, bb], H[c, g, bb])
print("gpu nonzero bins cell0 all:", np.nonzero(hist[0,3])[0][:20], "orc:", np.nonzero(H[0,3])[0][:20])
