"""Small runs of every libtcm kernel path for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).
usage: sanitize_run.py {fused|step1|step1tcm|step8|cluster|growth|edf|fgrow}  (development tool; results are also checked
against the oracle on the first replicas so a sanitizer-clean run is also a correct one)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import tracegen as T
from paper_2603_26498_b200 import tcm

mode = sys.argv[1]
R, n = (8, 300) if mode != "cluster" else (1, 3000)
if len(sys.argv) > 3:
    R, n = int(sys.argv[2]), int(sys.argv[3])
growth = mode in ("growth", "edf", "fgrow")
kv = 16384
reps = np.array([T.make_replica(7, r, n, 4.0, (0.5, 0.2, 0.3), kv - 2048 if growth else kv) for r in range(R)])
tr = T.generate(reps)
params = tcm.make_params(R, kv_capacity=kv)
params["policy"] = [tcm.POLICY_EDF if mode == "edf" else (tcm.POLICY_TCM if r % 2 or mode == "step1tcm" else tcm.POLICY_FCFS)
                    for r in range(R)]                   # step1tcm: every replica TCM -> the TCM-only k_step
if growth:
    params["flags"] = tcm.KV_GROWTH
if mode in ("step1", "step1tcm", "step8", "cluster"):
    os.environ["TCM_SW_GROUP"] = {"step1": "1", "step1tcm": "1", "step8": "8", "cluster": "cluster"}[mode]
engine = tcm.ENGINE_FUSED if mode in ("fused", "fgrow") else tcm.ENGINE_STEPWISE
dev = tcm.to_device(tr, params)
res = tcm.alloc_results(tr.n_requests, preemption=growth)
sim = tcm.Simulation(tcm.config(engine=engine))
sim.load(dev, res)
if mode == "step1tcm":          # single steps first: eager, then replayed CUDA graphs (the mapped active count)
    for _ in range(6):
        sim.step(1)
sim.run()
hist, cnt, st = sim.aggregate()
for r in range(min(R, 2)):
    a, b = int(tr.offset[r]), int(tr.offset[r + 1])
    kw = dict(policy=int(params["policy"][r]), kv_capacity=kv)
    o = O.simulate_trace_growth(tr, r, **kw) if growth else O.simulate_trace(tr, r, **kw)
    assert np.array_equal(res["first_token_us"][a:b].cpu().numpy(), o.first_token_us), (mode, r)
    assert np.array_equal(res["done_us"][a:b].cpu().numpy(), o.done_us), (mode, r)
sim.close()
print(f"{mode}: OK ({R} x {n}, requests done {st['requests_done']}, preemptions {st['preemptions']})")
