"""Time k_fgrow (NEXT-1 on the fused engine) on the C4-growth sweep with the libtcm at TCM_LIB_PATH and
print a digest of the results, for A/B of build variants (development tool)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_26498_b200 import tcm, workloads as W

R = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
N = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
sw = W.c4_growth(replicas_per_gpu=R, n_requests=N, policies=(tcm.POLICY_FCFS, tcm.POLICY_TCM))
tr = tcm.generate_device(sw.gen)
tr["params"] = tcm.to_device_params(sw.params)
res = tcm.alloc_results(sw.n_requests, preemption=True)
sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells))
sim.load(tr, res)
ts = []
for rep in range(3):
    sim.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); sim.run(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
st = sim.stats()
h = hashlib.sha256()
for k, x in res.items():
    x = x.view(torch.int64 if x.element_size() == 8 else (torch.int32 if x.element_size() == 4 else torch.uint8)).to(torch.int64)
    w = (torch.arange(x.numel(), device=x.device, dtype=torch.int64) % 65521) + 1
    h.update(k.encode() + str(int(x.sum())).encode() + b"/" + str(int((x * w).sum())).encode())
for k in ("iterations", "decisions", "sum_pending", "requests_done", "preemptions"):
    h.update(str(st[k]).encode())
name = os.path.basename(os.environ.get("TCM_LIB_PATH", "libtcm.so"))
print(f"{name} [fgrow {R}x{N}]: run ms {['%.1f' % t for t in ts]} scanned {st['scanned_decisions']} "
      f"preemptions {st['preemptions']} digest {h.hexdigest()[:16]}", flush=True)
