"""C2 per-call latency probe (development tool): one queue with 100k pending, tcm_step(1) kernel
time vs whole-call time, eager and replayed as a CUDA graph, both engines."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_26498_b200 import tcm

dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for eng, nm in ((tcm.ENGINE_STEPWISE, "stepwise"), (tcm.ENGINE_FUSED, "fused")):
    sim = bench._stage_c2(1, 100_000, eng, dev, stream)
    for g in ("0", "1"):
        os.environ["TCM_GRAPHS"] = g
        r = bench.c2_latency(sim, stream, reps, False, dev)
        print(f"{nm} graphs={g}: kernel {r['kernel_us']:.1f} us, call {r['call_us']:.1f} us, pending {r['pending']}", flush=True)
    sim.close()
