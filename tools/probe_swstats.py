"""k_step event counts per replica-iteration on C2' (development tool; needs the TCM_VAR_SWSTATS build:
python tools/build_variants.py SWSTATS; TCM_LIB_PATH=.../libtcm_swstats.so python tools/probe_swstats.py R P)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_26498_b200 import tcm, workloads as W

NAMES = ["decision iters", "passes", "chunks", "chunks taken", "refines live", "refines", "exact keys",
         "takes", "takes <=16", "entrants", "retunes", "prefills done", "nvalid"]
R = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
sw = W.c2prime(replicas=R, pending=P)
tr = tcm.generate_device(sw.gen)
first = tr["req_offset"][:-1].to(torch.int64)
tr["inline_us"].view(torch.int32)[first] = 60_000_000
tr["modality"][first] = 1
tr["footprint"].view(torch.int32)[first] = 800
tr["params"] = torch.from_numpy(sw.params.view(np.uint8)).cuda()
sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_STEPWISE))
sim.load(tr, tcm.alloc_results(sw.n_requests))
lib = tcm.lib()
lib.tcm_dev_swstats.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
sim.step(1)
sim.step(1)
lib.tcm_dev_swstats(buf, 1)
for it in range(3, 7):
    sim.step(1)
    lib.tcm_dev_swstats(buf, 1)
    v = np.array(buf[:13], dtype=np.float64)
    d = max(v[0], 1)
    print(f"iteration {it}: " + ", ".join(f"{n} {x / d:.2f}" for n, x in zip(NAMES, v)), flush=True)
