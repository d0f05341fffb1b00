"""k_fused pass / window statistics per C4 cell (development tool; needs the TCM_VAR_FSTATS build:
python tools/build_variants.py FSTATS; TCM_LIB_PATH=.../libtcm_fstats.so python tools/probe_fstats.py [per_cell] [N])."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_26498_b200 import tcm, workloads as W

NAMES = ["passes", "L3", "L4", "L4c", "L5", "scans", "win>fin", "win>arr", "win>arr(q nonempty)",
         "win>L4c-halve", "L4c tries", "win iters", "scans tok0", "scans no-admit"]
per = int(sys.argv[1]) if len(sys.argv) > 1 else 64
N = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
lib = tcm.lib()
lib.tcm_dev_fstats.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()
cells = W.c4_cells()
for ci in (16, 19, 23, 27, 31, 3, 15):
    c = cells[ci]
    sw = W._grid("probe", [c], per, N, 4044, list(range(per)))
    tr = tcm.generate_device(sw.gen)
    tr["params"] = torch.from_numpy(sw.params.view(np.uint8)).cuda()
    sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED))
    sim.load(tr, tcm.alloc_results(sw.n_requests))
    lib.tcm_dev_fstats(buf, 1)
    sim.run()
    lib.tcm_dev_fstats(buf, 1)
    v = np.array(buf[:14], dtype=np.float64) / per
    pol = "TCM" if c["policy"] == tcm.POLICY_TCM else "FCFS"
    print(f"{pol} lam={c['rate']} kv={c['kv']}: " + ", ".join(f"{n} {x:.0f}" for n, x in zip(NAMES, v)), flush=True)
    sim.close()
