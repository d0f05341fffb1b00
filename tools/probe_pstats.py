"""Per-cell pass statistics of k_fused on the C4 bench workload (development tool; needs the
TCM_VAR_PSTATS build variant: TCM_LIB_PATH=.../libtcm_pstats.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_26498_b200 import tcm, workloads as W

R = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
sw = W.c4(replicas_per_gpu=R)
dev = tcm.generate_device(sw.gen)
dev["params"] = tcm.to_device_params(sw.params)
sim = tcm.Simulation(tcm.config(engine=tcm.ENGINE_FUSED, n_cells=sw.n_cells))
L = tcm.lib()
L.tcm_dev_pstats.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((64, 16), np.uint64)
sim.load(dev, None)
L.tcm_dev_pstats(buf.ctypes.data, 1)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); sim.run(); e1.record(); torch.cuda.synchronize()
print(f"run {e0.elapsed_time(e1):.1f} ms", sim.stats()["scanned_decisions"])
L.tcm_dev_pstats(buf.ctypes.data, 1)
names = ["pass", "idle", "L3", "L4win", "L4c_try", "L4c_ok", "L5_try", "L5_ok", "scan", "trips", "exact", "n", "cyc",
         "maxpass", "ingest", "maxcyc"]
print("cell pol lam kv | per replica: " + " ".join(f"{n:>8s}" for n in names[:11]) + "  maxpass   Mcyc/rep  maxMcyc")
tot = buf[:32].astype(np.float64)
for c in range(sw.n_cells):
    d = sw.cells[c]
    n = float(buf[c, 11])
    row = buf[c].astype(np.float64)
    print(f"{c:2d} {d['policy']} {d['rate']:3.1f} {d['kv']:6d} | " + " ".join(f"{row[k]/n:8.0f}" for k in range(11))
          + f" {row[13]:8.0f} {row[12]/n/1e6:8.2f} {row[15]/1e6:8.2f}")
s = tot.sum(0)
print("all per replica: " + " ".join(f"{names[k]}={s[k]/s[11]:.0f}" for k in range(11)))
