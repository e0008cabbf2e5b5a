"""initialise() phase trace (SWAMP_TRACE=1) at config 5 from pinned host
rasters, warm block cache (the e2e setting): second create in the process."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2206_05761_b200 import cases, gpu

cfg, h, qx, qy, z = cases.river_flood(L=11)
L = cfg.L
hp, qxp, qyp, zp = (gpu.pinned_copy(np.asarray(a).reshape(1 << L, 1 << L)) for a in (h, qx, qy, z))
for k in range(3):
    if k == 2:
        os.environ["SWAMP_TRACE"] = "1"
    t0 = time.perf_counter()
    e = gpu.initialise(cfg, hp, qxp, qyp, zp)
    t1 = time.perf_counter()
    print(f"create {1e3 * (t1 - t0):.3f} ms", flush=True)
    e.close()
