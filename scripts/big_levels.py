import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2206_05761_b200 import cases, gpu
for L in (12, 13):
    cfg, h, qx, qy, z = cases.river_flood(L=L)
    t0 = time.time()
    a = gpu.initialise(cfg, h, qx, qy, z)
    a.advance(10)
    ia = a.info()
    fa = a.export_finest()[0]
    print(L, "single", ia, "finite", bool(np.isfinite(fa).all()), round(time.time() - t0, 1), "s", flush=True)
    if L == 12:
        b = gpu.initialise_partitioned(cfg, h, qx, qy, z, [0, 0])
        b.advance(10)
        ib = b.info()
        fb = b.export_finest()[0]
        print(L, "x2 partitions", ib, "bitwise equal finest h:", bool((fa.view(np.uint64) == fb.view(np.uint64)).all()), flush=True)
        del b
    del a
    gpu.trim_cache()
