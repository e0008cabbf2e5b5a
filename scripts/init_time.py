"""Wall time of initialise() at L=11 (e2e diagnosis)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu
cfg, h, qx, qy, z = cases.river_flood(L=11)
for k in range(3):
    t0 = time.perf_counter()
    e = gpu.initialise(cfg, h, qx, qy, z)
    t1 = time.perf_counter()
    e.advance(50)
    t2 = time.perf_counter()
    f = e.export_finest()
    t3 = time.perf_counter()
    print(f"init {1e3*(t1-t0):.1f} ms, 50 steps {1e3*(t2-t1):.1f} ms, export {1e3*(t3-t2):.1f} ms")
    del e
