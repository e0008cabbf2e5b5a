"""SWAMP_EXP_WHIST build: per-warp histograms of one config-5 FV1 (4 us bins):
tile-phase duration, per-leaf loop duration, work end after the kernel's
first start (from 20 us), and dynamic tail grabs per warp."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

cfg, h, qx, qy, z = cases.river_flood(L=11)
e = gpu.initialise(cfg, h, qx, qy, z)
e.advance(16)
for _ in range(2):
    a0 = e.debug()
    e.step_adaptive()
    a = e.debug()
    d = [a[k] - a0[k] for k in range(64)]
    print("tile  ", " ".join(f"{4*k}-{4*k+4}:{d[32+k]}" for k in range(8)))
    print("leaf  ", " ".join(f"{4*k}-{4*k+4}:{d[40+k]}" for k in range(8)))
    print("end   ", " ".join(f"{20+4*k}-{24+4*k}:{d[48+k]}" for k in range(8)))
    print("grabs ", " ".join(f"{k}:{d[56+k]}" for k in range(8)))
e.close()
