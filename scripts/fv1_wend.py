"""SWAMP_EXP_WEND build: histogram of k_fv1's warp end times (4 us bins after
the kernel's first CTA start) over one step, config 5 and the wet point."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

for name, mk in (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(16)
    for _ in range(2):
        a0 = e.debug()
        e.step_adaptive()
        a = e.debug()
        hist = [a[50 + k] - a0[50 + k] for k in range(14)]
        print(os.environ.get("TAG", "?"), name, " ".join(f"{4*k}-{4*k+4}us:{v}" for k, v in enumerate(hist) if v))
    e.close()
