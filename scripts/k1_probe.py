"""Phase stamps (ctl->dbg) of the first and last CTA of K1 and K3 at L = 11."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu
cfg, h, qx, qy, z = cases.river_flood(L=11)
e = gpu.initialise(cfg, h, qx, qy, z)
for k in range(4):
    e.step_adaptive()
    a = e.debug()
    tl = e.timeline()
    for name, base in (("K1", 0), ("K3", 16)):
        t0 = min(a[base + 7], a[base + 15])
        for c in (0, 8):
            b = base + c
            print(name, "first" if c == 0 else "last ", "entry", round((a[b + 7] - t0) / 1e3, 2), "->",
                  [round((a[b + i] - a[b + 7]) / 1e3, 2) if a[b + i] else None for i in range(7)])
    print("timeline", tl)
