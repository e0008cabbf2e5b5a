"""SWAMP_EXP_K3X build: K3 top phase 2 -> 3 split (tile listing, counts /
classification pass, 3-way scan), us after the top's entry, with stamps 2, 3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

for name, mk in (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    for _ in range(3):
        e.advance(16)
        a = e.debug()
        t0 = a[16 + 7]
        f = lambda v: round((v - t0) / 1e3, 2)
        print(name, "stamp2", f(a[18]), "tiles", f(a[32]), "counts", f(a[33]), "scan", f(a[34]), "stamp3", f(a[19]))
    e.close()
