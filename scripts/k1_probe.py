"""K1 probe stamps (ctl->dbg): per-phase globaltimer of the first and last CTA."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu
cfg, h, qx, qy, z = cases.river_flood(L=11)
e = gpu.initialise(cfg, h, qx, qy, z)
lib = gpu.lib(); lib.swamp_gpu_debug.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
for k in range(5):
    e.step_adaptive()
    a = (C.c_uint64 * 16)(); lib.swamp_gpu_debug(e._h, a)
    tl = e.timeline()
    t0 = min(a[0 + 7], a[8 + 7])
    for base in (0, 8):
        print("cta", "first" if base == 0 else "last ", "entry", round((a[base + 7] - t0) / 1e3, 2), "->",
              [round((a[base + i] - a[base + 7]) / 1e3, 2) if a[base + i] else None for i in range(6)], "K1 tl", tl[0:3])
