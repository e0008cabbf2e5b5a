"""k_fv1 phase durations per warp (SWAMP_EXP_PHASET build): tile phase,
quiet pass, per-leaf windows — mean and max over the warps of ONE step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_2206_05761_b200 import cases, gpu

SETS = {"big": (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))),
        "small": (("humpsL9", lambda: cases.quiescent_humps(L=9, t_end=1e30)),
                  ("p2dL8", lambda: cases.pseudo2d_dambreak(L=8, t_end=1e30)))}
for name, mk in SETS[os.environ.get("CASES", "big")]:
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(12)
    a0 = e.debug()
    e.step_adaptive()
    a = e.debug()
    n = a[47] - a0[47]
    names = ("tiles", "quiet", "per-leaf")
    out = " ".join(f"{names[k]}: mean {(a[40 + k] - a0[40 + k]) / max(1, n) / 1e3:.1f} max {a[44 + k] / 1e3:.1f} us" for k in range(3))
    print(name, f"warps {n}", out)
    e.close()
