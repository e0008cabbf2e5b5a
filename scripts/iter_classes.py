"""k_fv1 per-leaf loop (SWAMP_EXP_ITERT build): SM cycles per warp-iteration
by class (0 all quiet, 1 gathers only, 2 some wet physics), summed over the
warps of the run; counts and mean cycles per iteration."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

for name, mk in (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(8)
    a = e.debug()
    cls = [(a[44 + k], a[40 + k]) for k in range(3)]
    print(name, " ".join(f"class{k}: n={n} mean={c / max(1, n):.0f} cyc ({c / max(1, n) / 1965:.2f} us)" for k, (n, c) in enumerate(cls)))
