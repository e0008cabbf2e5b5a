"""Per-warp durations of k_fv1's per-leaf loop (SWAMP_EXP_WARPT build): max
and mean over the warps of one step, and the loop's span."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

for name, mk in (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(8)
    a = e.debug()
    print(os.environ.get("TAG", "?"), name, f"warps {a[42]} max {a[40]/1e3:.1f} us mean {a[41]/max(1,a[42])/1e3:.1f} us",
          f"span {(a[43]-a[44])/1e3:.1f} us (accumulated over 9 steps; span meaningless)")
