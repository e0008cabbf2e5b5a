"""Per-step leaf classes of FV1 (work counters): quiet (dry shortcut), tile
path, other (per-leaf gathers), for config 5 and the wet point."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

for name, mk in (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(8)
    w0 = e.work()
    e.advance(8)
    w1 = e.work()
    d = {k: (w1[k] - w0[k]) / 8 for k in w0}
    print(os.environ.get("TAG", "?").ljust(10), name, f"leaves {d['leaf_updates']:.0f} quiet {d['quiet_updates']:.0f} "
          f"tile {d['tile_updates']:.0f} other {d['leaf_updates'] - d['quiet_updates'] - d['tile_updates']:.0f}")
