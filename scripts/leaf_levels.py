"""Leaf-level histogram of config 5 (L = 11) after a few steps."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu
from paper_2206_05761_b200.abi import level_offset
cfg, h, qx, qy, z = cases.river_flood(L=11)
e = gpu.initialise(cfg, h, qx, qy, z)
e.advance(20)
lv, _ = e.leaves()
lvl = np.searchsorted([level_offset(n) for n in range(13)], lv, side="right") - 1
print("N", lv.size, "per level", {int(k): int(v) for k, v in zip(*np.unique(lvl, return_counts=True))})
fh = e.export_finest()[0]
print("wet fraction", float((fh > 1e-6).mean()))
