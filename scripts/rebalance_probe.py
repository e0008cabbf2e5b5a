"""Leaves per partition before / after rebalance for a few cases (virtual partitions on one GPU)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu
from paper_2206_05761_b200.abi import level_offset


def per_part(e, L, G):
    lv, _ = e.leaves()
    n = np.searchsorted([level_offset(k) for k in range(14)], lv, side="right") - 1
    first = (lv.astype(np.int64) - np.array([level_offset(k) for k in n])) << (2 * (L - n))
    return np.bincount(np.minimum(first * G // (4 ** L), G - 1), minlength=G)


for parts, name, kw in [(4, "river_flood", dict(L=8)), (4, "pseudo2d_dambreak", dict(L=8)),
                        (8, "monai_runup", dict(L=9)), (2, "circular_dambreak", dict(L=9))]:
    cfg, h, qx, qy, z = cases.CASES[name](**kw)
    e = gpu.initialise_partitioned(cfg, h, qx, qy, z, [0] * parts)
    e.advance(5)
    print(name, parts, "uniform-bounds leaves/partition", per_part(e, cfg.L, parts).tolist(), "moved:", e.rebalance())
