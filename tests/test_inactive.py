"""Inactive cells (D16) in the oracle: a finest
mask; mixed cells are always refined so every leaf is wholly active or
inactive; inactive leaves keep their state and are excluded from CFL and
s_max; an active leaf's inactive neighbour is a reflective wall."""
import numpy as np

from oracle import oracle as O
from paper_2206_05761_b200 import cases
from paper_2206_05761_b200.abi import level_offset


def _leaf_levels(leaves):
    lv = np.searchsorted([level_offset(n) for n in range(14)], leaves, side="right") - 1
    return lv, leaves - np.array([level_offset(n) for n in lv])


def _finest_ranges(L, leaves):
    lv, m = _leaf_levels(leaves.astype(np.int64))
    return m << (2 * (L - lv)), (m + 1) << (2 * (L - lv))


def _morton_mask(mask):
    n = mask.shape[0]
    L = n.bit_length() - 1
    out = np.zeros(n * n, dtype=bool)
    for j in range(n):
        for i in range(n):
            out[O.morton_encode(i, j)] = mask[j, i]
    return out, L


def test_leaves_are_pure_and_inactive_state_is_kept():
    cfg, h, qx, qy, z = cases.with_nodata_block(cases.river_flood, L=6)
    o = O.Oracle(cfg, h, qx, qy, z)
    mm, L = _morton_mask(np.asarray(cfg.inactive).reshape(64, 64))
    fin0 = o.export_finest()
    for _ in range(15):
        o.step()
    leaves, _ = o.leaves()
    a, b = _finest_ranges(L, leaves)
    for lo, hi in zip(a, b):
        seg = mm[lo:hi]
        assert seg.all() or not seg.any(), "a leaf mixes active and inactive cells"
    fin = o.export_finest()
    ina = np.asarray(cfg.inactive).reshape(64, 64)
    for q in range(3):
        np.testing.assert_array_equal(fin[q][ina], fin0[q][ina])


def test_still_water_around_an_island_stays_still():
    """C-property with reflective inactive walls: a lake at rest around a
    nodata island over the humps stays at rest."""
    cfg, h, qx, qy, z = cases.with_nodata_block(cases.quiescent_humps, L=6, t_end=5.0)
    o = O.Oracle(cfg, h, qx, qy, z)
    o.run()
    fh, fqx, fqy = o.export_finest()
    act = ~np.asarray(cfg.inactive).reshape(64, 64)
    assert np.abs(fqx[act]).max() < 1e-10 and np.abs(fqy[act]).max() < 1e-10


def test_rectangular_embedding_matches_walls():
    """The 70 x 30 m humps box embedded in the 70 m square:
    the inactive half keeps its state; water never enters it."""
    cfg, h, qx, qy, z = cases.rect_domain(cases.hump_dambreak, L=6, t_end=2.0)
    o = O.Oracle(cfg, h, qx, qy, z)
    o.run()
    fh, _, _ = o.export_finest()
    ina = np.asarray(cfg.inactive).reshape(64, 64)
    assert (fh[ina] == 0.0).all() and fh[~ina].max() > 0.1
