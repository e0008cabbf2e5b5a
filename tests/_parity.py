"""Shared helpers for GPU-vs-oracle parity checks (tests only)."""
from __future__ import annotations

import numpy as np

from paper_2206_05761_b200.abi import level_offset


def tree_mask(L: int, sig: np.ndarray) -> np.ndarray:
    """Cells on the current tree: the root and every child of a significant cell."""
    NH = level_offset(L + 1)
    m = np.zeros(NH, bool)
    m[0] = True
    for n in range(1, L + 1):
        a, b = level_offset(n), level_offset(n + 1)
        par = sig[level_offset(n - 1): level_offset(n)].astype(bool)
        m[a:b] = np.repeat(par, 4)
    return m


def compare_states(gpu, orc, what=""):
    """Bitwise comparison of leaves, descriptors, flags, tree values, t, dt."""
    gi, oi = gpu.info(), orc.info()
    assert gi["n_leaves"] == oi["n_leaves"], f"{what}: leaf count {gi['n_leaves']} vs {oi['n_leaves']}"
    assert gi["step"] == oi["step"], what
    assert gi["t"] == oi["t"], f"{what}: t {gi['t']!r} vs {oi['t']!r}"
    assert gi["dt"] == oi["dt"], f"{what}: dt {gi['dt']!r} vs {oi['dt']!r}"
    gl, gn = gpu.leaves()
    ol, on = orc.leaves()
    np.testing.assert_array_equal(gl, ol, err_msg=f"{what}: leaf list")
    np.testing.assert_array_equal(gn, on, err_msg=f"{what}: neighbour descriptors")
    (gh, gqx, gqy, gz), gsig = gpu.export_tree()
    (oh, oqx, oqy, oz), osig = orc.export_tree()
    np.testing.assert_array_equal(gsig, osig, err_msg=f"{what}: significance flags")
    m = tree_mask(gpu.L, osig)
    for name, a, b in (("h", gh, oh), ("qx", gqx, oqx), ("qy", gqy, oqy), ("z", gz, oz)):
        diff = np.flatnonzero(a[m].view(np.uint64) != b[m].view(np.uint64))
        assert diff.size == 0, (f"{what}: {name} differs on {diff.size} tree cells; first z="
                                f"{np.flatnonzero(m)[diff[0]]} gpu={a[m][diff[0]]!r} oracle={b[m][diff[0]]!r}")
