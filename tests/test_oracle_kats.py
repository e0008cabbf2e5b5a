"""Known-answer tests of the CPU oracle against SPEC.md's examples and
properties (the reference ships no tests; SPEC.md's [PAPER]/[DERIVED]
examples and acceptance criteria A1, A2 are its test contract).

These pin the oracle before it is trusted as the GPU's checker.
"""
import math
import random

import numpy as np
import pytest

from oracle import oracle as O
from paper_2206_05761_b200 import cases
from paper_2206_05761_b200.abi import BC_INFLOW, BC_REFLECTIVE, BC_TRANSMISSIVE, level_offset

G = 9.80665


# ------------------------------------------------------------------ mra
def test_encode_examples():
    # SPEC.md:134-135
    c = 0.37
    s, a, b, g = O.encode4([c, c, c, c])
    assert (s, a, b, g) == (2 * c, 0.0, 0.0, 0.0)
    assert O.encode4([1, 0, 0, 0]) == [0.5, 0.5, 0.5, 0.5]


def test_decode_examples():
    # SPEC.md:152-153
    assert O.decode4([0.5, 0.5, 0.5, 0.5]) == [1.0, 0.0, 0.0, 0.0]
    p = 1.234
    assert O.decode4([p, 0, 0, 0]) == [p / 2] * 4


def test_A1_perfect_reconstruction():
    """A1: 10,000 random quadruples per scale, 1e-12 relative."""
    rnd = np.random.RandomState(1)
    for scale in (1e-6, 1.0, 1e3, 1e6):
        for _ in range(10000 // 4):
            x = rnd.uniform(-1, 1, 4) * scale
            y = O.decode4(O.encode4(list(x)))
            # relative to the quadruple's magnitude: an element 1e5x smaller than
            # its siblings cannot be recovered to 1e-12 of itself in binary64
            assert np.all(np.abs(np.array(y) - x) <= 1e-12 * max(1.0, np.abs(x).max()))


def test_constant_preservation_and_zero_detail_roundtrip():
    rnd = random.Random(3)
    for _ in range(2000):
        c = rnd.uniform(-100, 100)
        assert O.encode4([c] * 4) == [2 * c, 0.0, 0.0, 0.0]
        # zero-detail decode then re-encode is exact (D1, D4)
        kids = O.decode4([c, 0.0, 0.0, 0.0])
        assert O.encode4(kids)[0] == c


def test_significance_examples():
    # SPEC.md:143-145
    assert not O.significance([0, 0, 0], 1.0, 3, 5, 1e-3)
    thr = math.ldexp(1e-3, 3 - 5)
    assert O.significance([thr, 0, 0], 1.0, 3, 5, 1e-3)          # ">=" boundary
    assert not O.significance([thr * (1 - 1e-15), 0, 0], 1.0, 3, 5, 1e-3)
    assert O.significance([0, 0, 0], 1.0, 3, 5, 0.0)              # eps = 0 flags everything
    assert not O.significance([5.0, 0, 0], 1e-13, 3, 5, 1e-3)     # s_max floor


def _morton_levels(field, L):
    """Finest raster (row j = south) -> level-L array in Morton order (i = x
    in the even bits, zorder.hpp:24-49), then every coarser level's s and
    details by the factored Haar filters (D1), in s-units, numpy float64."""
    n = 1 << L
    j, i = np.meshgrid(np.arange(n, dtype=np.uint64), np.arange(n, dtype=np.uint64), indexing="ij")
    m = np.zeros_like(i)
    for b in range(L):
        m |= ((i >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b)
        m |= ((j >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b + 1)
    s = np.empty(n * n)
    s[m.reshape(-1)] = np.asarray(field, dtype=np.float64).reshape(-1)
    out = {}
    for lev in range(L - 1, -1, -1):
        c = s.reshape(-1, 4)
        c0, c1, c2, c3 = c[:, 0], c[:, 1], c[:, 2], c[:, 3]
        a, b = c0 + c1, c2 + c3
        out[lev] = (0.5 * (a - b), 0.5 * ((c0 + c2) - (c1 + c3)), 0.5 * ((c0 + c3) - (c1 + c2)))
        s = 0.5 * (a + b)
    return out


def _near_count_numpy(fields, smax, L, eps):
    """Initialise's near-threshold count (D8), SPEC.md:124 literally:
    d_norm = max_q max|d_q| / s_max_q, |d_norm - eps 2^(n-L)| <= 1e-12 thr."""
    det = [_morton_levels(f, L) for f in fields]
    near = 0
    for n in range(L):
        dn = None
        for q, dq in enumerate(det):
            mq = np.maximum(np.maximum(np.abs(dq[n][0]), np.abs(dq[n][1])), np.abs(dq[n][2]))
            v = np.zeros_like(mq) if smax[q] < 1e-12 else mq / smax[q]
            dn = v if dn is None else np.maximum(dn, v)
        thr = math.ldexp(eps, n - L)
        near += int(np.count_nonzero(np.abs(dn - thr) <= 1e-12 * thr))
    return near


@pytest.mark.parametrize("eps", [2.0 ** -3, 2.0 ** -5, 0.0, 1e-3])
def test_near_threshold_counts_match_numpy(eps):
    """The oracle's near-threshold counts of initialise (flow and DEM) equal a
    numpy restatement of SPEC.md:124's division form on the same details."""
    cfg, h, qx, qy, z = cases.threshold_lattice(L=6, epsilon=eps)
    o = O.Oracle(cfg, h, qx, qy, z)
    got = o.near_threshold()
    smax = [float(np.max(np.abs(a))) for a in (h, qx, qy, z)]
    assert got["init"] == _near_count_numpy([h, qx, qy], smax[:3], cfg.L, eps)
    assert got["dem"] == _near_count_numpy([z], smax[3:], cfg.L, eps)
    if eps == 2.0 ** -3:
        assert got["init"] > 0 and got["dem"] > 0, "the lattice case must hit the threshold exactly"


def test_near_threshold_counts_real_cases():
    """On the analytic benchmark cases the same restatement agrees (the
    counts are typically 0 there: smooth data rarely lands within 1e-12)."""
    for name, kw in (("circular_dambreak", dict(L=8)), ("monai_runup", dict(L=7)), ("river_flood", dict(L=7))):
        cfg, h, qx, qy, z = cases.CASES[name](**kw)
        o = O.Oracle(cfg, h, qx, qy, z)
        smax = [float(np.max(np.abs(a))) for a in (h, qx, qy, z)]
        got = o.near_threshold()
        assert got["init"] == _near_count_numpy([h, qx, qy], smax[:3], cfg.L, cfg.epsilon), name
        assert got["dem"] == _near_count_numpy([z], smax[3:], cfg.L, cfg.epsilon), name


def test_threshold_monotonicity():
    """eps1 <= eps2 => significant set grows."""
    cfg, h, qx, qy, z = cases.circular_dambreak(L=7)
    prev = None
    for eps in (1e-1, 1e-2, 1e-3, 1e-4, 0.0):
        cfg.epsilon = eps
        o = O.Oracle(cfg, h, qx, qy, z)
        _, sig = o.export_tree()
        if prev is not None:
            assert np.all(sig >= prev)
        prev = sig


def test_dem_mask_examples():
    """flat bed -> empty mask; single raised cell -> its
    ancestor chain; checked through the t=0 tree with flat water."""
    cfg, h, qx, qy, z = cases.circular_dambreak(L=5)
    cfg.band_mode = 0
    h = np.full_like(h, 1.0)
    o = O.Oracle(cfg, h, qx, qy, z)
    _, sig = o.export_tree()
    assert sig.sum() == 0 and o.info()["n_leaves"] == 1
    z2 = z.copy()
    z2[9, 13] = 0.5
    o = O.Oracle(cfg, np.maximum(0, 1.0 - z2), qx, qy, z2)
    _, sig = o.export_tree()
    m = O.morton_encode(13, 9)
    expect = {level_offset(n) + (m >> (2 * (5 - n))) for n in range(5)}
    assert set(np.flatnonzero(sig)) == expect


# ------------------------------------------------------------------ traversal
def random_tree(L, rnd, p=0.45):
    sig = np.zeros(level_offset(L), np.uint8)
    sig[0] = 1 if rnd.random() < 0.95 else 0
    for n in range(1, L):
        a = level_offset(n)
        par = sig[level_offset(n - 1): a]
        kids = (rnd.random_sample(4 ** n) < p).astype(np.uint8)
        sig[a: a + 4 ** n] = kids & np.repeat(par, 4)
    return sig


def test_ptt_examples():
    # SPEC.md:233-235
    assert np.all(O.ptt(3, np.zeros(level_offset(3), np.uint8)) == 0)
    rec = O.ptt(3, np.ones(level_offset(3), np.uint8))
    assert np.array_equal(rec, level_offset(3) + np.arange(64))
    sig = np.zeros(level_offset(1), np.uint8)
    sig[0] = 1
    assert list(O.ptt(1, sig)) == [1, 2, 3, 4]


def test_L2_golden_vectors():
    """SURVEY §4 derived vectors: L=2, significant = {root, (1,1)}."""
    sig = np.zeros(level_offset(2), np.uint8)
    sig[0] = 1
    sig[level_offset(1) + 1] = 1
    rec = O.ptt(2, sig)
    assert list(rec) == [1, 1, 1, 1, 9, 10, 11, 12, 3, 3, 3, 3, 4, 4, 4, 4]
    leaves = O.compact(rec)
    assert list(leaves) == [1, 9, 10, 11, 12, 3, 4]
    B = 0xFFFFFFF0
    nb = O.neighbours(2, rec, leaves)
    expect = {  # W, E, N, S
        1: (B, 2, 3, B), 9: (1, 10, 11, B), 10: (9, B, 12, B), 11: (1, 12, 4, 9),
        12: (11, B, 4, 10), 3: (B, 4, B, 1), 4: (3, B, B, 2),
    }
    for k, z in enumerate(leaves):
        assert tuple(int(v) for v in nb[:, k]) == expect[int(z)]


def test_A2_ptt_equals_dft():
    """A2: 500 random ancestor-closed trees at L=6."""
    rnd = np.random.RandomState(11)
    for _ in range(500):
        sig = random_tree(6, rnd)
        leaves = O.compact(O.ptt(6, sig))
        dft = O.dft_leaves(6, sig)
        assert np.array_equal(leaves, dft)
        lv = np.floor(np.log2(3 * leaves.astype(np.int64) + 1)).astype(int) // 2
        assert int((4 ** (6 - lv)).sum()) == 4 ** 6  # tiling


def test_neighbour_symmetry_uniform():
    """SPEC.md:258 on a full tree: a's descriptor toward b is b and vice versa."""
    L = 4
    rec = O.ptt(L, np.ones(level_offset(L), np.uint8))
    lv = O.compact(rec)
    nb = O.neighbours(L, rec, lv)
    pos = {int(z): k for k, z in enumerate(lv)}
    opp = {0: 1, 1: 0, 2: 3, 3: 2}
    for k, z in enumerate(lv):
        for d in range(4):
            t = int(nb[d, k])
            if t < 0xFFFFFFF0:
                assert int(nb[opp[d], pos[t]]) == int(z)


# ------------------------------------------------------------------ swe
def test_flux_examples():
    # SPEC.md:301-303
    F = O.hll(1.0, 0.0, 0.0, 1.0, 0.0, 0.0)
    assert F[0] == 0.0 and F[2] == 0.0 and abs(F[1] - 0.5 * G) <= 1e-13
    assert O.hll(0.0, 0.0, 0.0, 0.0, 0.0, 0.0) == [0.0, 0.0, 0.0]
    rnd = random.Random(5)
    for _ in range(2000):  # consistency
        h, u, v = rnd.uniform(0.01, 10), rnd.uniform(-5, 5), rnd.uniform(-5, 5)
        F = O.hll(h, u, v, h, u, v)
        ex = [h * u, h * u * u + 0.5 * G * h * h, h * u * v]
        assert max(abs(a - b) for a, b in zip(F, ex)) <= 1e-13 * max(1.0, max(abs(e) for e in ex))


def test_reconstruction_examples():
    # z_L = z_R -> identity; wet beside dry higher bed -> h*_R = 0
    F, hs = O.face([1.0, 0.0, 0.0, 0.2], [0.7, 0.0, 0.0, 0.2])
    assert hs == [1.0, 0.7]
    F, hs = O.face([1.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 2.0])
    assert hs[0] == 0.0 and hs[1] == 0.0 and F == [0.0, 0.0, 0.0]


def test_lake_at_rest_cell():
    """constant eta, zero q, any bed, wet/dry -> no update."""
    rnd = random.Random(9)
    for _ in range(500):
        eta = 1.0
        zs = [rnd.uniform(-1, 1.5) for _ in range(5)]
        st = [[max(0.0, eta - z), 0.0, 0.0, z] for z in zs]
        if st[0][0] < 1e-6:
            continue
        out = O.fv1_cell(st[0], st[1:], dx=0.5, dt=0.01)
        assert abs(out[0] - st[0][0]) <= 1e-13 and abs(out[1]) <= 1e-13 and abs(out[2]) <= 1e-13


def test_spatial_operator_zero_for_uniform_flow():
    # SPEC.md:319-321
    s = [1.3, 0.4, -0.2, 0.0]
    assert O.fv1_cell(s, [s] * 4, 0.1, 0.01) == pytest.approx(s[:3], abs=1e-15)


def test_friction_example():
    # SPEC.md:328-330
    q = O.friction(1.0, 1.0, 0.0, 0.1, G, 0.018)
    assert q[0] == pytest.approx(1.0 / (1.0 + 0.1 * G * 0.018 ** 2), rel=1e-15)
    assert abs(q[0] - 0.9996823654637556) <= 2e-16
    assert O.friction(1.0, 1.0, 0.0, 0.1, G, 0.0) == [1.0, 0.0]
    assert O.friction(1.0, 0.0, 0.0, 0.1, G, 0.05) == [0.0, 0.0]
    for x in (1e-6, 0.3, 1.0, 8.0, 27.0, 1234.5):
        assert O.cbrt(x) == pytest.approx(x ** (1 / 3), rel=4e-16)


def test_cfl_examples():
    # SPEC.md:337-339; the oracle returns the CFL rate (max(|u|,|v|)+sqrt(gh))/dx
    # and dt = C / max rate (D13)
    assert 0.5 / O.cfl_cell(1.0, 0.0, 0.0, 1.0) == pytest.approx(0.5 / math.sqrt(G), rel=1e-15)
    assert abs(0.5 / O.cfl_cell(1.0, 0.0, 0.0, 1.0) - 0.15966497839052937) <= 1e-16
    assert O.cfl_cell(0.0, 0.0, 0.0, 1.0) == 0.0  # dry: no constraint
    # mixed levels: the level-L cell (smallest dx) dominates when states are equal
    assert O.cfl_cell(1.0, 0.2, 0.0, 0.25) > O.cfl_cell(1.0, 0.2, 0.0, 0.5)


def test_boundary_examples():
    # SPEC.md:346-348
    own = [2.0, 3.0, 1.0, 0.0]
    assert O.boundary(own, BC_REFLECTIVE, 0) == [2.0, -3.0, 1.0, 0.0]
    assert O.boundary(own, BC_TRANSMISSIVE, 0) == own
    g = O.boundary([1.0, 0.0, 0.0, 0.0], BC_INFLOW, 0, t=5.0, series_t=(0.0, 10.0), series_v=(1.0, 2.0))
    assert g[0] == 1.5 and g[2] == 0.0
    g = O.boundary([1.0, 0.0, 0.0, 0.0], BC_INFLOW, 0, t=50.0, series_t=(0.0, 10.0), series_v=(1.0, 2.0))
    assert g[0] == 2.0  # last value held


# ------------------------------------------------------------------ engine
def test_engine_examples():
    # SPEC.md:396-398 initial states
    cfg, h, *_ = cases.circular_dambreak(L=6)
    assert h.max() == 2.5 and h.min() == 0.5
    cfg, h, *_ = cases.pseudo2d_dambreak(L=6)
    assert h[0, 0] == 6.0 and h[0, -1] == 2.0


def test_quiescent_lake_invariant():
    """SPEC.md:405 + A3 (short): still water over the humps stays still."""
    cfg, h, qx, qy, z = cases.quiescent_humps(L=6)
    o = O.Oracle(cfg, h, qx, qy, z)
    n0 = o.info()["n_leaves"]
    o.step(200)
    _, fqx, fqy = o.export_finest()
    assert max(np.abs(fqx).max(), np.abs(fqy).max()) <= 1e-8
    assert o.info()["n_leaves"] == n0


def test_eps0_adaptive_equals_uniform_bitwise():
    """SPEC.md:406, A4: eps = 0 adaptive == uniform (bitwise here)."""
    cfg, h, qx, qy, z = cases.circular_dambreak(L=5, epsilon=0.0)
    a = O.Oracle(cfg, h, qx, qy, z)
    u = O.Oracle(cfg, h, qx, qy, z, uniform=True)
    assert a.info()["n_leaves"] == 4 ** 5
    for _ in range(30):
        a.step()
        u.step(uniform=True)
    for x, y in zip(a.export_finest(), u.export_finest()):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


def test_conservation_uniform_closed():
    """closed flat frictionless box conserves mass (uniform)."""
    cfg, h, qx, qy, z = cases.circular_dambreak(L=5)
    u = O.Oracle(cfg, h, qx, qy, z, uniform=True)
    m0 = u.export_finest()[0].sum()
    u.step(300, uniform=True)
    m1 = u.export_finest()[0].sum()
    assert abs(m1 - m0) <= 1e-10 * m0


def test_determinism_across_workers_A8():
    """A8: bitwise-identical results for worker counts 1/4/max."""
    cfg, h, qx, qy, z = cases.hump_dambreak(L=6, t_end=1.0)
    outs = []
    for nt in (1, 4, 8):
        O.set_threads(nt)
        o = O.Oracle(cfg, h, qx, qy, z)
        o.run()
        outs.append([a.view(np.uint64).copy() for a in o.export_finest()])
    O.set_threads(8)
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert np.array_equal(a, b)


def test_pseudo2d_dambreak_stoker_middle_state():
    """Config 1 sanity vs the exact Stoker middle depth (~3.6918 for 6/2)."""
    cfg, h, qx, qy, z = cases.pseudo2d_dambreak(L=7, t_end=2.5)
    o = O.Oracle(cfg, h, qx, qy, z)
    o.run()
    hf = o.export_finest()[0]
    row = hf[64]
    x = (np.arange(128) + 0.5) * cfg.dx
    mid = row[(x > 16) & (x < 22)]
    assert np.all(np.abs(mid - 3.6918) < 0.02)
