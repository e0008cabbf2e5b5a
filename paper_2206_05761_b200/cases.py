"""Benchmark cases (BASELINE.json configs 1-5).

Each case returns (SimConfig, h, qx, qy, z): finest-level physical fields
sampled at cell centres, row-major with row j = 0 the south row
and column i = 0 the west column. Every field is deterministic (seeded); the
same arrays are fed to the GPU engine and to the CPU oracle.

Rectangular domains of the paper are embedded in squares here (SPEC.md:445
allows an enclosing square; inactive cells are a next-round item, DESIGN.md
D9), so the 1-D and closed-box cases use walls on the square's edges.
"""
from __future__ import annotations

import numpy as np

from .abi import (
    BAND_NEIGHBOURS,
    BC_INFLOW,
    BC_REFLECTIVE,
    BC_TRANSMISSIVE,
    INFLOW_DEPTH,
    INFLOW_ETA,
    SimConfig,
)


def centres(cfg: SimConfig):
    n = cfg.side
    dx = cfg.dx
    x = cfg.x0 + (np.arange(n, dtype=np.float64) + 0.5) * dx
    y = cfg.y0 + (np.arange(n, dtype=np.float64) + 0.5) * dx
    X, Y = np.meshgrid(x, y)  # X[j, i], Y[j, i]; row j = south..north
    return X, Y


def _fields(cfg, h, z):
    h = np.ascontiguousarray(h, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    zero = np.zeros_like(h)
    return cfg, h, zero.copy(), zero.copy(), z


def pseudo2d_dambreak(L=8, epsilon=1e-3, t_end=2.5, band_mode=BAND_NEIGHBOURS, hL=6.0, hR=2.0, x_dam=10.0):
    """Config 1 — pseudo-2D dam break: 6 m / 2 m at x = 10 m,
    flat, frictionless; E/W transmissive. The 50 x 25 m channel is run on the
    50 x 50 m square with reflective N/S walls (identical 1-D flow)."""
    cfg = SimConfig(L=L, epsilon=epsilon, width=50.0, t_end=t_end, band_mode=band_mode,
                    bc=(BC_TRANSMISSIVE, BC_TRANSMISSIVE, BC_REFLECTIVE, BC_REFLECTIVE),
                    name="pseudo2d_dambreak")
    X, _ = centres(cfg)
    h = np.where(X < x_dam, hL, hR)
    return _fields(cfg, h, np.zeros_like(h))


def hump_topography(X, Y, variant="smooth"):
    """Three mounds: two of peak 1 m, one of peak 3 m, conical
    (smooth), steeper cones, or rectangular blocks. Geometry is builder-defined
    (the paper does not print it); centred vertically in the 70 m square."""
    if variant == "rectangular":
        z = np.zeros_like(X)
        for (cx, cy, hw, top) in ((30.0, 26.0, 4.0, 1.0), (30.0, 44.0, 4.0, 1.0), (47.5, 35.0, 6.0, 3.0)):
            z = np.maximum(z, np.where((np.abs(X - cx) <= hw) & (np.abs(Y - cy) <= hw), top, 0.0))
        return z
    k = 2.0 if variant == "steeper" else 1.0
    m1 = 1.0 - k * np.sqrt((X - 30.0) ** 2 + (Y - 26.0) ** 2) / 8.0
    m2 = 1.0 - k * np.sqrt((X - 30.0) ** 2 + (Y - 44.0) ** 2) / 8.0
    m3 = 3.0 - k * 3.0 * np.sqrt((X - 47.5) ** 2 + (Y - 35.0) ** 2) / 10.0
    return np.maximum(0.0, np.maximum(m1, np.maximum(m2, m3)))


def quiescent_humps(L=9, epsilon=1e-3, t_end=100.0, variant="smooth", band_mode=BAND_NEIGHBOURS):
    """Config 2 — quiescent still water over three humps:
    eta = 0.875 / 1.78 / 1.95 m, closed box, wet/dry fronts on the humps."""
    eta = {"smooth": 0.875, "steeper": 1.78, "rectangular": 1.95}[variant]
    cfg = SimConfig(L=L, epsilon=epsilon, width=70.0, t_end=t_end, band_mode=band_mode,
                    bc=(BC_REFLECTIVE,) * 4, name=f"quiescent_humps_{variant}")
    X, Y = centres(cfg)
    z = hump_topography(X, Y, variant)
    h = np.maximum(0.0, eta - z)
    return _fields(cfg, h, z)


def hump_dambreak(L=8, epsilon=1e-3, t_end=12.0, band_mode=BAND_NEIGHBOURS):
    """Hump dam-break: water surface 1.875 m behind x = 16 m,
    dry downstream, n_M = 0.018, snapshots at {0, 6, 12} s."""
    cfg = SimConfig(L=L, epsilon=epsilon, width=70.0, t_end=t_end, manning=0.018, band_mode=band_mode,
                    bc=(BC_REFLECTIVE,) * 4, output_times=(6.0, 12.0), name="hump_dambreak")
    X, Y = centres(cfg)
    z = hump_topography(X, Y, "smooth")
    h = np.where(X < 16.0, np.maximum(0.0, 1.875 - z), 0.0)
    return _fields(cfg, h, z)


def circular_dambreak(L=10, epsilon=1e-3, t_end=3.5, radius=2.5, band_mode=BAND_NEIGHBOURS):
    """Config 3 — circular dam break: [-20, 20]^2 closed,
    flat, frictionless, h = 2.5 m inside r < 2.5 m, 0.5 m outside."""
    cfg = SimConfig(L=L, epsilon=epsilon, width=40.0, x0=-20.0, y0=-20.0, t_end=t_end, band_mode=band_mode,
                    bc=(BC_REFLECTIVE,) * 4, name="circular_dambreak")
    X, Y = centres(cfg)
    h = np.where(X * X + Y * Y < radius * radius, 2.5, 0.5)
    return _fields(cfg, h, np.zeros_like(h))


def _value_noise(n, octaves, seed):
    """Multi-octave value noise on an n x n grid (deterministic, seeded)."""
    rng = np.random.RandomState(seed)
    out = np.zeros((n, n))
    amp, total = 1.0, 0.0
    for o in range(octaves):
        cells = 4 << o
        g = rng.uniform(-1.0, 1.0, size=(cells + 1, cells + 1))
        t = (np.arange(n) + 0.5) / n * cells
        i0 = np.minimum(np.floor(t).astype(int), cells - 1)
        f = t - i0
        f = f * f * (3 - 2 * f)
        a = g[np.ix_(i0, i0)]
        b = g[np.ix_(i0, i0 + 1)]
        c = g[np.ix_(i0 + 1, i0)]
        d = g[np.ix_(i0 + 1, i0 + 1)]
        fy, fx = f[:, None], f[None, :]
        out += amp * ((a * (1 - fx) + b * fx) * (1 - fy) + (c * (1 - fx) + d * fx) * fy)
        total += amp
        amp *= 0.5
    return out / total


def monai_runup(L=10, epsilon=1e-3, t_end=22.5, seed=2206, band_mode=BAND_NEIGHBOURS):
    """Config 4 — Monai-valley-like runup (BASELINE.json config 4). Synthetic
    bathymetry (builder-defined, seed recorded): a 0.125 m deep basin rising to
    a beach in the east, an island, a valley notch, plus seeded noise; a
    time-varying free-surface inflow (N-wave) on the west edge; n_M = 0.01."""
    cfg = SimConfig(L=L, epsilon=epsilon, width=5.488, t_end=t_end, manning=0.01, band_mode=band_mode,
                    bc=(BC_INFLOW, BC_REFLECTIVE, BC_REFLECTIVE, BC_REFLECTIVE), inflow_mode=INFLOW_ETA,
                    name="monai_runup")
    X, Y = centres(cfg)
    W = cfg.width
    beach = np.clip((X - 3.2) / (W - 3.2), 0.0, None) ** 1.4 * 0.25
    island = 0.14 * np.exp(-((X - 3.45) ** 2 + (Y - 1.75) ** 2) / 0.04)
    valley = -0.05 * np.exp(-((Y - 2.3) ** 2) / 0.02) * (X > 4.4)
    z = -0.125 + beach + island + valley + 0.003 * _value_noise(cfg.side, 4, seed)
    h = np.maximum(0.0, 0.0 - z)
    t = np.linspace(0.0, t_end, 451)
    eta = 0.0136 * np.exp(-(((t - 10.5) / 1.1) ** 2)) - 0.006 * np.exp(-(((t - 13.0) / 1.2) ** 2))
    cfg.inflow_t, cfg.inflow_v = tuple(t), tuple(eta)
    return _fields(cfg, h, z)


def river_flood(L=11, epsilon=1e-3, t_end=1e30, seed=5, band_mode=BAND_NEIGHBOURS):
    """Config 5 — synthetic-DEM river flood at L = 11 (2048 x 2048 cells of
    5 m, W = 10240 m). A meandering valley (Gaussian cross-section, 10 m
    walls) sloping 20 m west -> east, plus 3 octaves of seeded value noise
    (0.3 m); the channel starts filled 3 m above its thalweg; a west depth
    hydrograph (2 m -> 6 m); east transmissive, N/S walls; n_M = 0.03. Timed
    with a fixed step count (t_end effectively unbounded). At L < 11 the same
    geometry is sampled on a coarser grid (same W)."""
    W = 2048 * 5.0
    cfg = SimConfig(L=L, epsilon=epsilon, width=W, t_end=t_end, manning=0.03, band_mode=band_mode,
                    bc=(BC_INFLOW, BC_TRANSMISSIVE, BC_REFLECTIVE, BC_REFLECTIVE), inflow_mode=INFLOW_DEPTH,
                    dt_fallback=0.1, name="river_flood")
    X, Y = centres(cfg)
    yc = 0.5 * W + 0.06 * W * np.sin(2.0 * np.pi * X / (0.4 * W))
    thalweg = 20.0 * (1.0 - X / W)
    z = thalweg + 10.0 * (1.0 - np.exp(-(((Y - yc) / 600.0) ** 2))) + 0.3 * _value_noise(cfg.side, 3, seed)
    h = np.maximum(0.0, (thalweg + 3.0) - z)
    t = np.array([0.0, 600.0, 3600.0, 7200.0])
    d = np.array([2.0, 4.0, 6.0, 6.0])
    cfg.inflow_t, cfg.inflow_v = tuple(t), tuple(d)
    return _fields(cfg, h, z)


def rect_domain(case, height_fraction=3.0 / 7.0, wall_z=10.0, **kw):
    """a rectangular domain (e.g. the 70 m x 30 m humps box)
    embedded in the enclosing 2^L square; finest cells above the rectangle
    are inactive (reflective walls, D16) with a wall bed and no water."""
    cfg, h, qx, qy, z = case(**kw)
    X, Y = centres(cfg)
    ina = Y >= cfg.y0 + height_fraction * cfg.width
    h = np.where(ina, 0.0, h)
    z = np.where(ina, wall_z, z)
    cfg.inactive = ina
    cfg.name += "_rect"
    return cfg, h, np.zeros_like(h), np.zeros_like(h), z


def with_nodata_block(case, frac=(0.35, 0.55, 0.3, 0.5), wall_z=200.0, **kw):
    """A DEM with a nodata block: the block's finest cells are
    inactive (D16) — an island the flow goes around."""
    cfg, h, qx, qy, z = case(**kw)
    X, Y = centres(cfg)
    x0, x1, y0, y1 = (cfg.x0 + f * cfg.width for f in frac)
    ina = (X >= x0) & (X < x1) & (Y >= y0) & (Y < y1)
    cfg.inactive = ina
    cfg.name += "_nodata"
    return cfg, np.where(ina, 0.0, h), np.where(ina, 0.0, qx), np.where(ina, 0.0, qy), np.where(ina, wall_z, z)


def threshold_lattice(L=7, epsilon=2.0 ** -3, seed=11, t_end=1e30, band_mode=BAND_NEIGHBOURS, still=False):
    """Near-threshold exercise (north star; D8): depths on a 2^-4
    lattice in [0.5, 1] and a bed on a 2^-3 lattice in [0, 1], both with
    maximum exactly 1 (s_max = 1), so with a power-of-two epsilon many
    normalised details equal the threshold eps 2^(n-L) exactly. Closed box,
    still discharge; not a physical benchmark. still=True: a lake at rest
    (h = 2 - z, s_max = 2) that the well-balanced scheme keeps unchanged, so
    the same cells stay exactly at the threshold step after step."""
    cfg = SimConfig(L=L, epsilon=epsilon, width=10.0, t_end=t_end, band_mode=band_mode,
                    bc=(BC_REFLECTIVE,) * 4, name="threshold_lattice")
    rng = np.random.default_rng(seed)
    n = cfg.side
    h = 0.5 + rng.integers(0, 9, size=(n, n)) * 2.0 ** -4
    z = rng.integers(0, 9, size=(n, n)) * 2.0 ** -3
    h[0, 0] = 1.0
    z[0, 0] = 1.0
    if still:
        z[0, 1] = 0.0
        h = 2.0 - z
    return _fields(cfg, h, z)


CASES = {
    "pseudo2d_dambreak": pseudo2d_dambreak,
    "quiescent_humps": quiescent_humps,
    "hump_dambreak": hump_dambreak,
    "circular_dambreak": circular_dambreak,
    "monai_runup": monai_runup,
    "river_flood": river_flood,
    "threshold_lattice": threshold_lattice,
}
