"""compare on the device, and a DEM-file-driven engine
(Esri ASCII ingestion feeding the hot path)."""
import numpy as np
import pytest

from paper_2206_05761_b200 import cases, io

gpu = pytest.importorskip("paper_2206_05761_b200.gpu")
pytestmark = pytest.mark.gpu


def test_compare_identical_and_eps0_equals_uniform():
    cfg, h, qx, qy, z = cases.circular_dambreak(L=7, epsilon=0.0)
    a = gpu.initialise(cfg, h, qx, qy, z)
    b = gpu.initialise(cfg, h, qx, qy, z)
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    a.advance(20)
    b.advance(20)
    u.step_uniform(20)
    assert a.compare(b) == {"L1": 0.0, "Linf": 0.0}
    assert a.compare(u) == {"L1": 0.0, "Linf": 0.0}  # SPEC.md:432 identical runs; A4 eps = 0
    cfg2, *_ = cases.circular_dambreak(L=6)
    c = gpu.initialise(cfg2, *cases.circular_dambreak(L=6)[1:])
    with pytest.raises(gpu.SwampError):  # mismatched grids
        a.compare(c)


def test_hump_dambreak_adaptive_vs_uniform_l1():
    """PAPER §3.1 / SPEC.md:433-434: hump dam-break, adaptive eps = 1e-3 vs
    uniform at t = 6 s and 12 s: L1 of the depth 'of order' 4.6e-4 / 9.2e-4."""
    cfg, h, qx, qy, z = cases.hump_dambreak(L=8)
    a = gpu.initialise(cfg, h, qx, qy, z)
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    out = {}
    for t_stop in (6.0, 12.0):
        while a.info()["t"] < t_stop:
            a.step_adaptive()
        while u.info()["t"] < t_stop:
            u.step_uniform(1)
        assert a.info()["t"] == u.info()["t"] == t_stop  # output times are hit exactly (D13)
        out[t_stop] = a.compare(u)
    # A6: L1 <= 2e-3 at 6 s and <= 4e-3 at 12 s
    assert 0.0 < out[6.0]["L1"] <= 2e-3, out
    assert 0.0 < out[12.0]["L1"] <= 4e-3, out
    print("hump L1:", out)


def test_engine_from_esri_dem(tmp_path):
    """Config 5's DEM written as an Esri raster (top row first), read back and
    sampled onto the finest grid: the engine state equals the one built from
    the in-memory DEM, bit for bit."""
    cfg, h, qx, qy, z = cases.river_flood(L=8)
    n = 1 << cfg.L
    dx = cfg.width / n
    zz = np.asarray(z).reshape(n, n)
    io.write_esri(tmp_path / "dem.asc", io.Raster(zz[::-1].copy(), xllcorner=cfg.x0, yllcorner=cfg.y0, cellsize=dx))
    r = io.read_esri(tmp_path / "dem.asc")
    zd, ina = io.load_dem(r, cfg.L, cfg.x0, cfg.y0, cfg.width, strict=True)
    assert not ina.any()
    np.testing.assert_array_equal(zd.view(np.uint64), zz.view(np.uint64))
    a = gpu.initialise(cfg, h, qx, qy, z)
    b = gpu.initialise(cfg, h, qx, qy, zd)
    a.advance(15)
    b.advance(15)
    assert a.info() == b.info() and a.compare(b) == {"L1": 0.0, "Linf": 0.0}
    io.write_finest(tmp_path / "h.asc", b.export_finest()[0], cfg.L, cfg.x0, cfg.y0, cfg.width)
    back = io.read_esri(tmp_path / "h.asc").values[::-1]
    np.testing.assert_array_equal(back.view(np.uint64), b.export_finest()[0].view(np.uint64))


def test_A7_adaptivity_pays():
    """A7: pseudo-2D dam break, L = 10, eps = 1e-2, to 40 s:
    (a) leaves at 40 s <= 10 % of 4^L and strictly below the count at 2.5 s;
    (b) the adaptive run is faster than the uniform GPU-FV1 run (device time
    of the same simulation, both through run())."""
    import time

    cfg, h, qx, qy, z = cases.pseudo2d_dambreak(L=10, epsilon=1e-2, t_end=40.0)
    cfg.output_times = (2.5,)
    a = gpu.initialise(cfg, h, qx, qy, z)
    while a.info()["t"] < 2.5:
        a.step_adaptive()
    assert a.info()["t"] == 2.5
    n25 = a.info()["n_leaves"]
    a.close()
    gpu.initialise(cfg, h, qx, qy, z).run()  # warm: graphs, block cache
    gpu.initialise_uniform(cfg, h, qx, qy, z).step_uniform(8)
    t0 = time.perf_counter()
    a = gpu.initialise(cfg, h, qx, qy, z)
    a.run()
    ta = time.perf_counter() - t0
    t0 = time.perf_counter()
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    u.run()
    tu = time.perf_counter() - t0
    n40 = a.info()["n_leaves"]
    assert a.info()["t"] == 40.0 and u.info()["t"] == 40.0
    assert n40 <= 0.1 * 4 ** 10 and n40 < n25, (n40, n25)
    assert ta < tu, (ta, tu)
    print(f"A7: leaves 2.5 s {n25}, 40 s {n40}; adaptive {ta:.3f} s vs uniform {tu:.3f} s")
