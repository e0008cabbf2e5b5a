"""run(config) -> outputs: gauges by point sampling the
covering leaf, snapshots at the output times, the step-report CSV, and the
CLI's run / compare / validate commands on the GPU engine."""
import csv
import json

import numpy as np
import pytest

from paper_2206_05761_b200 import cases, io

gpu = pytest.importorskip("paper_2206_05761_b200.gpu")
pytestmark = pytest.mark.gpu


def test_gauges_sample_the_covering_leaf():
    cfg, h, qx, qy, z = cases.circular_dambreak(L=8)
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(30)
    fh, fqx, fqy = e.export_finest()  # the expansion holds the covering leaf's value in every finest cell
    rng = np.random.default_rng(0)
    xs = cfg.x0 + rng.uniform(0, cfg.width, 200)
    ys = cfg.y0 + rng.uniform(0, cfg.width, 200)
    xs[:2] = [cfg.x0, cfg.x0 + cfg.width * (1 - 1e-12)]  # domain corners
    ys[:2] = [cfg.y0, cfg.y0 + cfg.width * (1 - 1e-12)]
    g = e.sample_gauges(xs, ys)
    n = cfg.side
    i = np.floor((xs - cfg.x0) / cfg.width * n).astype(int)
    j = np.floor((ys - cfg.y0) / cfg.width * n).astype(int)
    zz = np.asarray(z).reshape(n, n)
    for k, f in enumerate((fh, fqx, fqy)):
        np.testing.assert_array_equal(g[k], f[j, i])
    assert not zz.any()  # flat bed: the leaf bed is 0 everywhere
    np.testing.assert_array_equal(g[3], fh[j, i])
    with pytest.raises(gpu.SwampError):
        e.sample_gauges([cfg.x0 - 1.0], [0.0])  # outside the domain
    assert e.sample_gauges([], []).shape == (4, 0)


def test_quiescent_gauge_is_constant(tmp_path):
    """a quiescent case gauge has a constant eta column."""
    from paper_2206_05761_b200 import runner

    cfg, h, qx, qy, z = cases.quiescent_humps(L=6, t_end=2.0)
    cfg.output_times = (1.0, 2.0)
    s = runner.run(cfg, h, qx, qy, z, str(tmp_path), gauges=[("lake", 10.0, 15.0), ("hump", 30.0, 6.0)])
    rows = list(csv.DictReader(open(tmp_path / "gauges.csv")))
    assert len(rows) == s["steps"] + 1 and float(rows[-1]["t"]) == 2.0
    eta = np.array([float(r["lake_eta"]) for r in rows])
    assert np.abs(eta - eta[0]).max() <= 1e-12, eta
    steps = list(csv.DictReader(open(tmp_path / "steps.csv")))
    assert len(steps) == s["steps"] and int(steps[-1]["step"]) == s["steps"]
    assert (tmp_path / "snap_h_t0.asc").exists() and (tmp_path / "snap_h_t1.asc").exists()
    assert (tmp_path / "snap_h_t2.asc").exists()


def test_run_to_zero_gives_initial_snapshot_only(tmp_path):
    from paper_2206_05761_b200 import runner

    cfg, h, qx, qy, z = cases.circular_dambreak(L=6, t_end=0.0)
    s = runner.run(cfg, h, qx, qy, z, str(tmp_path))  # SPEC.md:421 t_end = 0 -> initial snapshot only
    assert s["steps"] == 0 and s["snapshots"] == [f"snap_{q}_t0.asc" for q in ("h", "qx", "qy", "eta")]
    r = io.read_esri(tmp_path / "snap_h_t0.asc")
    np.testing.assert_array_equal(r.values[::-1].reshape(-1).view(np.uint64), np.asarray(h).reshape(-1).view(np.uint64))


def test_cli_run_and_compare(tmp_path, capsys):
    from paper_2206_05761_b200 import cli

    cfgf = tmp_path / "c.cfg"
    cfgf.write_text("[case]\nname = hump_dambreak\n[grid]\nL = 7\nepsilon = 1e-3\n[time]\nt_end = 1.0\n"
                    "output_times = 0.5, 1.0\n[output]\ngauges = g1 20 15\n")
    assert cli.main(["run", "--config", str(cfgf), "--out", str(tmp_path / "a")]) == 0
    assert cli.main(["run", "--config", str(cfgf), "--out", str(tmp_path / "b")]) == 0
    assert cli.main(["run", "--config", str(cfgf), "--out", str(tmp_path / "u"), "--set", "solver.kind=uniform"]) == 0
    summ = json.load(open(tmp_path / "a" / "summary.json"))
    assert summ["t"] == 1.0 and summ["config"]["grid.L"] == 7  # overrides round-trip into the report header
    capsys.readouterr()
    assert cli.main(["compare", str(tmp_path / "a"), str(tmp_path / "b")]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0] == "time,L1,Linf" and len(rows) == 4  # t = 0, 0.5, 1
    assert all(r.endswith(",0,0") for r in rows[1:])  # identical runs -> zeros
    assert cli.main(["compare", str(tmp_path / "a"), str(tmp_path / "u")]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert float(rows[-1].split(",")[1]) > 0.0


def test_cli_validate_subset():
    from paper_2206_05761_b200 import cli

    assert cli.main(["validate", "--only", "A4,A8", "--scale", "L=6"]) == 0


@pytest.mark.parametrize("L,n", [(8, 45), (11, 21)])
def test_advance_reports_equal_single_steps(L, n):
    """advance_reports (the step reports of back-to-back steps, read from the
    pinned ring as each step completes) equals n step_adaptive calls; at L = 8
    the run passes t_end (later reports repeat the final state)."""
    if L == 8:
        cfg, h, qx, qy, z = cases.pseudo2d_dambreak(L=8, t_end=0.3)
    else:
        cfg, h, qx, qy, z = cases.river_flood(L=11)
    a = gpu.initialise(cfg, h, qx, qy, z)
    b = gpu.initialise(cfg, h, qx, qy, z)
    ra = a.advance_reports(n)
    rb = [b.step_adaptive() for _ in range(n)]
    keys = ("step", "t", "dt", "dt_used", "n_leaves", "n_leaves_next", "n_near_threshold")
    assert len(ra) == n
    for k, (x, y) in enumerate(zip(ra, rb)):
        assert {q: x[q] for q in keys} == {q: y[q] for q in keys}, k
    if L == 8:
        assert ra[-1]["t"] == cfg.t_end and ra[-1]["step"] < n
    for fa, fb in zip(a.export_finest(), b.export_finest()):
        np.testing.assert_array_equal(fa.view(np.uint64), fb.view(np.uint64))
    # and again from where it stands (the ring's sequence words restart)
    assert a.advance_reports(3)[-1]["step"] == ra[-1]["step"] + (0 if L == 8 else 3)
    del a, b


def test_advance_reports_fallbacks():
    """Partitioned (virtual partitions) and uniform engines answer
    advance_reports with one synchronising step per report: the same
    reports as step_adaptive / step_uniform one at a time."""
    cfg, h, qx, qy, z = cases.circular_dambreak(L=8, t_end=1e30)
    a = gpu.initialise_partitioned(cfg, h, qx, qy, z, [0, 0])
    b = gpu.initialise_partitioned(cfg, h, qx, qy, z, [0, 0])
    ra = a.advance_reports(6)
    rb = [b.step_adaptive() for _ in range(6)]
    keys = ("step", "t", "dt", "n_leaves", "n_leaves_next", "n_near_threshold")
    assert [{k: r[k] for k in keys} for r in ra] == [{k: r[k] for k in keys} for r in rb]
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    ru = u.advance_reports(3)
    assert [r["step"] for r in ru] == [1, 2, 3]
    del a, b, u
