"""Command-line entry point: run, validate, bench, compare.

    python -m paper_2206_05761_b200.cli run --config case.cfg [--set section.key=value ...] [--out DIR]
    python -m paper_2206_05761_b200.cli validate [--only A3,A4,...] [--scale L=6]
    python -m paper_2206_05761_b200.cli bench --case pseudo2d --eps 1e-4,1e-3,1e-2 --levels 8,9,10 [--out DIR]
    python -m paper_2206_05761_b200.cli compare DIR_A DIR_B

Exit codes: 0 success, 1 validation / compare failure, 2 usage
or config error. Every command is non-interactive and reproducible from the
config + overrides. Simulation runs on the GPU engine (no CPU fallback); the
acceptance criteria that need an independent CPU oracle (A1, A2, A5, A9) are
in tests/ (test_oracle_kats.py, test_acceptance.py, test_zorder.py).
"""
from __future__ import annotations

import argparse
import csv
import glob
import json
import os
import sys
import time

import numpy as np


def _die(msg: str, code: int = 2) -> int:
    print(f"error: {msg}", file=sys.stderr)
    return code


def cmd_run(a) -> int:
    from . import config, runner

    try:
        ov = list(a.set or [])
        if a.out:
            ov.append(f"output.dir={a.out}")
        rc = config.load_config(a.config, ov)
        cfg, h, qx, qy, z = config.build_state(rc)
    except (config.ConfigError, OSError) as e:
        return _die(str(e))
    s = runner.run(cfg, h, qx, qy, z, config.out_dir(rc), gauges=rc.get("output.gauges"),
                   snapshots=rc.get("output.snapshots"), step_report=rc.get("output.step_report"),
                   gauge_every=rc.get("output.gauge_every"), solver=rc.get("solver.kind"),
                   device=rc.get("solver.device"))
    s["config"] = {k: (list(v) if isinstance(v, tuple) else v) for k, v in rc.values.items()}
    with open(os.path.join(config.out_dir(rc), "summary.json"), "w") as f:
        json.dump(s, f, indent=1)
    print(json.dumps({k: s[k] for k in ("solver", "L", "epsilon", "t", "steps", "n_leaves", "run_s")}))
    return 0


# ---- validate: the GPU-side acceptance criteria
def _a3(L):
    from . import cases, gpu

    cfg, h, qx, qy, z = cases.quiescent_humps(L=L, epsilon=1e-3, t_end=1e30)
    e = gpu.initialise(cfg, h, qx, qy, z)
    worst = 0.0
    for _ in range(2000 // 50):
        e.advance(50)
        _, qx_, qy_ = e.export_finest()
        worst = max(worst, float(np.abs(qx_).max()), float(np.abs(qy_).max()))
    return worst <= 1e-8, f"max |q| over 2000 steps = {worst:.3e} (<= 1e-8)"


def _a4(L):
    from . import cases, gpu

    cfg, h, qx, qy, z = cases.circular_dambreak(L=L, epsilon=0.0, t_end=3.5)
    cfg.output_times = (0.5, 1.0, 2.0, 3.5)
    a = gpu.initialise(cfg, h, qx, qy, z)
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    worst = 0.0
    for t in cfg.output_times:
        while a.info()["t"] < t:
            a.step_adaptive()
        while u.info()["t"] < t:
            u.step_uniform(1)
        worst = max(worst, a.compare(u)["Linf"])
    return worst <= 1e-8, f"max |h_adaptive - h_uniform| at the output times = {worst:.3e} (<= 1e-8)"


def _a6(L):
    from . import cases, gpu

    cfg, h, qx, qy, z = cases.hump_dambreak(L=max(L, 8))
    a = gpu.initialise(cfg, h, qx, qy, z)
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    out = {}
    for t in (6.0, 12.0):
        while a.info()["t"] < t:
            a.step_adaptive()
        while u.info()["t"] < t:
            u.step_uniform(1)
        out[t] = a.compare(u)["L1"]
    return out[6.0] <= 2e-3 and out[12.0] <= 4e-3, f"L1 6 s = {out[6.0]:.3e} (<= 2e-3), 12 s = {out[12.0]:.3e} (<= 4e-3)"


def _a7(L):
    from . import cases, gpu

    L = max(L, 10)
    cfg, h, qx, qy, z = cases.pseudo2d_dambreak(L=L, epsilon=1e-2, t_end=40.0)
    cfg.output_times = (2.5,)
    a = gpu.initialise(cfg, h, qx, qy, z)
    while a.info()["t"] < 2.5:
        a.step_adaptive()
    n25 = a.info()["n_leaves"]
    t0 = time.perf_counter()
    a = gpu.initialise(cfg, h, qx, qy, z)
    a.run()
    ta = time.perf_counter() - t0
    t0 = time.perf_counter()
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    u.run()
    tu = time.perf_counter() - t0
    n40 = a.info()["n_leaves"]
    ok = n40 <= 0.1 * 4 ** L and n40 < n25 and ta < tu
    return ok, f"leaves 2.5 s {n25}, 40 s {n40} (<= {0.1 * 4 ** L:.0f}); adaptive {ta:.3f} s < uniform {tu:.3f} s"


def _a8(L):
    from . import cases, gpu

    cfg, h, qx, qy, z = cases.hump_dambreak(L=L, t_end=1.0)
    outs = []
    for _ in range(2):
        e = gpu.initialise(cfg, h, qx, qy, z)
        e.run()
        outs.append([x.copy() for x in e.export_finest()])
        e.close()
    same = all(np.array_equal(x.view(np.uint64), y.view(np.uint64)) for x, y in zip(*outs))
    return same, "two runs bitwise identical" if same else "runs differ"


CRITERIA = {"A3": ("well-balancedness", _a3), "A4": ("adaptive == uniform at eps = 0", _a4),
            "A6": ("paper L1 figures", _a6), "A7": ("adaptivity pays", _a7), "A8": ("determinism", _a8)}


def cmd_validate(a) -> int:
    L = 6
    if a.scale:
        if not a.scale.startswith("L="):
            return _die("--scale takes L=<level>")
        L = int(a.scale[2:])
    only = [s.strip() for s in a.only.split(",")] if a.only else list(CRITERIA)
    bad = [s for s in only if s not in CRITERIA]
    if bad:
        return _die(f"unknown criteria {bad} (GPU-side: {', '.join(CRITERIA)})")
    fails = 0
    for k in only:
        name, fn = CRITERIA[k]
        t0 = time.perf_counter()
        ok, msg = fn(L)
        fails += 0 if ok else 1
        print(f"{k:3s} {'PASS' if ok else 'FAIL'}  {name}: {msg}  [{time.perf_counter() - t0:.1f} s]")
    return 1 if fails else 0


def cmd_bench(a) -> int:
    """Adaptive vs uniform over the {eps} x {L} matrix:
    CSV of wall times, leaf counts and the speed-up ratio."""
    from . import config, gpu

    if a.case not in config.CASES or a.case == "dem":
        return _die(f"unknown case {a.case}")
    eps = [float(x) for x in a.eps.split(",")]
    levels = [int(x) for x in a.levels.split(",")]
    os.makedirs(a.out, exist_ok=True)
    rows = []
    for L in levels:
        kw = {} if a.t_end is None else {"t_end": a.t_end}
        try:
            cfg, h, qx, qy, z = config.CASES[a.case](L=L, epsilon=0.0, **kw)
            u = gpu.initialise_uniform(cfg, h, qx, qy, z)
            t0 = time.perf_counter()
            u.run()
            tu = time.perf_counter() - t0
        except Exception as e:  # resource exhaustion: report the cell, continue
            print(f"L={L}: uniform failed: {e}", file=sys.stderr)
            continue
        for ep in eps:
            try:
                cfg, h, qx, qy, z = config.CASES[a.case](L=L, epsilon=ep, **kw)
                e = gpu.initialise(cfg, h, qx, qy, z)
                t0 = time.perf_counter()
                r = e.run()
                ta = time.perf_counter() - t0
                rows.append({"case": a.case, "L": L, "epsilon": ep, "t_end": cfg.t_end, "steps": r["step"],
                             "leaves_final": r["n_leaves_next"], "adaptive_s": ta, "uniform_s": tu,
                             "speedup": tu / ta})
                print(json.dumps(rows[-1]))
            except Exception as e:
                print(f"L={L} eps={ep}: adaptive failed: {e}", file=sys.stderr)
    with open(os.path.join(a.out, "bench.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["case", "L", "epsilon", "t_end", "steps", "leaves_final", "adaptive_s",
                                          "uniform_s", "speedup"])
        w.writeheader()
        w.writerows(rows)
    return 0


def cmd_compare(a) -> int:
    """L1 / L-infinity of the depth snapshots two run directories share."""
    from . import io

    snaps = {}
    for d in (a.a, a.b):
        if not os.path.isdir(d):
            return _die(f"{d}: not a run directory")
        snaps[d] = {os.path.basename(p): p for p in glob.glob(os.path.join(d, "snap_h_t*.asc"))}
    rc = 0
    print("time,L1,Linf")
    for name in sorted(set(snaps[a.a]) | set(snaps[a.b])):
        if name not in snaps[a.a] or name not in snaps[a.b]:
            print(f"warning: {name} missing in one run, skipped", file=sys.stderr)
            continue
        ra, rb = io.read_esri(snaps[a.a][name]), io.read_esri(snaps[a.b][name])
        if ra.values.shape != rb.values.shape or ra.cellsize != rb.cellsize:
            print(f"error: {name}: grids differ", file=sys.stderr)
            rc = 1
            continue
        act = (ra.values != ra.nodata) & (rb.values != rb.nodata)
        d = np.abs(ra.values - rb.values)[act]
        area = act.sum() * ra.cellsize ** 2
        l1 = float(d.sum() * ra.cellsize ** 2 / area) if area else 0.0
        print(f"{name[len('snap_h_t'):-4]},{l1:.17g},{float(d.max()) if d.size else 0.0:.17g}")
    return rc


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="paper_2206_05761_b200.cli", description=__doc__.split("\n\n")[0])
    sub = p.add_subparsers(dest="cmd")
    r = sub.add_parser("run", help="run one simulation from a config file")
    r.add_argument("--config", required=True)
    r.add_argument("--set", action="append", metavar="SECTION.KEY=VALUE", help="override a config key")
    r.add_argument("--out", help="output directory (= --set output.dir=...)")
    v = sub.add_parser("validate", help="GPU-side acceptance criteria (A3, A4, A6, A7, A8)")
    v.add_argument("--only", help="comma list of criteria")
    v.add_argument("--scale", help="L=<level> (default L=6)")
    b = sub.add_parser("bench", help="adaptive vs uniform over an eps x L matrix")
    b.add_argument("--case", default="pseudo2d")
    b.add_argument("--eps", default="1e-4,1e-3,1e-2")
    b.add_argument("--levels", default="8,9,10")
    b.add_argument("--t-end", type=float, default=None)
    b.add_argument("--out", default="bench_out")
    c = sub.add_parser("compare", help="L1 / Linf between two run directories")
    c.add_argument("a")
    c.add_argument("b")
    try:
        a = p.parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0) and 2
    if not a.cmd:
        p.print_usage(sys.stderr)
        return 2
    return {"run": cmd_run, "validate": cmd_validate, "bench": cmd_bench, "compare": cmd_compare}[a.cmd](a)


if __name__ == "__main__":
    sys.exit(main())
