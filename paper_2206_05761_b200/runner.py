"""run(config) -> outputs: step the GPU engine to t_end,
write a finest-grid snapshot (zero-detail expansion) at t = 0
and at every output time, gauge time series by point sampling the covering
leaf (Engine.sample_gauges), and the per-step StepReport CSV
(include/swamp_io.h). The engine already clips dt to hit every output time
exactly (D13), so the loop only watches t.

Output files in `out_dir`: snap_<name>_t<time>.asc (name = h, qx, qy, eta),
gauges.csv, steps.csv, summary.json.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np

from . import gpu, io


def _tag(t: float) -> str:
    return f"{t:.6f}".rstrip("0").rstrip(".") or "0"


def snapshot(engine, cfg, z, out_dir: str, t: float) -> list:
    h, qx, qy = engine.export_finest()
    ina = None if cfg.inactive is None else np.asarray(cfg.inactive).reshape(h.shape)
    files = []
    for name, f in (("h", h), ("qx", qx), ("qy", qy), ("eta", h + np.asarray(z).reshape(h.shape))):
        p = os.path.join(out_dir, f"snap_{name}_t{_tag(t)}.asc")
        io.write_finest(p, f, cfg.L, cfg.x0, cfg.y0, cfg.width, inactive=ina)
        files.append(p)
    return files


def run(cfg, h, qx, qy, z, out_dir: str, gauges=(), snapshots: bool = True, step_report: bool = True,
        gauge_every: int = 1, solver: str = "adaptive", device: int = 0) -> dict:
    """Drive one simulation; returns a summary (also written as summary.json)."""
    os.makedirs(out_dir, exist_ok=True)
    t0 = time.perf_counter()
    eng = (gpu.initialise_uniform if solver == "uniform" else gpu.initialise)(cfg, h, qx, qy, z, device=device)
    t_init = time.perf_counter() - t0
    gx = [g[1] for g in gauges]
    gy = [g[2] for g in gauges]
    g_times, g_vals, reports, snaps = [], [], [], []
    step_csv = os.path.join(out_dir, "steps.csv")
    if step_report:
        io.write_step_reports(step_csv, [])
    pending = [t for t in cfg.output_times if t > 0.0]
    info = eng.info()
    if snapshots:
        snaps += snapshot(eng, cfg, z, out_dir, info["t"])
    if gauges:
        g_times.append(info["t"])
        g_vals.append(eng.sample_gauges(gx, gy))
    t1 = time.perf_counter()
    steps = 0
    while info["t"] < cfg.t_end:
        r = eng.step_uniform(1) if solver == "uniform" else eng.step_adaptive()
        steps += 1
        info = {"t": r["t"], "step": r["step"]}
        if step_report:
            reports.append(r)
            if len(reports) >= 4096:
                io.write_step_reports(step_csv, reports, append=True)
                reports = []
        at_out = bool(pending) and r["t"] >= pending[0]
        while pending and r["t"] >= pending[0]:
            pending.pop(0)
        if gauges and (steps % gauge_every == 0 or at_out or r["t"] >= cfg.t_end):
            g_times.append(r["t"])
            g_vals.append(eng.sample_gauges(gx, gy))
        if snapshots and at_out:
            snaps += snapshot(eng, cfg, z, out_dir, r["t"])
        if r["dt_used"] == 0.0 and r["t"] < cfg.t_end:  # the engine stopped (t_end reached on the device)
            break
    wall = time.perf_counter() - t1
    if step_report and reports:
        io.write_step_reports(step_csv, reports, append=True)
    if gauges:
        io.write_gauges(os.path.join(out_dir, "gauges.csv"), g_times, g_vals, names=[g[0] for g in gauges])
    if snapshots and cfg.t_end not in cfg.output_times and info["t"] > 0.0:
        snaps += snapshot(eng, cfg, z, out_dir, info["t"])
    fin = eng.info()
    summary = {"solver": solver, "L": cfg.L, "epsilon": cfg.epsilon, "t": fin["t"], "steps": fin["step"],
               "n_leaves": fin["n_leaves"], "init_s": t_init, "run_s": wall,
               "near_threshold": eng.near_threshold() if solver == "adaptive" else None,
               "snapshots": [os.path.basename(p) for p in snaps]}
    eng.close()
    with open(os.path.join(out_dir, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    return summary
