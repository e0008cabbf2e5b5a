#!/usr/bin/env python
"""bench.py — adaptive GPU-HWFV1 time step on B200 (BASELINE.json metric).

A "step" is one adaptive time step (Alg. 3 iteration: re-encode -> flag ->
band/closure -> decode -> traverse/compact -> FV1 -> CFL) of config 5, the
synthetic-DEM river flood at L = 11 (2048^2 finest cells), on one GPU. The
headline `value` is adapted-cell updates/s (sum over steps of the leaf count
N / device time) of K steps back to back right after W warm-up steps — the
same step window the reference arm times; `e2e` is the same metric through
the public C-ABI with host buffers (initial upload, per-step StepReport
read-back, final finest-grid export), `e2e_cold` the same in a fresh process
(no block cache, first graph instantiation).

Extra keys: per-kernel device times (a second pass of K steps, L2 flushed
before each) with each kernel's algorithmic bytes from its own work counters
(DESIGN.md §3), the ncu DRAM bytes / FP64 issue of each kernel
(profiles/ncu_kernels.json), a wet-dominated L = 11 point (Monai-like runup,
84 % wet, ~2 M leaves), the GPU-FV1 comparator (uniform solver vs adaptive,
PAPER.md:339, 361), sim runtimes of configs 1-4, and the CPU-HWFV1 oracle.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) the same L = 11 problem is split into N Morton-subtree
partitions, one per GPU and per process (strong scaling): each rank creates
its partition on its GPU, the ranks exchange CUDA IPC handles over gloo and
then read each other's arrays in place over NVLink, synchronising on the
device between phases. Each rank times its own stream with CUDA events; the
reported step time is the max over ranks.

`--impl reference` times the CPU-HWFV1 oracle (oracle/, the spec
restatement — the reference ships no engine to build) on this host's cores,
rank 0 only, over the same step window.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2206_05761_b200 import cases  # noqa: E402

METRIC = "adapted-cell updates/s (config 5 river flood, L=11, eps=1e-3)"
UNIT = "cell-updates/s"

# Algorithmic bytes per unit of each kernel's own work (FP64
# double4 cells {h, qx, qy, z}, z static so a cell write needs 24 B):
FV1_ACTIVE = 192   # own 32 + 4 neighbours x 32 + 4 neighbour flags + 4 B leaf id + 24 B write
FV1_QUIET = 60     # dry-subtree shortcut: own 32 + 4 B leaf id + 24 B write
FV1_FUSED = 25     # fused next-step re-encode of a level-(L-1) cell: 24 B write + 1 B pre flag
FV1_TILED = 56     # tile path (neighbours come from the block itself): own 32 B read + 24 B write
ENC_CELL = 120     # re-encoded cell: 4 children x 24 B read + 24 B parent write
K1_FLAG = 3        # per detail cell of the subtree levels: previous-tree flag + DEM flag read, pre flag write
K2_FLAG = 2        # per detail cell: pre flag read, final flag write
K3_FLAG = 2        # per detail cell: current + previous flag read
K3_LEAF = 4        # per leaf: u32 z-index list entry
DEC_CELL = 120     # newly significant cell: parent read + 4 children written


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_json(rel):
    try:
        with open(os.path.join(ROOT, rel)) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML
    every 0.5 ms (a back-to-back region lasts only a few ms), nvidia-smi as
    the fallback when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, [reason active flags])
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
            self._sample_nvml()  # one sample now: fall back to nvidia-smi if NVML misbehaves
        except Exception:
            self._nvml = None
            self.rows = []

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.rows.append((float(sm), float(mx), [bool(r & b) for b in bits]))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        for line in out.stdout.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            self.rows.append((float(f[0]), float(f[1]), [x.lower().startswith("active") for x in f[2:6]]))

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self._sample_nvml()
                else:
                    self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.0005 if self._nvml else 0.2)

    def __enter__(self):
        self.rows = []
        if self._nvml:
            try:
                self._sample_nvml()  # one sample at the start of the region
            except Exception:
                pass
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        sm = [r[0] for r in self.rows]
        mx = self.rows[-1][1] if self.rows else None
        reasons = sorted({nm for r in self.rows for nm, on in zip(self.NAMES, r[2]) if on})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(sm), "source": "nvml" if self._nvml else "nvidia-smi"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ CPU legs
def oracle_window(cfg, h, qx, qy, z, steps, warmup, threads=None, budget_s=None):
    """CPU-HWFV1 oracle over the step window [warmup, warmup + steps):
    updates = leaves each timed step updated (read AFTER the step: the grid
    the step adapted to and computed on). Returns (updates/s, details)."""
    from oracle import oracle as O

    used = O.set_threads(threads or os.cpu_count() or 1)
    t0 = time.perf_counter()
    o = O.Oracle(cfg, h, qx, qy, z)
    t_init = time.perf_counter() - t0
    for _ in range(warmup):
        o.step()
    upd, tt, k = 0, 0.0, 0
    while k < steps:
        a = time.perf_counter()
        o.step()
        tt += time.perf_counter() - a
        upd += o.info()["n_leaves"]
        k += 1
        if budget_s is not None and tt > budget_s:
            break
    return upd / tt, {"threads": used, "steps": k, "seconds": tt, "updates": upd, "init_s": t_init}


def reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg, h, qx, qy, z = cases.river_flood(L=args.L, epsilon=args.eps)
    v, info = oracle_window(cfg, h, qx, qy, z, args.steps, args.warmup)
    e2e = info["updates"] / (info["seconds"] + info["init_s"])
    K = info["steps"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": K,
        "warmup": args.warmup, "ms_per_step": 1e3 * info["seconds"] / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"river_flood_L{args.L}_eps{args.eps:g}", "L": args.L, "epsilon": args.eps,
                   "leaves_mean": info["updates"] / K, "finest_cells": 4 ** args.L,
                   "window": f"steps {args.warmup}..{args.warmup + K - 1} (after {args.warmup} warm-up steps)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": info["threads"], "kind": "port",
                         "sample": f"{K} timed steps after {args.warmup} warm-up of the L={args.L} case "
                                   "(oracle/ CPU-HWFV1 restatement of SPEC.md; the reference ships no engine)"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "note": "oracle initialise + timed steps"},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def kernel_bytes(w0, w1, steps, R_levels_detail):
    """Algorithmic bytes per step of each kernel from the work counters of
    `steps` steps."""
    d = {k: (w1[k] - w0[k]) / steps for k in w1}
    N = d["leaf_updates"]
    quiet = d["quiet_updates"]
    tiled = d["tile_updates"]
    active = N - quiet - tiled
    # stable quiet subtrees move no bytes: FV1 skips their
    # leaves (counted in quiet_updates) and their quads' fused re-encodes
    # (counted in fv1_reencoded); K1's skipped re-encodes likewise (counted
    # in k1_reencoded, a skipped subtree adding its cached count)
    skipped = d.get("fv1_skipped_leaves", 0.0)
    k1skip = d.get("k1_skipped_cells", 0.0)
    det = R_levels_detail
    return {
        "k_encode_step": ENC_CELL * (d["k1_reencoded"] - k1skip) + K1_FLAG * det,
        "k_band": K2_FLAG * det,
        "k_traverse": K3_FLAG * det + K3_LEAF * (N - skipped) + DEC_CELL * d["decoded"],
        "k_fv1": FV1_ACTIVE * active + FV1_QUIET * (quiet - skipped) + FV1_TILED * tiled
                 + FV1_FUSED * (d["fv1_reencoded"] - skipped / 4.0),
    }, {"leaves": N, "active_leaves": active, "quiet_leaves": quiet - skipped, "tiled_leaves": tiled,
        "skipped_leaves": skipped, "k1_skipped_cells": k1skip,
        "k1_reencoded": d["k1_reencoded"],
        "fv1_reencoded": d["fv1_reencoded"], "decoded": d["decoded"]}


STAGE_OF = {"k_encode_step": "ms_encode_flag", "k_band": "ms_band_closure", "k_traverse": "ms_decode_traverse",
            "k_fv1": "ms_fv1"}


def measure_workload(gpu, torch, eng, dev, steps, warmup, L, hbm_peak, ncu, fp64_peak, flushed=True):
    """Headline window (K steps back to back after W warm-up) + a flushed pass
    with per-kernel device times and per-kernel algorithmic bytes."""
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=torch.device("cuda", dev))
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    eng.advance(warmup)
    torch.cuda.synchronize(dev)
    u0 = eng.work()["leaf_updates"]
    with ClockSampler(dev) as clk:
        ev0.record(stream)
        eng.enqueue(steps)
        ev1.record(stream)
        ev1.synchronize()
    b2b_ms = ev0.elapsed_time(ev1)
    u1 = eng.work()["leaf_updates"]
    out = {"b2b_ms": b2b_ms, "updates": float(u1 - u0), "clocks": clk.summary()}
    if not flushed:
        return out
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    stage = {v: 0.0 for v in STAGE_OF.values()}
    dev_ms = 0.0
    w0 = {**eng.work(), **eng.skips()}
    leaves = []
    for _ in range(steps):
        flush.fill_(1)  # L2 flush (256 MiB > 126 MB L2) outside the timed interval
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        eng.enqueue(1)
        ev1.record(stream)
        ev1.synchronize()
        dev_ms += ev0.elapsed_time(ev1)
        r = eng.advance(0)  # StepReport of that step (device stage timeline)
        leaves.append(r["n_leaves"])
        for k in stage:
            stage[k] += r[k]
    w1 = {**eng.work(), **eng.skips()}
    K = steps
    det = sum(4 ** n for n in range(L - min(L, 6), L))  # detail cells of the subtree levels R..L-1
    alg, counts = kernel_bytes(w0, w1, K, det)
    per = {}
    for kname, sname in STAGE_OF.items():
        ms = stage[sname] / K
        gbs = alg[kname] / (ms * 1e-3) / 1e9 if ms > 0 else None
        ent = {"ms": ms, "alg_bytes": alg[kname], "GBps": gbs, "frac": (gbs / hbm_peak) if gbs else None}
        nk = (ncu or {}).get("kernels", {})
        src = [v for k, v in nk.items() if k.startswith(kname if kname != "k_traverse" else "k_traverse_tiles")]
        if src:
            s = src[0]
            extra = 0.0
            if kname == "k_traverse" and "k_traverse_top" in nk:
                extra = nk["k_traverse_top"]["dram_bytes"]
            db = s["dram_bytes"] + extra
            ent["dram_bytes_ncu"] = db
            ent["dram_frac_ncu"] = db / s["duration_s"] / 1e9 / hbm_peak if s["duration_s"] > 0 else None
            if fp64_peak and s.get("fp64_thread_inst_per_smsp_cycle"):
                ent["fp64_pipe_pct_ncu"] = s.get("fp64_pipe_pct_active")
        per[kname] = ent
    out.update({"flushed_ms": dev_ms / K, "stage_ms": {k: v / K for k, v in stage.items()}, "kernels": per,
                "counts": counts, "leaves": leaves})
    return out


def e2e_run(gpu, cfg, h, qx, qy, z, K, dev, rank=0, ws=1, allgather=None):
    """initialise from pinned host rasters + K steps (advance_reports: each
    step's StepReport read back as it completes) + finest export into pinned
    buffers, wall clock."""
    L = cfg.L
    hp, qxp, qyp, zp = (gpu.pinned_copy(np.asarray(a).reshape(1 << L, 1 << L)) for a in (h, qx, qy, z))
    outs = [gpu.pinned_empty((1 << L, 1 << L)) for _ in range(3)]
    t0 = time.perf_counter()
    e = (gpu.initialise_rank(cfg, hp, qxp, qyp, zp, rank, ws, dev, allgather) if ws > 1
         else gpu.initialise(cfg, hp, qxp, qyp, zp, device=dev))
    t1 = time.perf_counter()
    # every step's StepReport read back as the step completes (pinned ring;
    # no host round trip between steps)
    up = sum(r["n_leaves"] for r in e.advance_reports(K))
    t2 = time.perf_counter()
    e.export_finest(out=outs)
    t3 = time.perf_counter()
    e.close()
    nf = 4 ** L
    return {"value": up / (t3 - t0), "unit": UNIT, "h2d_bytes_per_step": 4 * nf * 8 // K,
            "d2h_bytes_per_step": (3 * nf * 8 + K * 104) // K, "seconds": t3 - t0,
            "seconds_by_phase": {"initialise": t1 - t0, "steps": t2 - t1, "export": t3 - t2}}


def e2e_cold_child(args):
    """Run in a fresh process (bench.py --e2e-cold-child): no block cache, no
    instantiated graphs; the CUDA context is created first (outside the
    timed region, as any CUDA process start does)."""
    import torch

    torch.cuda.init()
    torch.cuda.set_device(0)
    torch.empty(1, device="cuda")
    from paper_2206_05761_b200 import gpu

    cfg, h, qx, qy, z = cases.river_flood(L=args.L, epsilon=args.eps)
    r = e2e_run(gpu, cfg, h, qx, qy, z, args.steps, 0)
    print(json.dumps(r), flush=True)
    return 0


def comparator(gpu, torch, dev, steps):
    """GPU-FV1 (uniform grid) vs GPU-HWFV1 (PAPER.md:339,
    361): sim runtime of configs 1 and 3 to t_end at L = 8..11 through run(),
    and the step time of config 5 at L = 11. ratio = uniform / adaptive
    (> 1: the adaptive solver is faster)."""
    out = {}
    runs = [("pseudo2d", cases.pseudo2d_dambreak, dict(t_end=2.5), (8, 9, 10)),
            ("circular_eps1e-3", cases.circular_dambreak, dict(epsilon=1e-3), (8, 9, 10, 11))]
    for name, fn, kw, Ls in runs:
        for L in Ls:
            cfg, h, qx, qy, z = fn(L=L, **kw)
            res = {}
            for mode in ("adaptive", "uniform"):
                mk = gpu.initialise_uniform if mode == "uniform" else gpu.initialise
                mk(cfg, h, qx, qy, z, device=dev).close()  # (block cache of this shape, graphs warm)
                t0 = time.perf_counter()
                e = mk(cfg, h, qx, qy, z, device=dev)
                r = e.run()
                res[mode] = {"seconds": time.perf_counter() - t0, "steps": r["step"]}
                e.close()
            res["ratio_uniform_over_adaptive"] = res["uniform"]["seconds"] / res["adaptive"]["seconds"]
            out[f"{name}_L{L}"] = res
    # config 5 at L = 11: per-step device time of both solvers
    cfg, h, qx, qy, z = cases.river_flood(L=11)
    res = {}
    for mode in ("adaptive", "uniform"):
        e = (gpu.initialise_uniform if mode == "uniform" else gpu.initialise)(cfg, h, qx, qy, z, device=dev)
        stream = torch.cuda.ExternalStream(e.stream_ptr(), device=torch.device("cuda", dev))
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e.advance(5)
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        e.enqueue(steps)
        ev1.record(stream)
        ev1.synchronize()
        res[mode] = {"ms_per_step": ev0.elapsed_time(ev1) / steps}
        e.close()
    res["ratio_uniform_over_adaptive"] = res["uniform"]["ms_per_step"] / res["adaptive"]["ms_per_step"]
    out["river_L11_per_step"] = res
    return out


def sim_runtimes(gpu, dev):
    """Sim runtime (s) of configs 1-4 through the public API (paper metric)."""
    out = {}
    runs = [
        ("pseudo2d_L8_2.5s", cases.pseudo2d_dambreak, dict(L=8, t_end=2.5)),
        ("quiescent_humps_L9_100s", cases.quiescent_humps, dict(L=9, t_end=100.0)),
        ("circular_L10_eps1e-3_3.5s", cases.circular_dambreak, dict(L=10, epsilon=1e-3)),
        ("circular_L10_eps1e-2_3.5s", cases.circular_dambreak, dict(L=10, epsilon=1e-2)),
        ("circular_L10_eps1e-4_3.5s", cases.circular_dambreak, dict(L=10, epsilon=1e-4)),
        ("monai_L10_22.5s", cases.monai_runup, dict(L=10)),
    ]
    cfg, h, qx, qy, z = runs[0][1](**runs[0][2])  # warm-up (clocks idle after the CPU leg)
    gpu.initialise(cfg, h, qx, qy, z, device=dev).run()
    # one engine of every shape first, so each timed run takes its buffers from
    # the block cache as a long-running process would (a first cudaMalloc of a
    # shape costs 3-150 ms and would dominate the short runs)
    for L in sorted({kw["L"] for _, _, kw in runs}):
        name, fn, kw = next(r for r in runs if r[2]["L"] == L)
        cfg, h, qx, qy, z = fn(**kw)
        gpu.initialise(cfg, h, qx, qy, z, device=dev).close()
    for name, fn, kw in runs:
        cfg, h, qx, qy, z = fn(**kw)
        best = None
        for _ in range(2):  # (the faster of two whole runs: a single short run is noisy)
            t0 = time.perf_counter()
            e = gpu.initialise(cfg, h, qx, qy, z, device=dev)
            r = e.run()
            dt = time.perf_counter() - t0
            e.close()
            best = dt if best is None else min(best, dt)
        out[name] = {"seconds": best, "steps": r["step"], "final_leaves": r["n_leaves_next"], "runs": 2}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--L", type=int, default=11)
    ap.add_argument("--eps", type=float, default=1e-3)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-sims", action="store_true", help="skip the configs 1-4 runtime table and the comparator")
    ap.add_argument("--no-wet", action="store_true", help="skip the wet-dominated L = 11 point")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--e2e-cold-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--virtual-parts", type=int, default=1,
                    help="N=1 only: run the partitioned engine with this many partitions on one GPU (testing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        return reference_arm(args)
    if args.e2e_cold_child:
        return e2e_cold_child(args)

    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")  # host plumbing only: IPC blobs, barriers, max over ranks
    ndev = torch.cuda.device_count()
    dev = local % ndev  # more ranks than GPUs only when testing the multi-process path on a small box
    torch.cuda.set_device(dev)
    from paper_2206_05761_b200 import gpu
    from paper_2206_05761_b200.ranks import max_over_ranks, torch_allgather

    hbm_peak, peak_src = peaks()
    ncu = load_json("profiles/ncu_kernels.json")
    fp64 = load_json("profiles/fp64_peak.json")
    fp64_peak = fp64.get("dfma_per_s") if fp64 else None

    cfg, h, qx, qy, z = cases.river_flood(L=args.L, epsilon=args.eps)
    parallelism = "single"
    if ws > 1:
        eng = gpu.initialise_rank(cfg, h, qx, qy, z, rank, ws, dev, torch_allgather)
        parallelism = f"morton-subtree x{ws} (one process per GPU, CUDA IPC peer reads, device barriers)"
        if ws > ndev:
            parallelism += f" [oversubscribed: {ws} ranks on {ndev} GPU(s), time-sliced — not a scaling number]"
    elif args.virtual_parts > 1:
        eng = gpu.initialise_partitioned(cfg, h, qx, qy, z, [dev] * args.virtual_parts)
        parallelism = f"morton-subtree x{args.virtual_parts} virtual partitions on one GPU"
    else:
        eng = gpu.initialise(cfg, h, qx, qy, z, device=dev)
    if ws > 1:
        dist.barrier()
    m = measure_workload(gpu, torch, eng, dev, args.steps, args.warmup, args.L, hbm_peak, ncu, fp64_peak)
    K = args.steps
    dev_ms_max = max_over_ranks(m["b2b_ms"]) if ws > 1 else m["b2b_ms"]
    value = m["updates"] / (dev_ms_max * 1e-3)
    flushed_ms = max_over_ranks(m["flushed_ms"]) if ws > 1 else m["flushed_ms"]
    launches = eng.launches_per_step()  # kernel nodes of the one-step graph (5 at one partition)
    per = m["kernels"]
    dominant = max(per, key=lambda k: per[k]["ms"])
    d = per[dominant]
    near = eng.near_threshold()

    # ---- e2e through the public API with host buffers (engine buffers from
    #      the process block cache: the timed-loop engine is destroyed first)
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()  # every rank done before any rank frees memory its peers map
    eng.close()
    del eng
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    e2e = e2e_run(gpu, cfg, h, qx, qy, z, K, dev, rank, ws, torch_allgather)
    if ws > 1:
        e2e["seconds"] = max_over_ranks(e2e["seconds"])
        e2e["value"] = e2e["value"]  # (rank 0's count; every rank steps the same global leaves)
        dist.barrier()
    e2e["note"] = ("initialise from pinned host rasters (h, qx, qy, z) + K steps (advance_reports: every step's StepReport "
                   "written to pinned host memory as the step completes and read by the host) + "
                   "finest export (h, qx, qy) into pinned buffers; engine buffers from the process block cache")
    e2e_cold = None
    if rank == 0 and ws == 1:
        try:
            runs = []
            for _ in range(3):  # (fresh processes vary by 10x on host jitter: the median of three)
                r = subprocess.run([sys.executable, os.path.abspath(__file__), "--e2e-cold-child", "--steps", str(K),
                                    "--L", str(args.L), "--eps", str(args.eps)], capture_output=True, text=True,
                                   timeout=600, env={**os.environ, "CUDA_VISIBLE_DEVICES": str(dev)})
                runs.append(json.loads(r.stdout.strip().splitlines()[-1]))
            runs.sort(key=lambda x: x["seconds"])
            e2e_cold = runs[1]
            e2e_cold["seconds_all_runs"] = [x["seconds"] for x in runs]
            e2e_cold["note"] = ("same as e2e in a fresh process (median of three processes): device buffers from "
                                "cudaMalloc, graphs instantiated; the CUDA context created before the timed region")
        except Exception as ex:  # reported, never fatal
            e2e_cold = {"error": str(ex)[:200]}

    wet = None
    if rank == 0 and ws == 1 and not args.no_wet:
        wcfg, wh, wqx, wqy, wz = cases.monai_runup(L=11)
        we = gpu.initialise(wcfg, wh, wqx, wqy, wz, device=dev)
        wm = measure_workload(gpu, torch, we, dev, K, args.warmup, 11, hbm_peak, None, None)
        we.close()
        del we
        wet = {"workload": "monai_runup_L11_eps0.001 (84 % of the 4.19 M finest cells wet, ~2 M leaves)",
               "value": wm["updates"] / (wm["b2b_ms"] * 1e-3), "unit": UNIT, "ms_per_step": wm["b2b_ms"] / K,
               "ms_per_step_l2_flushed": wm["flushed_ms"], "leaves_mean": float(np.mean(wm["leaves"])),
               "stage_ms_per_step": wm["stage_ms"], "kernels": wm["kernels"], "counts": wm["counts"],
               "clocks": wm["clocks"]}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        v, info = oracle_window(cfg, h, qx, qy, z, steps=K, warmup=args.warmup, budget_s=args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": info["threads"], "kind": "port",
               "sample": f"{info['steps']} oracle steps of the same L={args.L} case after {args.warmup} warm-up "
                         f"steps (the headline's window; {info['seconds']:.1f} s CPU wall, {info['threads']} "
                         "threads)"}

    sims = comp = None
    if rank == 0 and ws == 1 and not args.no_sims:
        sims = sim_runtimes(gpu, dev)
        comp = comparator(gpu, torch, dev, K)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": args.warmup,
        "ms_per_step": dev_ms_max / K, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"river_flood_L{args.L}_eps{args.eps:g}", "L": args.L, "epsilon": args.eps,
                   "finest_cells": 4 ** args.L, "leaves_mean": float(np.mean(m["leaves"])),
                   "leaves_min": min(m["leaves"]), "leaves_max": max(m["leaves"]), "parallelism": parallelism,
                   "window": f"steps {args.warmup}..{args.warmup + K - 1} back to back (8-step graph replays)",
                   "l2": "inputs larger than L2: ~150 MB touched per step (2 x 179 MB cell buffers) > 126 MB L2; "
                         "ms_per_step_l2_flushed = the next K steps one launch each after a 256 MiB flush"},
        "ms_per_step_l2_flushed": flushed_ms,
        "mra_ms_per_step": sum(m["stage_ms"][s] for s in ("ms_encode_flag", "ms_band_closure", "ms_decode_traverse")),
        "stage_ms_per_step": m["stage_ms"],
        "kernels": per,
        "work_per_step": m["counts"],
        "work_note": ("leaves = leaf updates per step (the metric's unit); skipped_leaves of them belong to stable "
                      "dry subtrees whose update FV1 skips because the buffer it writes already holds the result "
                      "(DESIGN.md §8, bitwise-checked against the engine without the skip); they are charged no "
                      "bytes in the roofline, and k1_skipped_cells likewise for K1"),
        "near_threshold": near,
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": d["GBps"], "peak": hbm_peak, "unit": "GB/s",
                     "frac": d["frac"], "traffic": d.get("dram_bytes_ncu"), "peak_source": peak_src,
                     "alg_bytes_per_unit": {"active_leaf": FV1_ACTIVE, "quiet_leaf": FV1_QUIET,
                                            "tiled_leaf": FV1_TILED, "fused_reencode": FV1_FUSED}
                     if dominant == "k_fv1" else None,
                     "dram_frac_ncu": d.get("dram_frac_ncu"),
                     "note": "achieved = the kernel's algorithmic bytes (per-class counts of its own work, "
                             "DESIGN.md §3) / its device time; traffic = ncu DRAM bytes of one launch "
                             "(profiles/ncu_kernels.json); no step kernel is bandwidth-bound (DESIGN.md §9)"},
        "fp64": {"peak_dfma_per_s": fp64_peak, "source": "profiles/fp64_peak.json (scripts/fp64_peak.cu)",
                 "fv1_fp64_pipe_pct_ncu": per.get("k_fv1", {}).get("fp64_pipe_pct_ncu")} if fp64 else None,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_cold": e2e_cold,
        "wet_point": wet,
        "comparator_gpu_fv1": comp,
        "gpu_launches": launches * K,
        "timing": "CUDA events on the engine stream around K back-to-back steps (8-step graph replays); "
                  "leaf updates from the device counter; stage times from the kernels' %globaltimer stamps in "
                  "the flushed per-step pass",
        "clocks": m["clocks"],
        "sim_runtimes_s": sims,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
