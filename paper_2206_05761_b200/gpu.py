"""Python host binding of the C-ABI (include/swamp_gpu.h) via ctypes.

Mirrors the reference engine interface: `initialise`
returns an `Engine` (SimState owner) with `step_adaptive`, `advance`, `run`,
and exports of the LeafAssembly / hierarchy / finest-grid expansion.
`initialise_uniform` gives the GPU-FV1 comparator (`step_uniform`).

There is no CPU fallback: if libswamp_gpu.so or a CUDA device is missing,
construction raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .abi import STATUS, SimConfig, as_f64, dptr, level_offset, swamp_config, swamp_step_report, u8ptr, u32ptr

_HERE = os.path.dirname(os.path.abspath(__file__))
RANK_BLOB_BYTES = 1024  # SWAMP_RANK_BLOB_BYTES (include/swamp_gpu.h)
LIB_PATH = os.environ.get("SWAMP_GPU_LIB") or os.path.join(_HERE, "libswamp_gpu.so")
_LIB = None


def lib():
    """Load the in-tree sm_100a library (fails loudly when missing)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} missing — build it with `python -m paper_2206_05761_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        dp = C.POINTER(C.c_double)
        u32p = C.POINTER(C.c_uint32)
        i64p = C.POINTER(C.c_int64)
        rp = C.POINTER(swamp_step_report)
        L.swamp_gpu_create.argtypes = [C.POINTER(swamp_config), dp, dp, dp, dp, C.c_int, C.POINTER(P)]
        L.swamp_gpu_create_uniform.argtypes = L.swamp_gpu_create.argtypes
        L.swamp_gpu_create_partitioned.argtypes = [C.POINTER(swamp_config), dp, dp, dp, dp, C.c_int,
                                                   C.POINTER(C.c_int), C.POINTER(P)]
        L.swamp_gpu_rank_create.argtypes = [C.POINTER(swamp_config), dp, dp, dp, dp, C.c_int, C.c_int, C.c_int,
                                            C.POINTER(P), C.POINTER(C.c_uint8)]
        L.swamp_gpu_rank_connect.argtypes = [P, C.POINTER(C.c_uint8)]
        L.swamp_gpu_rank_ready.argtypes = [P]
        L.swamp_gpu_compare.argtypes = [P, P, dp, dp]
        L.swamp_gpu_rebalance.argtypes = [P, C.POINTER(C.c_int32)]
        L.swamp_gpu_destroy.argtypes = [P]
        L.swamp_gpu_trim_cache.argtypes = [C.c_int]
        L.swamp_gpu_step.argtypes = [P, rp]
        L.swamp_gpu_advance.argtypes = [P, C.c_int64, rp]
        if hasattr(L, "swamp_gpu_advance_reports"):
            L.swamp_gpu_advance_reports.argtypes = [P, C.c_int64, rp]
        L.swamp_gpu_run.argtypes = [P, rp]
        L.swamp_gpu_step_uniform.argtypes = [P, C.c_int64, rp]
        L.swamp_gpu_set_profiling.argtypes = [P, C.c_int]
        L.swamp_gpu_info.argtypes = [P, dp, dp, i64p, i64p]
        L.swamp_gpu_copy_leaves.argtypes = [P, u32p, u32p, u32p, u32p, u32p, C.c_int64, i64p]
        L.swamp_gpu_export_tree.argtypes = [P, dp, dp, dp, dp, C.POINTER(C.c_uint8)]
        L.swamp_gpu_export_finest.argtypes = [P, dp, dp, dp]
        L.swamp_gpu_last_error.argtypes = [P, C.POINTER(C.c_int32), u32p, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int32), C.c_char_p, C.c_size_t]
        L.swamp_gpu_counters.argtypes = [P, i64p]
        L.swamp_gpu_near_threshold.argtypes = [P, i64p]
        L.swamp_gpu_work_counters.argtypes = [P, i64p]
        if hasattr(L, "swamp_gpu_skip_counters"):
            L.swamp_gpu_skip_counters.argtypes = [P, i64p]
        L.swamp_gpu_enqueue.argtypes = [P, C.c_int64]
        L.swamp_gpu_timeline.argtypes = [P, dp]
        L.swamp_gpu_debug.argtypes = [P, C.POINTER(C.c_uint64)]
        L.swamp_gpu_stream.argtypes = [P, C.POINTER(C.c_void_p)]
        if hasattr(L, "swamp_gpu_sample_gauges"):  # (older builds, A/B timing only)
            L.swamp_gpu_sample_gauges.argtypes = [P, C.c_int32, dp, dp, dp]
        L.swamp_gpu_build_info.restype = C.c_char_p
        _LIB = L
    return _LIB


EXPORTED_SYMBOLS = (
    "swamp_gpu_create", "swamp_gpu_destroy", "swamp_gpu_step", "swamp_gpu_advance", "swamp_gpu_run",
    "swamp_gpu_advance_reports",
    "swamp_gpu_create_uniform", "swamp_gpu_step_uniform", "swamp_gpu_set_profiling", "swamp_gpu_info",
    "swamp_gpu_copy_leaves", "swamp_gpu_export_tree", "swamp_gpu_export_finest", "swamp_gpu_last_error",
    "swamp_gpu_counters", "swamp_gpu_build_info", "swamp_gpu_enqueue", "swamp_gpu_stream",
    "swamp_gpu_timeline", "swamp_gpu_create_partitioned", "swamp_gpu_debug",
    "swamp_gpu_rank_create", "swamp_gpu_rank_connect", "swamp_gpu_rank_ready", "swamp_gpu_compare",
    "swamp_gpu_rebalance", "swamp_gpu_trim_cache", "swamp_gpu_near_threshold", "swamp_gpu_work_counters",
    "swamp_gpu_sample_gauges", "swamp_gpu_skip_counters", "swamp_partition_plan", "swamp_partition_owner",
    "swamp_io_read_esri", "swamp_io_write_esri", "swamp_io_free_raster", "swamp_io_load_dem", "swamp_io_write_finest",
    "swamp_io_write_gauges", "swamp_io_write_step_reports",
)


class SwampError(RuntimeError):
    pass


class Engine:
    """SimState owner on one GPU."""

    def __init__(self, cfg: SimConfig, h, qx, qy, z, device: int = 0, uniform: bool = False, parts=None,
                 rank=None):
        self.cfg = cfg
        self.L = int(cfg.L)
        self.uniform = uniform
        self._c = cfg.to_c()
        n = cfg.side * cfg.side
        arrs = [as_f64(a).reshape(-1) for a in (h, qx, qy, z)]
        if any(a.size != n for a in arrs):
            raise ValueError(f"fields must be 2^L x 2^L = {cfg.side} x {cfg.side}")
        self._h = C.c_void_p()
        self.blob = None
        if rank is not None:  # one partition of a multi-process engine: (rank, world); connect() follows
            r, w = rank
            self.blob = (C.c_uint8 * RANK_BLOB_BYTES)()
            st = lib().swamp_gpu_rank_create(C.byref(self._c), *[dptr(a) for a in arrs], int(r), int(w), int(device),
                                              C.byref(self._h), self.blob)
        elif parts is not None:  # Morton-subtree partitions: list of CUDA devices, one per partition
            devs = (C.c_int * len(parts))(*[int(d) for d in parts])
            st = lib().swamp_gpu_create_partitioned(C.byref(self._c), *[dptr(a) for a in arrs], len(parts), devs,
                                                     C.byref(self._h))
        else:
            f = lib().swamp_gpu_create_uniform if uniform else lib().swamp_gpu_create
            st = f(C.byref(self._c), *[dptr(a) for a in arrs], int(device), C.byref(self._h))
        if st != 0:
            raise SwampError(f"initialise failed: {STATUS.get(st, st)}")
        self.report = swamp_step_report()

    def connect(self, blobs):
        """Rank engines: map the peers (all ranks' blobs, rank order) and enqueue initialise."""
        buf = (C.c_uint8 * (RANK_BLOB_BYTES * len(blobs))).from_buffer_copy(b"".join(bytes(b) for b in blobs))
        self._check(lib().swamp_gpu_rank_connect(self._h, buf), "rank_connect")

    def ready(self):
        """Rank engines: wait for initialise (every rank connected) and build the step graphs."""
        self._check(lib().swamp_gpu_rank_ready(self._h), "rank_ready")

    def close(self):
        if getattr(self, "_h", None):
            lib().swamp_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st, what):
        if st != 0:
            code, z, q, stg = C.c_int32(), C.c_uint32(), C.c_int32(), C.c_int32()
            buf = C.create_string_buffer(256)
            lib().swamp_gpu_last_error(self._h, C.byref(code), C.byref(z), C.byref(q), C.byref(stg), buf, 256)
            raise SwampError(f"{what}: {STATUS.get(st, st)} (z={z.value}, quantity={q.value}, stage={stg.value}; "
                             f"{buf.value.decode()})")

    # ---- engine operations
    def step_adaptive(self) -> dict:
        self._check(lib().swamp_gpu_step(self._h, C.byref(self.report)), "step_adaptive")
        return self.report.as_dict()

    def step_uniform(self, n: int = 1) -> dict:
        self._check(lib().swamp_gpu_step_uniform(self._h, int(n), C.byref(self.report)), "step_uniform")
        return self.report.as_dict()

    def advance(self, n: int) -> dict:
        self._check(lib().swamp_gpu_advance(self._h, int(n), C.byref(self.report)), "advance")
        return self.report.as_dict()

    def advance_reports(self, n: int) -> list:
        """Advance n steps back to back; every step's StepReport (read into
        host memory as the step completes, no host round trip between steps)."""
        n = int(n)
        if n <= 0:
            return []
        reps = (swamp_step_report * n)()
        self._check(lib().swamp_gpu_advance_reports(self._h, n, reps), "advance_reports")
        return [r.as_dict() for r in reps]

    def run(self) -> dict:
        self._check(lib().swamp_gpu_run(self._h, C.byref(self.report)), "run")
        return self.report.as_dict()

    def enqueue(self, n: int):
        """Launch n steps asynchronously on the engine's stream (no sync)."""
        self._check(lib().swamp_gpu_enqueue(self._h, int(n)), "enqueue")

    def stream_ptr(self) -> int:
        s = C.c_void_p()
        self._check(lib().swamp_gpu_stream(self._h, C.byref(s)), "stream")
        return s.value or 0

    def set_profiling(self, on: bool):
        lib().swamp_gpu_set_profiling(self._h, 1 if on else 0)

    # ---- state
    def info(self) -> dict:
        t, dt = C.c_double(), C.c_double()
        s, nl = C.c_int64(), C.c_int64()
        self._check(lib().swamp_gpu_info(self._h, C.byref(t), C.byref(dt), C.byref(s), C.byref(nl)), "info")
        return {"t": t.value, "dt": dt.value, "step": s.value, "n_leaves": nl.value}

    def leaves(self, with_neighbours: bool = True):
        n = C.c_int64()
        self._check(lib().swamp_gpu_copy_leaves(self._h, None, None, None, None, None, 0, C.byref(n)), "leaves")
        N = n.value
        lv = np.zeros(N, np.uint32)
        nb = np.zeros((4, N), np.uint32)
        ptrs = [u32ptr(nb[d]) for d in range(4)] if with_neighbours else [None] * 4
        self._check(lib().swamp_gpu_copy_leaves(self._h, u32ptr(lv), *ptrs, N, C.byref(n)), "leaves")
        return lv, nb

    def export_tree(self):
        NH, ND = level_offset(self.L + 1), level_offset(self.L)
        out = [np.zeros(NH) for _ in range(4)]
        sig = np.zeros(ND, np.uint8)
        self._check(lib().swamp_gpu_export_tree(self._h, *[dptr(a) for a in out], u8ptr(sig)), "export_tree")
        return out, sig

    def export_finest(self, out=None):
        """Finest-grid expansion (h, qx, qy), row 0 = south. `out`: three
        C-contiguous float64 (2^L, 2^L) arrays to fill (e.g. pinned_empty:
        device-to-host copies at full speed)."""
        n = self.cfg.side
        if out is None:
            out = [np.zeros((n, n)) for _ in range(3)]
        for a in out:
            if a.dtype != np.float64 or not a.flags.c_contiguous or a.size != n * n:
                raise ValueError("export_finest: out arrays must be C-contiguous float64 2^L x 2^L")
        self._check(lib().swamp_gpu_export_finest(self._h, *[dptr(a) for a in out]), "export_finest")
        return out

    def sample_gauges(self, xs, ys) -> np.ndarray:
        """Gauges: (4, n) array [h, qx, qy, eta] of the leaves
        covering the points (xs[k], ys[k])."""
        x = as_f64(xs).reshape(-1)
        y = as_f64(ys).reshape(-1)
        if x.size != y.size:
            raise ValueError("gauge x / y lengths differ")
        out = np.zeros((4, x.size))
        if x.size:
            self._check(lib().swamp_gpu_sample_gauges(self._h, x.size, dptr(x), dptr(y), dptr(out)), "sample_gauges")
        return out

    def timeline(self):
        """Stage timeline (us) of the last profiled step: K1/K2/K3/K5 x
        (first CTA start, last CTA elected, done)."""
        a = (C.c_double * 12)()
        self._check(lib().swamp_gpu_timeline(self._h, a), "timeline")
        return [round(v, 2) for v in a]

    def debug(self):
        """Raw phase stamps (ns) of probe CTAs (swamp_gpu_debug)."""
        a = (C.c_uint64 * 64)()
        self._check(lib().swamp_gpu_debug(self._h, a), "debug")
        return list(a)

    def rebalance(self) -> bool:
        """Dynamic repartitioning: equalise the partitions' leaf counts; True when boundaries moved."""
        ch = C.c_int32()
        self._check(lib().swamp_gpu_rebalance(self._h, C.byref(ch)), "rebalance")
        return bool(ch.value)

    def compare(self, other) -> dict:
        """compare: L1 and L-infinity of the depth against
        another engine on the same device and grid."""
        l1, li = C.c_double(), C.c_double()
        self._check(lib().swamp_gpu_compare(self._h, other._h, C.byref(l1), C.byref(li)), "compare")
        return {"L1": l1.value, "Linf": li.value}

    def counters(self):
        """[N last step, re-encoded cells (cum.), decoded cells (cum.), 4^L, leaf updates (cum.)]"""
        a = (C.c_int64 * 8)()
        self._check(lib().swamp_gpu_counters(self._h, a), "counters")
        return list(a)[:5]

    def near_threshold(self) -> dict:
        """Near-threshold cell counts (D8): last step, all steps,
        initialise (flow quantities), initialise (DEM mask)."""
        a = (C.c_int64 * 4)()
        self._check(lib().swamp_gpu_near_threshold(self._h, a), "near_threshold")
        return {"last": a[0], "total": a[1], "init": a[2], "dem": a[3]}

    def work(self) -> dict:
        """Cumulative work counters (swamp_gpu_work_counters)."""
        a = (C.c_int64 * 8)()
        self._check(lib().swamp_gpu_work_counters(self._h, a), "work_counters")
        keys = ("k1_reencoded", "fv1_reencoded", "decoded", "leaf_updates", "quiet_updates", "tile_updates", "steps",
                "detail_cells")
        return dict(zip(keys, (int(x) for x in a)))

    def skips(self) -> dict:
        """Stable-quiet skips (swamp_gpu_skip_counters): leaves FV1 skipped,
        re-encoded cells K1 skipped (cumulative; both inside work())."""
        a = (C.c_int64 * 2)()
        self._check(lib().swamp_gpu_skip_counters(self._h, a), "skip_counters")
        return {"fv1_skipped_leaves": int(a[0]), "k1_skipped_cells": int(a[1])}

    def launches_per_step(self) -> int:
        """Kernels one adaptive step launches (kernel nodes of the one-step graph)."""
        a = (C.c_int64 * 8)()
        self._check(lib().swamp_gpu_counters(self._h, a), "counters")
        return int(a[5])


def trim_cache(device: int = -1) -> None:
    """Release the device buffers destroyed engines left in the process-wide
    block cache (swamp_gpu_trim_cache; -1: every device)."""
    lib().swamp_gpu_trim_cache(device)


def pinned_empty(shape, dtype=np.float64):
    """A numpy array in page-locked host memory (torch's pinned allocator):
    host <-> device copies through the C-ABI run at full PCIe speed."""
    import torch

    t = torch.empty(int(np.prod(shape)), dtype=torch.from_numpy(np.empty(0, dtype)).dtype, pin_memory=True)
    return t.numpy().reshape(shape)


def pinned_copy(a):
    """A pinned-memory copy of array `a`."""
    p = pinned_empty(np.shape(a), np.asarray(a).dtype)
    p[...] = a
    return p


def initialise(cfg: SimConfig, h, qx, qy, z, device: int = 0) -> Engine:
    """engine.initialise on `device`."""
    return Engine(cfg, h, qx, qy, z, device=device)


def initialise_partitioned(cfg: SimConfig, h, qx, qy, z, devices) -> Engine:
    """Morton-subtree partitioned engine: partition k on CUDA device devices[k]
    (repeat a device to run virtual partitions on one GPU)."""
    return Engine(cfg, h, qx, qy, z, parts=list(devices))


def initialise_rank(cfg: SimConfig, h, qx, qy, z, rank: int, world: int, device: int, allgather) -> Engine:
    """One Morton-subtree partition per process (torchrun rank): partition
    `rank` of `world` on CUDA `device`. `allgather(bytes) -> list[bytes]`
    exchanges the ranks' CUDA IPC blobs (rank order), e.g.
    paper_2206_05761_b200.ranks.torch_allgather."""
    e = Engine(cfg, h, qx, qy, z, device=device, rank=(rank, world))
    e.connect(allgather(bytes(e.blob)))
    e.ready()
    return e


def initialise_uniform(cfg: SimConfig, h, qx, qy, z, device: int = 0) -> Engine:
    """The uniform GPU-FV1 solver state."""
    return Engine(cfg, h, qx, qy, z, device=device, uniform=True)


def partition_plan(L: int, G: int, leaves_before=None):
    """The engine's partition plan (swamp_partition_plan, host code): subtree
    boundaries of G partitions, balanced on the cumulative leaf counts when
    given (as swamp_gpu_rebalance), else equal subtree counts (creation)."""
    L_ = lib()
    L_.swamp_partition_plan.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
    out = (C.c_uint32 * (G + 1))()
    if leaves_before is None:
        st = L_.swamp_partition_plan(int(L), int(G), None, out)
    else:
        a = np.ascontiguousarray(np.asarray(leaves_before, dtype=np.uint64))
        st = L_.swamp_partition_plan(int(L), int(G), a.ctypes.data_as(C.POINTER(C.c_uint64)), out)
    if st != 0:
        raise SwampError(f"partition_plan: {STATUS.get(st, st)}")
    return list(out)


def partition_owner(bounds, L: int, n: int, m: int) -> int:
    """Owner of cell (n, m) under `bounds` (swamp_partition_owner)."""
    L_ = lib()
    L_.swamp_partition_owner.argtypes = [C.POINTER(C.c_uint32), C.c_int32, C.c_int32, C.c_int32, C.c_uint32]
    b = (C.c_uint32 * len(bounds))(*bounds)
    r = L_.swamp_partition_owner(b, len(bounds) - 1, int(L), int(n), int(m))
    if r < 0:
        raise SwampError(f"partition_owner: {STATUS.get(r, r)}")
    return r
