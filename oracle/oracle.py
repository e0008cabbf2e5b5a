"""ctypes wrapper of the CPU-HWFV1 oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY — the checker for the GPU path and the timed CPU
baseline. Importable from tests/, __graft_entry__.smoke() and bench.py's CPU
legs; never from the product package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2206_05761_b200.abi import (
    SimConfig,
    as_f64,
    dptr,
    level_offset,
    swamp_config,
    u8ptr,
    u32ptr,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        L = C.CDLL(path)
        P = C.c_void_p
        dp = C.POINTER(C.c_double)
        L.oracle_create.argtypes = [C.POINTER(swamp_config), dp, dp, dp, dp, C.POINTER(P)]
        L.oracle_create_uniform.argtypes = L.oracle_create.argtypes
        L.oracle_destroy.argtypes = [P]
        L.oracle_step.argtypes = [P]
        L.oracle_step_uniform.argtypes = [P]
        L.oracle_set_threads.argtypes = [C.c_int]
        L.oracle_info.argtypes = [P, dp, dp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        u32p = C.POINTER(C.c_uint32)
        L.oracle_copy_leaves.argtypes = [P, u32p, u32p, u32p, u32p, u32p, C.c_int64, C.POINTER(C.c_int64)]
        L.oracle_export_tree.argtypes = [P, dp, dp, dp, dp, C.POINTER(C.c_uint8)]
        L.oracle_export_finest.argtypes = [P, dp, dp, dp]
        L.oracle_counters.argtypes = [P, C.POINTER(C.c_int64)]
        L.oracle_near_threshold.argtypes = [P, C.POINTER(C.c_int64)]
        L.oracle_last_error.argtypes = [P]
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_import_tree.argtypes = [P, dp, dp, dp, C.POINTER(C.c_uint8), C.c_double, C.c_double,
                                         C.c_double, C.c_int64]
        L.oracle_morton_encode.argtypes = [C.c_uint32, C.c_uint32]
        L.oracle_morton_encode.restype = C.c_uint32
        L.oracle_morton_decode.argtypes = [C.c_uint32, u32p, u32p]
        L.oracle_neighbour.argtypes = [C.c_int, C.c_uint32, C.c_int]
        L.oracle_neighbour.restype = C.c_int64
        L.oracle_encode4.argtypes = [dp, dp]
        L.oracle_decode4.argtypes = [dp, dp]
        L.oracle_significance.argtypes = [dp, C.c_double, C.c_int, C.c_int, C.c_double]
        L.oracle_hll.argtypes = [C.c_double] * 7 + [dp]
        L.oracle_face.argtypes = [dp, dp, C.c_double, C.c_double, dp, dp]
        L.oracle_fv1_cell.argtypes = [dp, dp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, dp]
        L.oracle_friction.argtypes = [C.c_double] * 7 + [dp]
        L.oracle_cfl_cell.argtypes = [C.c_double] * 6
        L.oracle_cfl_cell.restype = C.c_double
        L.oracle_cbrt.argtypes = [C.c_double]
        L.oracle_cbrt.restype = C.c_double
        L.oracle_boundary.argtypes = [dp, C.c_int, C.c_int, C.c_double, dp, dp, C.c_int, C.c_int, C.c_double, dp]
        L.oracle_ptt.argtypes = [C.c_int, C.POINTER(C.c_uint8), u32p]
        L.oracle_compact.argtypes = [u32p, C.c_int64, u32p]
        L.oracle_compact.restype = C.c_int64
        L.oracle_neighbours.argtypes = [C.c_int, u32p, u32p, C.c_int64, C.POINTER(C.c_int32), u32p]
        L.oracle_dft_leaves.argtypes = [C.c_int, C.POINTER(C.c_uint8), u32p]
        L.oracle_dft_leaves.restype = C.c_int64
        _LIB = L
    return _LIB


def set_threads(n: int) -> int:
    return lib().oracle_set_threads(int(n))


class OracleError(RuntimeError):
    pass


class Oracle:
    """CPU-HWFV1 engine: initialise on construction, step(), exports."""

    def __init__(self, cfg: SimConfig, h, qx, qy, z, uniform: bool = False):
        self.cfg = cfg
        self.L = int(cfg.L)
        self._c = cfg.to_c()
        arrs = [as_f64(a).reshape(-1) for a in (h, qx, qy, z)]
        n = cfg.side * cfg.side
        if any(a.size != n for a in arrs):
            raise ValueError("fields must be 2^L x 2^L")
        self._h = C.c_void_p()
        f = lib().oracle_create_uniform if uniform else lib().oracle_create
        st = f(C.byref(self._c), *[dptr(a) for a in arrs], C.byref(self._h))
        if st != 0:
            raise OracleError(f"oracle_create failed: {st}")

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.oracle_destroy(self._h)
            self._h = None

    def step(self, n: int = 1, uniform: bool = False):
        f = lib().oracle_step_uniform if uniform else lib().oracle_step
        for _ in range(n):
            st = f(self._h)
            if st != 0:
                raise OracleError(f"oracle_step: {st} {lib().oracle_last_error(self._h).decode()}")

    def info(self):
        t, dt = C.c_double(), C.c_double()
        s, nl = C.c_int64(), C.c_int64()
        lib().oracle_info(self._h, C.byref(t), C.byref(dt), C.byref(s), C.byref(nl))
        return {"t": t.value, "dt": dt.value, "step": s.value, "n_leaves": nl.value}

    def run(self, max_steps: int = 10**9):
        k = 0
        while self.info()["t"] < self.cfg.t_end and k < max_steps:
            self.step()
            k += 1
        return k

    def leaves(self):
        n = C.c_int64()
        lib().oracle_copy_leaves(self._h, None, None, None, None, None, 0, C.byref(n))
        N = n.value
        lv = np.zeros(N, np.uint32)
        nb = np.zeros((4, N), np.uint32)
        lib().oracle_copy_leaves(self._h, u32ptr(lv), *[u32ptr(nb[d]) for d in range(4)], N, C.byref(n))
        return lv, nb

    def export_tree(self):
        NH = level_offset(self.L + 1)
        ND = level_offset(self.L)
        out = [np.zeros(NH) for _ in range(4)]
        sig = np.zeros(ND, np.uint8)
        lib().oracle_export_tree(self._h, *[dptr(a) for a in out], u8ptr(sig))
        return out, sig

    def export_finest(self):
        n = self.cfg.side
        out = [np.zeros((n, n)) for _ in range(3)]
        lib().oracle_export_finest(self._h, *[dptr(a) for a in out])
        return out

    def counters(self):
        a = (C.c_int64 * 4)()
        lib().oracle_counters(self._h, a)
        return list(a)

    def near_threshold(self):
        """Near-threshold cell counts (D8): last step, all steps, initialise
        (flow), initialise (DEM mask)."""
        a = (C.c_int64 * 4)()
        lib().oracle_near_threshold(self._h, a)
        return {"last": a[0], "total": a[1], "init": a[2], "dem": a[3]}

    def import_tree(self, h, qx, qy, sig, t, dt, t_next, step):
        arrs = [as_f64(a) for a in (h, qx, qy)]
        sig = np.ascontiguousarray(sig, dtype=np.uint8)
        st = lib().oracle_import_tree(self._h, *[dptr(a) for a in arrs], u8ptr(sig), t, dt, t_next, step)
        if st != 0:
            raise OracleError(f"oracle_import_tree: {st}")


# ------------------------------------------------------------ per-op helpers
def _d(n):
    return (C.c_double * n)()


def encode4(c):
    o = _d(4)
    lib().oracle_encode4((C.c_double * 4)(*c), o)
    return list(o)


def decode4(v):
    o = _d(4)
    lib().oracle_decode4((C.c_double * 4)(*v), o)
    return list(o)


def significance(d, smax, n, L, eps):
    return bool(lib().oracle_significance((C.c_double * 3)(*d), smax, n, L, eps))


def hll(hL, uL, vL, hR, uR, vR, g=9.80665):
    o = _d(3)
    lib().oracle_hll(hL, uL, vL, hR, uR, vR, g, o)
    return list(o)


def face(Lc, Rc, g=9.80665, hdry=1e-6):
    F, hs = _d(3), _d(2)
    lib().oracle_face((C.c_double * 4)(*Lc), (C.c_double * 4)(*Rc), g, hdry, F, hs)
    return list(F), list(hs)


def fv1_cell(own, nbrs, dx, dt, g=9.80665, hdry=1e-6, nM=0.0):
    o = _d(3)
    flat = [v for nb in nbrs for v in nb]
    lib().oracle_fv1_cell((C.c_double * 4)(*own), (C.c_double * 16)(*flat), dx, dt, g, hdry, nM, o)
    return list(o)


def friction(h, qx, qy, dt, g, nM, hdry=1e-6):
    o = _d(2)
    lib().oracle_friction(h, qx, qy, dt, g, nM, hdry, o)
    return list(o)


def cfl_cell(h, qx, qy, dx, g=9.80665, hdry=1e-6):
    return lib().oracle_cfl_cell(h, qx, qy, dx, g, hdry)


def cbrt(x):
    return lib().oracle_cbrt(x)


def boundary(own, kind, direction, t=0.0, series_t=(), series_v=(), mode=0, hdry=1e-6):
    o = _d(4)
    n = len(series_t)
    ts = (C.c_double * max(n, 1))(*series_t)
    vs = (C.c_double * max(n, 1))(*series_v)
    lib().oracle_boundary((C.c_double * 4)(*own), kind, direction, t, ts, vs, n, mode, hdry, o)
    return list(o)


def ptt(L, sig):
    sig = np.ascontiguousarray(sig, np.uint8)
    rec = np.zeros(1 << (2 * L), np.uint32)
    lib().oracle_ptt(L, u8ptr(sig), u32ptr(rec))
    return rec


def compact(rec):
    rec = np.ascontiguousarray(rec, np.uint32)
    n = lib().oracle_compact(u32ptr(rec), rec.size, None)
    out = np.zeros(n, np.uint32)
    lib().oracle_compact(u32ptr(rec), rec.size, u32ptr(out))
    return out


def neighbours(L, rec, leaves, bc=(0, 0, 0, 0)):
    rec = np.ascontiguousarray(rec, np.uint32)
    leaves = np.ascontiguousarray(leaves, np.uint32)
    out = np.zeros((4, leaves.size), np.uint32)
    st = lib().oracle_neighbours(L, u32ptr(rec), u32ptr(leaves), leaves.size, (C.c_int32 * 4)(*bc), u32ptr(out))
    if st != 0:
        raise OracleError("find_neighbours: malformed recorded grid")
    return out


def dft_leaves(L, sig):
    sig = np.ascontiguousarray(sig, np.uint8)
    n = lib().oracle_dft_leaves(L, u8ptr(sig), None)
    out = np.zeros(n, np.uint32)
    lib().oracle_dft_leaves(L, u8ptr(sig), u32ptr(out))
    return out


def morton_encode(i, j):
    return lib().oracle_morton_encode(i, j)


def morton_decode(m):
    i, j = C.c_uint32(), C.c_uint32()
    lib().oracle_morton_decode(m, C.byref(i), C.byref(j))
    return i.value, j.value


def neighbour(n, m, d):
    r = lib().oracle_neighbour(n, m, d)
    return None if r < 0 else r


# ---------------------------------------------------------------- io
def load_dem_ref(values, xll, yll, cs, nodata, L, x0, y0, W, wall_z):
    """numpy restatement of load_dem, the checker of
    swamp_io_load_dem: finest-cell centres sampled nearest-cell when the raster
    cellsize equals W / 2^L, bilinear between raster cell centres otherwise
    (edge cells clamped); outside / nodata -> inactive with z = wall_z.
    values[row, col] with row 0 the TOP row; returns (z, inactive) with row 0
    the SOUTH row. Same IEEE operations, same order as the C++."""
    vals = np.asarray(values, dtype=np.float64)
    nr, nc = vals.shape
    side = 1 << L
    dx = W / side
    z = np.full((side, side), wall_z)
    ina = np.ones((side, side), dtype=bool)

    def val(ci, rj):
        return vals[nr - 1 - rj, ci]

    def nod(v):
        return v == nodata or not np.isfinite(v)

    for j in range(side):
        for i in range(side):
            x = x0 + (i + 0.5) * dx
            y = y0 + (j + 0.5) * dx
            if dx == cs:
                fi, fj = np.floor((x - xll) / cs), np.floor((y - yll) / cs)
                if 0 <= fi < nc and 0 <= fj < nr:
                    v = val(int(fi), int(fj))
                    if not nod(v):
                        z[j, i], ina[j, i] = v, False
            else:
                u = (x - xll) / cs - 0.5
                w = (y - yll) / cs - 0.5
                if -0.5 <= u <= nc - 0.5 and -0.5 <= w <= nr - 0.5:
                    i0, j0 = int(np.floor(u)), int(np.floor(w))
                    a, b = u - i0, w - j0
                    if i0 < 0:
                        i0, a = 0, 0.0
                    if j0 < 0:
                        j0, b = 0, 0.0
                    if i0 >= nc - 1:
                        i0, a = nc - 1, 0.0
                    if j0 >= nr - 1:
                        j0, b = nr - 1, 0.0
                    i1 = i0 + 1 if i0 + 1 < nc else i0
                    j1 = j0 + 1 if j0 + 1 < nr else j0
                    v00, v10, v01, v11 = val(i0, j0), val(i1, j0), val(i0, j1), val(i1, j1)
                    bad = nod(v00) or (a > 0 and nod(v10)) or (b > 0 and nod(v01)) or (a > 0 and b > 0 and nod(v11))
                    if not bad:
                        s0 = v00 + a * (v10 - v00) if a > 0 else v00
                        s1 = v01 + a * (v11 - v01) if a > 0 else v01
                        z[j, i] = s0 + b * (s1 - s0) if b > 0 else s0
                        ina[j, i] = False
    return z, ina
