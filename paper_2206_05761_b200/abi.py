"""ctypes mirror of the C-ABI types in include/swamp_gpu.h.

`SimConfig` is the Python form of SPEC.md's SimConfig; it
keeps the numpy arrays that back the C struct's pointers alive for as long as
the struct is in use.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

BC_REFLECTIVE, BC_TRANSMISSIVE, BC_INFLOW = 0, 1, 2
BAND_NONE, BAND_PARENTS, BAND_NEIGHBOURS = 0, 1, 2
INFLOW_DEPTH, INFLOW_ETA = 0, 1
BOUNDARY_BASE = 0xFFFFFFF0

STATUS = {
    0: "ok",
    -1: "invalid argument",
    -2: "CUDA failure",
    -3: "non-finite coefficient or flux",
    -4: "dt <= 0 or non-finite",
    -5: "invalid state",
    -6: "device allocation failed",
    -7: "a partition never reached a barrier",
}

_dp = C.POINTER(C.c_double)


class swamp_config(C.Structure):
    _fields_ = [
        ("L", C.c_int32),
        ("band_mode", C.c_int32),
        ("epsilon", C.c_double),
        ("width", C.c_double),
        ("x0", C.c_double),
        ("y0", C.c_double),
        ("cfl", C.c_double),
        ("g", C.c_double),
        ("manning", C.c_double),
        ("h_dry", C.c_double),
        ("t_end", C.c_double),
        ("dt_fallback", C.c_double),
        ("bc", C.c_int32 * 4),
        ("inflow_mode", C.c_int32),
        ("inflow_n", C.c_int32),
        ("n_outputs", C.c_int32),
        ("inflow_t", _dp),
        ("inflow_v", _dp),
        ("output_times", _dp),
        ("inactive", C.POINTER(C.c_uint8)),
    ]


class swamp_step_report(C.Structure):
    _fields_ = [
        ("step", C.c_int64),
        ("t", C.c_double),
        ("dt", C.c_double),
        ("dt_used", C.c_double),
        ("n_leaves", C.c_int64),
        ("n_leaves_next", C.c_int64),
        ("ms_encode_flag", C.c_double),
        ("ms_band_closure", C.c_double),
        ("ms_decode_traverse", C.c_double),
        ("ms_neighbours", C.c_double),
        ("ms_fv1", C.c_double),
        ("ms_total", C.c_double),
        ("n_near_threshold", C.c_int64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


@dataclass
class SimConfig:
    """SimConfig with the defaults of SPEC.md:290, 359, 362."""

    L: int
    epsilon: float
    width: float
    x0: float = 0.0
    y0: float = 0.0
    cfl: float = 0.5
    g: float = 9.80665
    manning: float = 0.0
    h_dry: float = 1e-6
    t_end: float = 1.0
    dt_fallback: float = 1e-3
    bc: Sequence[int] = (BC_REFLECTIVE,) * 4  # W, E, N, S
    band_mode: int = BAND_NEIGHBOURS
    inflow_mode: int = INFLOW_DEPTH
    inflow_t: Sequence[float] = ()
    inflow_v: Sequence[float] = ()
    output_times: Sequence[float] = ()
    inactive: object = None  # 2^L x 2^L bool/uint8 (south row first) or None (D16)
    name: str = ""
    _keep: list = field(default_factory=list, repr=False)

    def validate(self) -> None:
        """L in [1, 13], epsilon >= 0 (load_config errors)."""
        if not (1 <= int(self.L) <= 13):
            raise ValueError(f"L={self.L} outside [1, 13] (z-index must stay below 2^28)")
        if not (self.epsilon >= 0.0):
            raise ValueError(f"epsilon={self.epsilon} must be >= 0")
        if not (self.width > 0.0):
            raise ValueError("width must be > 0")
        if not (0.0 < self.cfl <= 1.0):
            raise ValueError("CFL number must be in (0, 1]")
        if not (self.h_dry > 0.0):
            raise ValueError("h_dry must be > 0")
        if not (self.g > 0.0) or not (self.manning >= 0.0):
            raise ValueError("g must be > 0 and manning >= 0")
        if not (self.dt_fallback > 0.0):
            raise ValueError("dt_fallback must be > 0")
        if len(self.bc) != 4 or any(int(b) not in (BC_REFLECTIVE, BC_TRANSMISSIVE, BC_INFLOW) for b in self.bc):
            raise ValueError(f"bc={self.bc}: four edge kinds in {{0, 1, 2}}")
        if int(self.band_mode) not in (BAND_NONE, BAND_PARENTS, BAND_NEIGHBOURS):
            raise ValueError(f"band_mode={self.band_mode}")
        if int(self.inflow_mode) not in (INFLOW_DEPTH, INFLOW_ETA):
            raise ValueError(f"inflow_mode={self.inflow_mode}")
        if BC_INFLOW in [int(b) for b in self.bc] and len(self.inflow_t) == 0:
            raise ValueError("an inflow edge needs an inflow series")
        if len(self.inflow_t) != len(self.inflow_v):
            raise ValueError("inflow series t / v lengths differ")

    def to_c(self) -> swamp_config:
        self.validate()
        c = swamp_config()
        c.L = int(self.L)
        c.band_mode = int(self.band_mode)
        c.epsilon = float(self.epsilon)
        c.width = float(self.width)
        c.x0, c.y0 = float(self.x0), float(self.y0)
        c.cfl, c.g, c.manning, c.h_dry = float(self.cfl), float(self.g), float(self.manning), float(self.h_dry)
        c.t_end, c.dt_fallback = float(self.t_end), float(self.dt_fallback)
        for k in range(4):
            c.bc[k] = int(self.bc[k])
        c.inflow_mode = int(self.inflow_mode)
        self._keep = []

        def arr(v):
            a = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
            self._keep.append(a)
            return a.ctypes.data_as(_dp) if a.size else None

        c.inflow_n = len(self.inflow_t)
        c.inflow_t = arr(self.inflow_t)
        c.inflow_v = arr(self.inflow_v)
        c.n_outputs = len(self.output_times)
        c.output_times = arr(self.output_times)
        if self.inactive is not None:
            m = np.ascontiguousarray(np.asarray(self.inactive).reshape(-1) != 0, dtype=np.uint8)
            if m.size != self.side * self.side:
                raise ValueError("inactive mask must be 2^L x 2^L")
            self._keep.append(m)
            c.inactive = m.ctypes.data_as(C.POINTER(C.c_uint8))
        return c

    @property
    def side(self) -> int:
        return 1 << int(self.L)

    @property
    def dx(self) -> float:
        return self.width / self.side


def as_f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def u32ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def u8ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def level_offset(n: int) -> int:
    return ((1 << (2 * n)) - 1) // 3


def level_of(z):
    """Vectorised O(1) level_of (zorder.hpp:83-87 semantics)."""
    z = np.asarray(z, dtype=np.int64)
    v = 3 * z + 1
    return (np.floor(np.log2(v.astype(np.float64))).astype(np.int64)) // 2
