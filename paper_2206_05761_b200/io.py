"""Data formats either side of the hot path (include/swamp_io.h; SPEC.md io
module :541-600): Esri ASCII rasters, DEM ingestion onto the finest grid
(top row first -> south row first, nodata / outside -> inactive), finest-grid
snapshots. Host code in libswamp_gpu.so (no GPU needed)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .abi import STATUS


class swamp_raster(C.Structure):
    _fields_ = [("ncols", C.c_int32), ("nrows", C.c_int32), ("xllcorner", C.c_double), ("yllcorner", C.c_double),
                ("cellsize", C.c_double), ("nodata", C.c_double), ("values", C.POINTER(C.c_double))]


@dataclass
class Raster:
    """RasterGrid; values[row, col], row 0 = TOP row."""
    values: np.ndarray
    xllcorner: float = 0.0
    yllcorner: float = 0.0
    cellsize: float = 1.0
    nodata: float = -9999.0

    @property
    def nrows(self):
        return self.values.shape[0]

    @property
    def ncols(self):
        return self.values.shape[1]

    def _c(self):
        v = np.ascontiguousarray(self.values, dtype=np.float64)
        r = swamp_raster(self.ncols, self.nrows, self.xllcorner, self.yllcorner, self.cellsize, self.nodata,
                         v.ctypes.data_as(C.POINTER(C.c_double)))
        return r, v


class IoError(RuntimeError):
    pass


def _lib():
    from .gpu import lib

    L = lib()
    if not getattr(L, "_io_bound", False):
        rp = C.POINTER(swamp_raster)
        L.swamp_io_read_esri.argtypes = [C.c_char_p, rp, C.c_char_p, C.c_size_t]
        L.swamp_io_write_esri.argtypes = [C.c_char_p, rp]
        L.swamp_io_free_raster.argtypes = [rp]
        L.swamp_io_free_raster.restype = None
        L.swamp_io_load_dem.argtypes = [rp, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_uint8)]
        L.swamp_io_write_finest.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_double,
                                            C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.c_double]
        L.swamp_io_write_gauges.argtypes = [C.c_char_p, C.c_int32, C.POINTER(C.c_char_p), C.c_int32,
                                            C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.swamp_io_write_step_reports.argtypes = [C.c_char_p, C.c_int32, C.c_void_p, C.c_int]
        L._io_bound = True
    return L


def read_esri(path: str) -> Raster:
    r = swamp_raster()
    msg = C.create_string_buffer(256)
    st = _lib().swamp_io_read_esri(str(path).encode(), C.byref(r), msg, 256)
    if st != 0:
        raise IoError(f"{path}: {STATUS.get(st, st)}: {msg.value.decode()}")
    try:
        v = np.ctypeslib.as_array(r.values, shape=(r.nrows * r.ncols,)).reshape(r.nrows, r.ncols).copy()
    finally:
        _lib().swamp_io_free_raster(C.byref(r))
    return Raster(v, r.xllcorner, r.yllcorner, r.cellsize, r.nodata)


def write_esri(path: str, raster: Raster) -> None:
    r, _keep = raster._c()
    st = _lib().swamp_io_write_esri(str(path).encode(), C.byref(r))
    if st != 0:
        raise IoError(f"{path}: {STATUS.get(st, st)}")


def load_dem(raster: Raster, L: int, x0: float, y0: float, W: float, wall_z: float = 1e3, strict: bool = False):
    """load_dem -> (z, inactive), 2^L x 2^L, row 0 = SOUTH row."""
    n = 1 << L
    z = np.empty(n * n)
    ina = np.empty(n * n, dtype=np.uint8)
    r, _keep = raster._c()
    st = _lib().swamp_io_load_dem(C.byref(r), int(L), float(x0), float(y0), float(W), float(wall_z), int(strict),
                                  z.ctypes.data_as(C.POINTER(C.c_double)), ina.ctypes.data_as(C.POINTER(C.c_uint8)))
    if st != 0:
        raise IoError(f"load_dem: {STATUS.get(st, st)}")
    return z.reshape(n, n), ina.reshape(n, n).astype(bool)


def write_finest(path: str, field, L: int, x0: float, y0: float, W: float, inactive=None, nodata: float = -9999.0):
    """A finest-grid field (row 0 = south) as an Esri raster."""
    f = np.ascontiguousarray(field, dtype=np.float64).reshape(-1)
    ia = None if inactive is None else np.ascontiguousarray(inactive, dtype=np.uint8).reshape(-1)
    st = _lib().swamp_io_write_finest(str(path).encode(), int(L), float(x0), float(y0), float(W),
                                      f.ctypes.data_as(C.POINTER(C.c_double)),
                                      None if ia is None else ia.ctypes.data_as(C.POINTER(C.c_uint8)), float(nodata))
    if st != 0:
        raise IoError(f"{path}: {STATUS.get(st, st)}")


def write_gauges(path: str, times, samples, names=None) -> None:
    """write_gauges: `samples[k]` = the (4, n_gauges)
    array Engine.sample_gauges returned at times[k]; one CSV record per time."""
    t = np.ascontiguousarray(np.asarray(times, dtype=np.float64).reshape(-1))
    ng = len(names) if names is not None else (np.asarray(samples[0]).shape[1] if len(samples) else 0)
    v = np.ascontiguousarray(np.asarray(samples, dtype=np.float64).reshape(t.size, 4 * ng) if t.size else
                             np.zeros(0))
    nm = None
    if names is not None:
        nm = (C.c_char_p * ng)(*[str(x).encode() for x in names])
    st = _lib().swamp_io_write_gauges(str(path).encode(), int(ng), nm, int(t.size),
                                      t.ctypes.data_as(C.POINTER(C.c_double)), v.ctypes.data_as(C.POINTER(C.c_double)))
    if st != 0:
        raise IoError(f"{path}: {STATUS.get(st, st)}")


def write_step_reports(path: str, reports, append: bool = False) -> None:
    """write_step_report: StepReport dicts (Engine.step_adaptive
    results) as CSV rows, columns in include/swamp_io.h's stable order."""
    from .abi import swamp_step_report

    arr = (swamp_step_report * max(1, len(reports)))()
    for k, r in enumerate(reports):
        for f, _ in swamp_step_report._fields_:
            setattr(arr[k], f, r[f])
    st = _lib().swamp_io_write_step_reports(str(path).encode(), len(reports), C.cast(arr, C.c_void_p),
                                            1 if append else 0)
    if st != 0:
        raise IoError(f"{path}: {STATUS.get(st, st)}")
