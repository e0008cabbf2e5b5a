"""io and the DEM ingestion row of SURVEY.md §8(f): Esri
ASCII rasters through the library's C-ABI (host code, no GPU), checked
bitwise against the oracle's numpy restatement of load_dem and against the
SPEC examples."""
import numpy as np
import pytest

from oracle.oracle import load_dem_ref
from paper_2206_05761_b200 import io


def test_roundtrip_bit_exact(tmp_path):
    rng = np.random.default_rng(7)
    v = rng.standard_normal((5, 7)) * 10.0 ** rng.integers(-300, 300, (5, 7))
    v[0, 0] = -0.0
    v[1, 2] = 5e-324
    r = io.Raster(v, xllcorner=-12.5, yllcorner=3.25, cellsize=0.02, nodata=-9999.0)
    io.write_esri(tmp_path / "a.asc", r)
    b = io.read_esri(tmp_path / "a.asc")
    assert (b.ncols, b.nrows) == (7, 5)
    assert (b.xllcorner, b.yllcorner, b.cellsize, b.nodata) == (-12.5, 3.25, 0.02, -9999.0)
    np.testing.assert_array_equal(b.values.view(np.uint64), v.view(np.uint64))


def test_header_forms_and_errors(tmp_path):
    p = tmp_path / "c.asc"
    p.write_text("NCOLS 2\nNROWS 1\nXLLCENTER 0.5\nYLLCENTER 1.5\nCELLSIZE 1\nnodata_value -1\n3 4\n")
    r = io.read_esri(p)
    assert (r.xllcorner, r.yllcorner) == (0.0, 1.0) and r.values.tolist() == [[3.0, 4.0]]
    p.write_text("ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\n1 2 3\n")
    with pytest.raises(io.IoError, match="expected 4 values"):
        io.read_esri(p)
    p.write_text("ncols 2\nnrows 1\nxllcorner 0\nyllcorner 0\ncellsize 1\n1 x\n")
    with pytest.raises(io.IoError, match="non-numeric value 'x' at row 0, column 1"):
        io.read_esri(p)
    p.write_text("ncols 2\nxllcorner 0\nyllcorner 0\ncellsize 1\n1 2\n")
    with pytest.raises(io.IoError, match="missing nrows"):
        io.read_esri(p)
    p.write_text("ncols 2\nnrows 1\ncolour 3\n")
    with pytest.raises(io.IoError, match="unknown key colour"):
        io.read_esri(p)


def test_spec_examples():
    # 2x2 raster of zeros, L=1 -> flat bed, no inactive cells
    z, ina = io.load_dem(io.Raster(np.zeros((2, 2))), 1, 0.0, 0.0, 2.0)
    assert (z == 0).all() and not ina.any()
    # one nodata corner -> that region inactive, at the wall height
    v = np.zeros((2, 2))
    v[0, 1] = -9999.0  # top row, east column = north-east corner
    z, ina = io.load_dem(io.Raster(v), 1, 0.0, 0.0, 2.0, wall_z=50.0)
    assert ina.tolist() == [[False, False], [False, True]] and z[1, 1] == 50.0
    # a 1800 x 180 DEM needs L = 11 in strict mode
    r = io.Raster(np.zeros((180, 1800)), cellsize=0.02)
    with pytest.raises(io.IoError):
        io.load_dem(r, 10, 0.0, 0.0, 36.0, strict=True)
    io.load_dem(r, 11, 0.0, 0.0, 0.02 * 2048, strict=True)


def test_rows_flip_south_first():
    v = np.arange(12, dtype=float).reshape(3, 4)  # row 0 = top
    z, ina = io.load_dem(io.Raster(v), 2, 0.0, 0.0, 4.0, wall_z=-1.0)
    assert z[0].tolist() == v[2].tolist()      # south row of the grid = bottom raster row
    assert z[2].tolist() == v[0].tolist()
    assert ina[3].all() and not ina[:3].any()  # the raster covers 3 of 4 rows


@pytest.mark.parametrize("cs,L,x0,y0,W", [(1.0, 4, 0.0, 0.0, 16.0), (0.7, 4, -0.3, 0.2, 12.0), (2.5, 5, 1.0, -1.0, 40.0)])
def test_load_dem_matches_restatement(cs, L, x0, y0, W):
    rng = np.random.default_rng(int(cs * 10) + L)
    v = rng.standard_normal((11, 13)) * 3.0
    v[4, 5] = -9999.0
    v[0, 12] = np.nan
    r = io.Raster(v, xllcorner=0.1, yllcorner=-0.4, cellsize=cs)
    z, ina = io.load_dem(r, L, x0, y0, W, wall_z=77.0)
    zr, ir = load_dem_ref(v, 0.1, -0.4, cs, -9999.0, L, x0, y0, W, 77.0)
    np.testing.assert_array_equal(ina, ir)
    np.testing.assert_array_equal(z.view(np.uint64), zr.view(np.uint64))


def test_write_finest_roundtrip(tmp_path):
    rng = np.random.default_rng(3)
    f = rng.standard_normal((8, 8))
    ina = np.zeros((8, 8), dtype=bool)
    ina[0, 0] = True
    io.write_finest(tmp_path / "s.asc", f, 3, 1.0, 2.0, 8.0, inactive=ina, nodata=-5.0)
    r = io.read_esri(tmp_path / "s.asc")
    assert (r.xllcorner, r.yllcorner, r.cellsize, r.nodata) == (1.0, 2.0, 1.0, -5.0)
    back = r.values[::-1]  # to south-first
    assert back[0, 0] == -5.0
    m = ~ina
    np.testing.assert_array_equal(back[m].view(np.uint64), f[m].view(np.uint64))
