"""zorder (reference proj/include/swamp/zorder.hpp).

Pins three implementations to the reference: the product's host/device header
include/swamp/zorder.hpp (compiled here through tests/cpp/zorder_shim.cpp),
the oracle's loop restatement, and — when this container has /root/reference
— the reference header itself compiled into oracle/_ref. The committed golden
file tests/golden/zorder_ref.json was produced from oracle/_ref by
tests/golden/make_golden.py.
"""
import ctypes as C
import json
import os
import subprocess

import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "zorder_ref.json")))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libzorder_ref.so")


@pytest.fixture(scope="module")
def pz():
    out = os.path.join(ROOT, "tests", "cpp", "_build")
    os.makedirs(out, exist_ok=True)
    so = os.path.join(out, "libzorder_product.so")
    src = os.path.join(ROOT, "tests", "cpp", "zorder_shim.cpp")
    hdr = os.path.join(ROOT, "include", "swamp", "zorder.hpp")
    if not os.path.exists(so) or os.path.getmtime(so) < max(os.path.getmtime(src), os.path.getmtime(hdr)):
        subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-fPIC", "-shared",
                               "-I", os.path.join(ROOT, "include"), "-o", so, src])
    L = C.CDLL(so)
    for f in ("pz_morton_encode", "pz_parent_z_index", "pz_same_level_neighbour", "pz_neighbour_dev"):
        getattr(L, f).restype = C.c_int64
    L.pz_hierarchy_cells.restype = C.c_uint64
    L.pz_detail_cells.restype = C.c_uint64
    L.pz_level_offset.restype = C.c_uint32
    L.pz_finest_under.restype = C.c_uint32
    L.pz_cells_under.restype = C.c_uint32
    return L


def test_fig5b_table_A9(pz):
    """A9: the 4x4 decimal table of Fig. 5b."""
    table = [[0, 1, 4, 5], [2, 3, 6, 7], [8, 9, 12, 13], [10, 11, 14, 15]]
    assert GOLD["morton"]["2"] == table
    assert [[pz.pz_morton_encode(i, j, 2) for i in range(4)] for j in range(4)] == table
    assert [[O.morton_encode(i, j) for i in range(4)] for j in range(4)] == table


def test_spec_examples(pz):
    # SPEC.md:43-45, 52-54, 61-63, 70-72, 79-81
    assert pz.pz_morton_encode(0, 0, 2) == 0
    assert pz.pz_morton_encode(3, 2, 2) == 13
    assert pz.pz_morton_encode(2, 1, 2) == 6
    i, j = C.c_uint32(), C.c_uint32()
    for code, ij in ((0, (0, 0)), (13, (3, 2)), (11, (1, 3))):
        assert pz.pz_morton_decode(code, 2, C.byref(i), C.byref(j)) == 0
        assert (i.value, j.value) == ij
        assert O.morton_decode(code) == ij
    assert [pz.pz_level_offset(n) for n in (0, 1, 2)] == [0, 1, 5]
    assert pz.pz_hierarchy_cells(2) == 21
    o = (C.c_uint32 * 4)()
    assert pz.pz_child_z_indices(0, 0, 2, o) == 0 and list(o) == [1, 2, 3, 4]
    assert pz.pz_child_z_indices(1, 3, 2, o) == 0 and list(o) == [17, 18, 19, 20]
    assert pz.pz_parent_z_index(2, 7) == pz.pz_level_offset(1) + 1
    assert pz.pz_same_level_neighbour(2, 0, 0) == -1  # west of m=0 absent
    assert pz.pz_same_level_neighbour(2, 0, 1) == 1
    assert pz.pz_same_level_neighbour(2, 3, 2) == 9
    # PAPER.md:237 footnote: finest Morton 3 at L=2 sits at z = 8
    assert pz.pz_level_offset(2) + 3 == 8


def test_product_matches_golden(pz):
    g = GOLD
    assert [pz.pz_level_offset(n) for n in range(14)] == g["level_offset"]
    assert [pz.pz_hierarchy_cells(n) for n in range(14)] == g["hierarchy_cells"]
    assert [pz.pz_detail_cells(n) for n in range(14)] == g["detail_cells"]
    for n, tab in g["morton"].items():
        n = int(n)
        assert [[pz.pz_morton_encode(i, j, n) for i in range(1 << n)] for j in range(1 << n)] == tab
    for i, j, n, r in g["morton_errors"]:
        assert pz.pz_morton_encode(i, j, n) == r
    for code, n, r, ii, jj in g["morton_decode"]:
        a, b = C.c_uint32(), C.c_uint32()
        assert pz.pz_morton_decode(code, n, C.byref(a), C.byref(b)) == r
        if r == 0:
            assert (a.value, b.value) == (ii, jj)
    for z, lv in g["level_of"]:
        assert pz.pz_level_of(z) == lv, z
    for n, m, Lv, r, kids in g["child_z_indices"]:
        o = (C.c_uint32 * 4)()
        assert pz.pz_child_z_indices(n, m, Lv, o) == r
        if r == 0:
            assert list(o) == kids
    for n, m, r in g["parent_z_index"]:
        assert pz.pz_parent_z_index(n, m) == r
    for n, m, Lv, fu, cu in g["finest_under"]:
        assert pz.pz_finest_under(n, m, Lv) == fu and pz.pz_cells_under(n, Lv) == cu
    for n, rows in g["neighbours"].items():
        n = int(n)
        for m, row in enumerate(rows):
            assert [pz.pz_same_level_neighbour(n, m, d) for d in range(4)] == row
            assert [pz.pz_neighbour_dev(n, m, d) for d in range(4)] == row


def test_oracle_matches_golden():
    for n, rows in GOLD["neighbours"].items():
        n = int(n)
        for m, row in enumerate(rows):
            assert [(-1 if O.neighbour(n, m, d) is None else O.neighbour(n, m, d)) for d in range(4)] == row
    for n, tab in GOLD["morton"].items():
        n = int(n)
        assert [[O.morton_encode(i, j) for i in range(1 << n)] for j in range(1 << n)] == tab


def test_bijectivity_and_dilated_neighbours(pz):
    """bijection for n <= 8 (exhaustive); the device dilated
    neighbour formula equals decode/shift/encode for every cell and direction."""
    import numpy as np

    for n in range(0, 9):
        side = 1 << n
        seen = np.zeros(side * side, bool)
        a, b = C.c_uint32(), C.c_uint32()
        for j in range(side):
            for i in range(side):
                m = pz.pz_morton_encode(i, j, n)
                assert 0 <= m < side * side and not seen[m]
                seen[m] = True
                assert pz.pz_morton_decode(m, n, C.byref(a), C.byref(b)) == 0 and (a.value, b.value) == (i, j)
        assert seen.all()
        if n <= 7:
            for m in range(side * side):
                for d in range(4):
                    assert pz.pz_neighbour_dev(n, m, d) == pz.pz_same_level_neighbour(n, m, d)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (no /root/reference here)")
def test_product_vs_live_reference(pz):
    R = C.CDLL(REF_SO)
    R.ref_same_level_neighbour.restype = C.c_int64
    R.ref_morton_encode.restype = C.c_int64
    import random

    rnd = random.Random(7)
    for _ in range(20000):
        n = rnd.randint(0, 13)
        m = rnd.randrange(1 << (2 * n))
        d = rnd.randrange(4)
        assert pz.pz_same_level_neighbour(n, m, d) == R.ref_same_level_neighbour(n, m, d)
        assert pz.pz_neighbour_dev(n, m, d) == R.ref_same_level_neighbour(n, m, d)
        i, j = rnd.randrange(1 << 14), rnd.randrange(1 << 14)
        assert pz.pz_morton_encode(i, j, n) == R.ref_morton_encode(i, j, n)
        z = rnd.randrange(int(GOLD["hierarchy_cells"][13]))
        assert pz.pz_level_of(z) == R.ref_level_of(z)
