"""Generate tests/golden/zorder_ref.json from the REFERENCE's own index algebra.

Runs oracle/_ref/libzorder_ref.so — /root/reference/proj/include/swamp/
zorder.hpp compiled where it lies by oracle/Makefile — and records its outputs
so the tests can pin the oracle and the product without /root/reference
(which does not exist on the GPU box). Re-run: `make -C oracle ref &&
python tests/golden/make_golden.py`.
"""
import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "..", "..", "oracle", "_ref", "libzorder_ref.so")


def main():
    L = C.CDLL(REF)
    L.ref_morton_encode.restype = C.c_int64
    L.ref_parent_z_index.restype = C.c_int64
    L.ref_same_level_neighbour.restype = C.c_int64
    L.ref_hierarchy_cells.restype = C.c_uint64
    L.ref_detail_cells.restype = C.c_uint64
    L.ref_level_offset.restype = C.c_uint32
    L.ref_finest_under.restype = C.c_uint32
    L.ref_cells_under.restype = C.c_uint32
    out = {"source": "/root/reference/proj/include/swamp/zorder.hpp via oracle/_ref/libzorder_ref.so"}
    out["level_offset"] = [L.ref_level_offset(n) for n in range(14)]
    out["hierarchy_cells"] = [L.ref_hierarchy_cells(n) for n in range(14)]
    out["detail_cells"] = [L.ref_detail_cells(n) for n in range(14)]
    # Morton tables for n <= 5 (row j, column i)
    out["morton"] = {str(n): [[L.ref_morton_encode(i, j, n) for i in range(1 << n)] for j in range(1 << n)]
                     for n in range(0, 6)}
    out["morton_errors"] = [[i, j, n, L.ref_morton_encode(i, j, n)] for (i, j, n) in
                            [(4, 0, 2), (0, 4, 2), (0, 0, -1), (0, 0, 14), (1 << 13, 0, 13), ((1 << 13) - 1, 5, 13)]]
    dec = []
    for n, code in [(2, 13), (2, 11), (2, 0), (2, 16), (3, 63), (13, (1 << 26) - 1), (14, 0)]:
        i, j = C.c_uint32(), C.c_uint32()
        r = L.ref_morton_decode(code, n, C.byref(i), C.byref(j))
        dec.append([code, n, r, i.value if r == 0 else None, j.value if r == 0 else None])
    out["morton_decode"] = dec
    # level_of at every level boundary (n <= 13) and a stride through
    lo = []
    for n in range(14):
        a = L.ref_level_offset(n)
        for z in (a, a + 1, max(a, L.ref_level_offset(n + 1) - 1) if n < 13 else a + 7):
            lo.append([z, L.ref_level_of(z)])
    out["level_of"] = lo
    kids = []
    for (n, m, Lv) in [(0, 0, 2), (1, 3, 2), (2, 7, 4), (1, 0, 1), (-1, 0, 3), (5, 1000, 9)]:
        o = (C.c_uint32 * 4)()
        r = L.ref_child_z_indices(n, m, Lv, o)
        kids.append([n, m, Lv, r, list(o) if r == 0 else None])
    out["child_z_indices"] = kids
    out["parent_z_index"] = [[n, m, L.ref_parent_z_index(n, m)] for (n, m) in [(2, 7), (1, 3), (0, 0), (5, 999), (13, 12345)]]
    out["finest_under"] = [[n, m, Lv, L.ref_finest_under(n, m, Lv), L.ref_cells_under(n, Lv)]
                           for (n, m, Lv) in [(0, 0, 4), (1, 3, 4), (3, 17, 8), (8, 100, 8), (2, 5, 11)]]
    nb = {}
    for n in range(0, 6):
        nb[str(n)] = [[L.ref_same_level_neighbour(n, m, d) for d in range(4)] for m in range(1 << (2 * n))]
    out["neighbours"] = nb
    with open(os.path.join(HERE, "zorder_ref.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote zorder_ref.json")


if __name__ == "__main__":
    main()
