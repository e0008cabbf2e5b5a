"""Workload for the compute-sanitizer tier: small
engines that exercise every kernel of the product library — initialise,
adaptive steps (K1, K2 + its top CTA, K3 top + subtrees, FV1 with the fused
re-encode), the near-threshold lattice, the uniform solver, inactive cells,
4 virtual partitions (peer tables, k_part_barrier, k_finalize), a rebalance,
and the exports (tree, Morton leaves + descriptors, finest grid, compare).

  compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_run.py [L]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2206_05761_b200 import cases, gpu  # noqa: E402


def main(L):
    runs = [
        ("river_flood", lambda: cases.river_flood(L=L)),
        ("monai_runup", lambda: cases.monai_runup(L=L)),
        ("lattice", lambda: cases.threshold_lattice(L=L, epsilon=2.0 ** -3, still=True)),
        ("nodata_river", lambda: cases.with_nodata_block(cases.river_flood, L=L)),
    ]
    for name, make in runs:
        cfg, h, qx, qy, z = make()
        e = gpu.initialise(cfg, h, qx, qy, z)
        for _ in range(3):
            e.step_adaptive()
        e.advance(9)  # one 8-step graph replay + one
        e.leaves()
        e.export_tree()
        e.export_finest()
        print(name, e.info(), e.near_threshold(), flush=True)
        e.close()
    cfg, h, qx, qy, z = cases.monai_runup(L=L)
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    u.step_uniform(4)
    a = gpu.initialise(cfg, h, qx, qy, z)
    a.advance(4)
    print("compare", a.compare(u), flush=True)
    u.close()
    a.close()
    if L >= 7:
        cfg, h, qx, qy, z = cases.rect_domain(cases.hump_dambreak, L=L)
        p = gpu.initialise_partitioned(cfg, h, qx, qy, z, [0] * 4)
        p.advance(5)
        p.rebalance()
        p.advance(5)
        p.leaves()
        p.export_finest()
        print("partitioned", p.info(), flush=True)
        p.close()
    # the L = 11 defaults forced on at this size: FV1's tile phase and the
    # stable-quiet skip (K2's change test, K3's skip state, K1 / FV1 skips).
    # Both K2 -> K3 paths: the cooperative fused grid (k_23, the default
    # below 1024 subtrees) and the split K3.
    os.environ.update({"SWAMP_FV1_TILES": "1", "SWAMP_QSKIP": "1"})
    for k23 in ("0", "1"):
        os.environ["SWAMP_K23"] = k23
        for name, make in runs[:2]:
            cfg, h, qx, qy, z = make()
            e = gpu.initialise(cfg, h, qx, qy, z)
            e.advance(12)
            e.step_adaptive()
            e.export_finest()
            print("forced", k23, name, e.info(), e.skips(), e.work()["tile_updates"], flush=True)
            e.close()
    # the stable-quiet skip needs dry subtrees: the Monai-like beach at L = 10
    cfg, h, qx, qy, z = cases.monai_runup(L=max(L, 10))
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(16)
    e.step_adaptive()
    e.export_tree()
    sk = e.skips()
    print("quiet skip", e.info(), sk, flush=True)
    assert sk["fv1_skipped_leaves"] > 0 and sk["k1_skipped_cells"] > 0, sk
    e.close()
    for k in ("SWAMP_FV1_TILES", "SWAMP_QSKIP", "SWAMP_K23"):
        os.environ.pop(k, None)
    gpu.trim_cache()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
