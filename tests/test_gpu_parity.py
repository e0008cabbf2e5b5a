"""GPU (sm_100a, through the C-ABI) vs the CPU oracle on identical inputs.

The bar: leaf lists, neighbour descriptors, significance flags
and every scale coefficient on the tree are BIT-identical after initialise and
after every checked step; t and dt are bit-identical. The oracle is the
checker only.
"""
import numpy as np
import pytest

from paper_2206_05761_b200 import cases
from paper_2206_05761_b200.abi import BAND_NONE, BAND_PARENTS
from tests._parity import compare_states

gpu = pytest.importorskip("paper_2206_05761_b200.gpu")
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = [
    ("pseudo2d_dambreak", dict(L=6)),
    ("pseudo2d_dambreak", dict(L=8)),
    ("circular_dambreak", dict(L=7)),
    ("circular_dambreak", dict(L=8, epsilon=1e-2)),
    ("quiescent_humps", dict(L=7)),
    ("hump_dambreak", dict(L=7)),
    ("monai_runup", dict(L=7)),
    ("river_flood", dict(L=7)),
    ("pseudo2d_dambreak", dict(L=3)),
    ("circular_dambreak", dict(L=1)),
    ("circular_dambreak", dict(L=2)),
]


@pytest.mark.parametrize("name,kw", CASES, ids=[f"{n}-{'-'.join(f'{k}{v}' for k, v in kw.items())}" for n, kw in CASES])
def test_step_parity(name, kw):
    cfg, h, qx, qy, z = cases.CASES[name](**kw)
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    compare_states(g, o, f"{name} init")
    for k in range(1, 41):
        g.step_adaptive()
        o.step()
        if k in (1, 2, 3, 5, 10, 20, 40):
            compare_states(g, o, f"{name} step {k}")


def test_block_cache_reuse_is_clean():
    """Destroyed engines hand their device buffers (with stale contents) to the
    next engine of the same shape (swamp_gpu_trim_cache): a second engine on a
    different case, and a re-created first one, still match the oracle
    bitwise — no state survives in reused memory."""
    import gc

    def run(name, steps=12):
        cfg, h, qx, qy, z = cases.CASES[name](L=8)
        g = gpu.initialise(cfg, h, qx, qy, z)
        o = O.Oracle(cfg, h, qx, qy, z)
        for _ in range(steps):
            g.step_adaptive()
            o.step()
        compare_states(g, o, f"{name} after reuse")
        g.export_finest()
        del g
        gc.collect()

    gpu.trim_cache()
    run("circular_dambreak")
    run("hump_dambreak")      # reuses the first engine's blocks
    run("circular_dambreak")  # and back
    gpu.trim_cache()
    run("monai_runup")        # fresh blocks after a trim


def test_graph_advance_matches_single_steps():
    cfg, h, qx, qy, z = cases.circular_dambreak(L=8)
    a = gpu.initialise(cfg, h, qx, qy, z)
    b = gpu.initialise(cfg, h, qx, qy, z)
    for _ in range(19):
        a.step_adaptive()
    b.advance(19)
    (ah, *_), asig = a.export_tree()
    (bh, *_), bsig = b.export_tree()
    np.testing.assert_array_equal(asig, bsig)
    assert a.info() == b.info()
    fa = a.export_finest()[0]
    fb = b.export_finest()[0]
    np.testing.assert_array_equal(fa.view(np.uint64), fb.view(np.uint64))


@pytest.mark.parametrize("band", [BAND_NONE, BAND_PARENTS])
def test_band_modes(band):
    cfg, h, qx, qy, z = cases.pseudo2d_dambreak(L=7, band_mode=band)
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    for _ in range(15):
        g.step_adaptive()
        o.step()
    compare_states(g, o, f"band {band}")


def test_full_run_to_t_end():
    """Config 1 to t_end = 2.5 s: whole-run parity, finest expansion equal."""
    cfg, h, qx, qy, z = cases.pseudo2d_dambreak(L=7, t_end=2.5)
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    g.run()
    o.run()
    compare_states(g, o, "run")
    assert g.info()["t"] == 2.5
    for a, b in zip(g.export_finest(), o.export_finest()):
        np.testing.assert_array_equal(a.view(np.uint64), b.view(np.uint64))


def test_output_time_clipping():
    cfg, h, qx, qy, z = cases.hump_dambreak(L=6, t_end=1.0)
    cfg.output_times = (0.3, 0.7)
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    ts = []
    while g.info()["t"] < 1.0:
        g.step_adaptive()
        o.step()
        ts.append(g.info()["t"])
    compare_states(g, o, "clipped")
    assert 0.3 in ts and 0.7 in ts and ts[-1] == 1.0


def test_uniform_parity_and_eps0_equivalence():
    """step_uniform parity, and adaptive at eps = 0 == uniform (A4) bitwise."""
    cfg, h, qx, qy, z = cases.circular_dambreak(L=6, epsilon=0.0)
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    ou = O.Oracle(cfg, h, qx, qy, z, uniform=True)
    a = gpu.initialise(cfg, h, qx, qy, z)
    assert a.info()["n_leaves"] == 4 ** 6
    for _ in range(25):
        u.step_uniform(1)
        ou.step(uniform=True)
        a.step_adaptive()
    fu = u.export_finest()
    fo = ou.export_finest()
    fa = a.export_finest()
    for x, y, w in zip(fu, fo, fa):
        np.testing.assert_array_equal(x.view(np.uint64), y.view(np.uint64))
        np.testing.assert_array_equal(x.view(np.uint64), w.view(np.uint64))


def test_profiling_report_has_stage_times():
    cfg, h, qx, qy, z = cases.circular_dambreak(L=8)
    g = gpu.initialise(cfg, h, qx, qy, z)
    g.set_profiling(True)
    r = g.step_adaptive()
    assert r["ms_fv1"] > 0 and r["ms_encode_flag"] > 0 and r["ms_total"] >= r["ms_fv1"]
    assert r["n_leaves"] > 0 and r["step"] == 1


@pytest.mark.parametrize("parts,name,kw", [
    (2, "river_flood", dict(L=8)),
    (4, "circular_dambreak", dict(L=8)),
    (8, "monai_runup", dict(L=8)),
    (4, "pseudo2d_dambreak", dict(L=9)),
    (2, "quiescent_humps", dict(L=7)),
])
def test_partitioned_equals_single(parts, name, kw):
    """Morton-subtree partitions (virtual, on one GPU) == one partition, bitwise."""
    cfg, h, qx, qy, z = cases.CASES[name](**kw)
    one = gpu.initialise(cfg, h, qx, qy, z)
    many = gpu.initialise_partitioned(cfg, h, qx, qy, z, [0] * parts)
    compare_states(many, one, f"{name} x{parts} init")
    for k in range(1, 31):
        one.step_adaptive()
        many.step_adaptive()
        if k in (1, 2, 5, 30):
            compare_states(many, one, f"{name} x{parts} step {k}")
    many.advance(10)
    one.advance(10)
    compare_states(many, one, f"{name} x{parts} advance")
    for a, b in zip(many.export_finest(), one.export_finest()):
        np.testing.assert_array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("variant", ["l2-prefetch", "ahead", "ahead-flags", "tail"])
@pytest.mark.parametrize("name,kw", [("river_flood", dict(L=9)), ("monai_runup", dict(L=9))])
def test_active_subtree_paths(monkeypatch, variant, name, kw):
    """L = 9 (64 subtrees of 64 x 64): FV1's dry-subtree shortcut with each
    load-ahead stage of k_fv1 (SWAMP_FV1_STAGE 0 / 2 / 3 / 5) == the oracle,
    bitwise."""
    monkeypatch.setenv("SWAMP_FV1_STAGE", {"ahead": "2", "ahead-flags": "3", "tail": "5"}.get(variant, "0"))
    cfg, h, qx, qy, z = cases.CASES[name](**kw)
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    for k in range(1, 31):
        g.step_adaptive()
        o.step()
        if k in (1, 10, 30):
            compare_states(g, o, f"{name} {variant} step {k}")


@pytest.mark.parametrize("name,kw", [("river_flood", dict(L=9)), ("monai_runup", dict(L=9)),
                                     ("circular_dambreak", dict(L=9, epsilon=0.0)),
                                     ("circular_dambreak", dict(L=7, epsilon=0.0))])
def test_tile_path_parity(monkeypatch, name, kw):
    """FV1's tile path (active fully refined subtrees updated as 64 x 64
    blocks, every face computed once for both cells; default from L = 11,
    forced on here) == the oracle bitwise, and it is actually taken."""
    monkeypatch.setenv("SWAMP_FV1_TILES", "1")
    cfg, h, qx, qy, z = cases.CASES[name](**kw)
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    for k in range(1, 21):
        g.step_adaptive()
        o.step()
        if k in (1, 2, 10, 20):
            compare_states(g, o, f"{name} tiles step {k}")
    assert g.work()["tile_updates"] > 0, "no subtree took the tile path"


MASKED = [
    ("rect humps dambreak L7", lambda: cases.rect_domain(cases.hump_dambreak, L=7)),
    ("rect quiescent humps L7", lambda: cases.rect_domain(cases.quiescent_humps, L=7)),
    ("nodata river L8", lambda: cases.with_nodata_block(cases.river_flood, L=8)),
    ("nodata monai L7", lambda: cases.with_nodata_block(cases.monai_runup, L=7)),
]


@pytest.mark.parametrize("name,make", MASKED, ids=[m[0] for m in MASKED])
def test_inactive_cells_parity(name, make):
    """D16 inactive cells == the oracle, bitwise."""
    cfg, h, qx, qy, z = make()
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    compare_states(g, o, f"{name} init")
    for k in range(1, 31):
        g.step_adaptive()
        o.step()
        if k in (1, 10, 30):
            compare_states(g, o, f"{name} step {k}")


def test_inactive_cells_uniform_and_partitioned():
    cfg, h, qx, qy, z = cases.with_nodata_block(cases.river_flood, L=8)
    u = gpu.initialise_uniform(cfg, h, qx, qy, z)
    ou = O.Oracle(cfg, h, qx, qy, z, uniform=True)
    one = gpu.initialise(cfg, h, qx, qy, z)
    many = gpu.initialise_partitioned(cfg, h, qx, qy, z, [0] * 4)
    for _ in range(20):
        u.step_uniform(1)
        ou.step(uniform=True)
        one.step_adaptive()
        many.step_adaptive()
    for a, b in zip(u.export_finest(), ou.export_finest()):
        np.testing.assert_array_equal(a.view(np.uint64), b.view(np.uint64))
    compare_states(many, one, "nodata river x4")


@pytest.mark.parametrize("parts,name,kw", [(4, "pseudo2d_dambreak", dict(L=8)), (4, "monai_runup", dict(L=8)),
                                            (8, "monai_runup", dict(L=9))])
def test_rebalance_keeps_results(parts, name, kw):
    """Dynamic repartitioning: boundaries move to equalise
    the leaf counts, subtrees are pulled from their old owners, and the run
    stays bitwise equal to one partition."""
    cfg, h, qx, qy, z = cases.CASES[name](**kw)
    one = gpu.initialise(cfg, h, qx, qy, z)
    many = gpu.initialise_partitioned(cfg, h, qx, qy, z, [0] * parts)
    moved = 0
    for k in range(1, 31):
        one.step_adaptive()
        many.step_adaptive()
        if k % 5 == 0:
            moved += many.rebalance()
            compare_states(many, one, f"{name} x{parts} after rebalance at step {k}")
    assert moved > 0, "the leaf distribution never moved a boundary"
    many.advance(10)
    one.advance(10)
    compare_states(many, one, f"{name} x{parts} end")
