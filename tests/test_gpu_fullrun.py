"""Output-time parity over whole simulations (BASELINE configs 1-5 at their
benchmark levels): the GPU engine and the CPU oracle run each case from
initialise to t_end with dt clipped to the output times (D13),
and at every output time the leaf list, neighbour descriptors, significance
flags, every tree coefficient, the finest-grid expansion, t, dt and the
near-threshold counts (D8) must be identical — bit for bit, count for
count. This covers the regimes the short-horizon tests never reach: the
Monai N-wave's runup and the wetting of the beach (t ~ 10-17 s), late
friction, the hump dam break's long relaxation, every epsilon of config 3.

The oracle drives the pace (it is the slow side); the GPU advances the same
number of steps between output times through swamp_gpu_advance (CUDA graph
replays) and is compared there. Runtime on a 16-core host: a few minutes,
mostly Monai (about 9 k steps at L = 10).
"""
import numpy as np
import pytest

from paper_2206_05761_b200 import cases
from tests._parity import compare_states

gpu = pytest.importorskip("paper_2206_05761_b200.gpu")
from oracle import oracle as O  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RUNS = [
    # config 1: pseudo-2D dam break, L = 8, Stoker time 2.5 s and the 40 s performance horizon
    ("pseudo2d_dambreak", dict(L=8, t_end=40.0), [2.5, 10.0, 20.0, 30.0, 40.0]),
    # config 2: quiescent humps (C-property), L = 9, 100 s
    ("quiescent_humps", dict(L=9, t_end=100.0), [25.0, 50.0, 75.0, 100.0]),
    # config 3: circular dam break, L = 10, every epsilon of the sweep, 3.5 s
    ("circular_dambreak", dict(L=10, epsilon=1e-4), [1.0, 2.0, 3.5]),
    ("circular_dambreak", dict(L=10, epsilon=1e-3), [1.0, 2.0, 3.5]),
    ("circular_dambreak", dict(L=10, epsilon=1e-2), [1.0, 2.0, 3.5]),
    # config 4: Monai-like runup, L = 10, through the N-wave (peak ~10.5 s) to 22.5 s
    ("monai_runup", dict(L=10, t_end=22.5), [5.0, 10.0, 12.5, 15.0, 17.5, 20.0, 22.5]),
]


def _finest_equal(g, o, what):
    for name, a, b in zip(("h", "qx", "qy"), g.export_finest(), o.export_finest()):
        d = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
        assert d.size == 0, f"{what}: finest {name} differs at {d.size} cells"


@pytest.mark.parametrize("name,kw,outs", RUNS, ids=[f"{n}-" + "-".join(f"{k}{v}" for k, v in kw.items()) for n, kw, _ in RUNS])
def test_full_run_parity(name, kw, outs):
    cfg, h, qx, qy, z = cases.CASES[name](**kw)
    cfg.output_times = tuple(outs)
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    compare_states(g, o, f"{name} init")
    assert g.near_threshold()["init"] == o.near_threshold()["init"]
    assert g.near_threshold()["dem"] == o.near_threshold()["dem"]
    steps = 0
    for T in outs:
        k = 0
        while o.info()["t"] < T:
            o.step()
            k += 1
        assert o.info()["t"] == T, f"{name}: oracle did not stop on the output time {T}"
        g.advance(k)
        steps += k
        what = f"{name} t={T} (step {steps})"
        compare_states(g, o, what)
        _finest_equal(g, o, what)
        gn, on = g.near_threshold(), o.near_threshold()
        assert gn["total"] == on["total"], f"{what}: near-threshold cells {gn} vs {on}"
    assert g.info()["t"] == cfg.t_end


def test_river_l11_parity():
    """Config 5 (river flood, L = 11, the benchmark workload): 200 steps,
    compared after 1, 50, 100 and 200."""
    cfg, h, qx, qy, z = cases.river_flood(L=11)
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    done = 0
    for k in (1, 50, 100, 200):
        o.step(k - done)
        g.advance(k - done)
        done = k
        compare_states(g, o, f"river L11 step {k}")
        assert g.near_threshold()["total"] == o.near_threshold()["total"]
    _finest_equal(g, o, "river L11 step 200")
