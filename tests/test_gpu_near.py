"""Near-threshold cells (BASELINE north star: "except where a normalised
detail lies within FP tolerance of eps (such cells are counted and
reported)"; D7, D8).

The GPU evaluates SPEC.md:124's division form d_norm = max|d| / s_max (with
an exact screen, hwfv1::sig_class) and counts the cells with
|d_norm - eps 2^(n-L)| <= 1e-12 eps 2^(n-L) among those it re-encodes. The
oracle evaluates the same expression literally. The lattice cases put
hundreds of cells exactly on the threshold; flags, trees and counts must
match the oracle bit for bit and count for count, through the C-ABI's
StepReport.
"""
import pytest

from paper_2206_05761_b200 import cases
from tests._parity import compare_states

gpu = pytest.importorskip("paper_2206_05761_b200.gpu")
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

LATTICE = [(L, eps, still) for L in (7, 9) for eps in (2.0 ** -3, 2.0 ** -2, 0.0) for still in (False, True)]


@pytest.mark.parametrize("L,eps,still", LATTICE, ids=[f"L{a}-eps{b}-{'still' if c else 'moving'}" for a, b, c in LATTICE])
def test_near_threshold_lattice(L, eps, still):
    cfg, h, qx, qy, z = cases.threshold_lattice(L=L, epsilon=eps, still=still)
    g = gpu.initialise(cfg, h, qx, qy, z)
    o = O.Oracle(cfg, h, qx, qy, z)
    gn, on = g.near_threshold(), o.near_threshold()
    assert (gn["init"], gn["dem"]) == (on["init"], on["dem"]), (gn, on)
    if eps > 0:
        assert on["init"] > 0, "the lattice must put cells on the threshold"
    compare_states(g, o, "init")
    for k in range(1, 13):
        rep = g.step_adaptive()
        o.step()
        want = o.near_threshold()["last"]
        assert rep["n_near_threshold"] == want, f"step {k}: gpu {rep['n_near_threshold']} oracle {want}"
        if k in (1, 2, 6, 12):
            compare_states(g, o, f"step {k}")
    assert g.near_threshold()["total"] == o.near_threshold()["total"]
    g.advance(8)
    o.step(8)
    assert g.near_threshold()["total"] == o.near_threshold()["total"]
    compare_states(g, o, "advance")


@pytest.mark.parametrize("parts", [2, 4])
def test_near_threshold_partitioned(parts):
    """Virtual partitions count their own subtrees (and partition 0 the
    replicated top levels): the sums equal one engine's and the oracle's."""
    cfg, h, qx, qy, z = cases.threshold_lattice(L=9, epsilon=2.0 ** -2, still=True)
    many = gpu.initialise_partitioned(cfg, h, qx, qy, z, [0] * parts)
    o = O.Oracle(cfg, h, qx, qy, z)
    gn, on = many.near_threshold(), o.near_threshold()
    assert (gn["init"], gn["dem"]) == (on["init"], on["dem"])
    for k in range(1, 7):
        rep = many.step_adaptive()
        o.step()
        assert rep["n_near_threshold"] == o.near_threshold()["last"], f"step {k}"
    assert many.near_threshold()["total"] == o.near_threshold()["total"]
    compare_states(many, o, "partitioned")
