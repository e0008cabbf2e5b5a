"""CPU-HWFV1 oracle baselines for BASELINE.md §5: every config at its
BASELINE level, a bounded number of steps after a short warm-up, at 1 thread
and at all host threads; ms/step and leaf updates/s. Oracle = test
infrastructure (this script only measures it). Writes one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
from paper_2206_05761_b200 import cases

CFGS = [("1_pseudo2d_L8", cases.pseudo2d_dambreak, dict(L=8), 40),
        ("2_humps_L9", cases.quiescent_humps, dict(L=9), 30),
        ("3_circular_L10_eps1e-3", cases.circular_dambreak, dict(L=10), 12),
        ("4_monai_L10", cases.monai_runup, dict(L=10), 12),
        ("5_river_L11", cases.river_flood, dict(L=11), 6)]
nproc = os.cpu_count() or 1
out = {"nproc": nproc}
for name, mk, kw, steps in CFGS:
    cfg, h, qx, qy, z = mk(**kw)
    row = {}
    for th in (1, nproc):
        O.set_threads(th)
        o = O.Oracle(cfg, h, qx, qy, z)
        o.step(2)
        n0 = o.counters()
        t0 = time.perf_counter()
        o.step(steps)
        dt = time.perf_counter() - t0
        leaves = o.info()["n_leaves"]
        row[f"threads_{th}"] = {"ms_per_step": 1e3 * dt / steps, "leaf_updates_per_s": leaves * steps / dt,
                                "steps": steps, "leaves_last": leaves}
        del o
    out[name] = row
    print(name, json.dumps(row), file=sys.stderr)
print(json.dumps(out))
