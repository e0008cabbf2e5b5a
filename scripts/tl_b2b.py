"""Device stage timeline of the last step of a back-to-back advance (8-step
graph replays): K1/K2/K3/K5 first-CTA start and last-CTA end (us from K1's
start), averaged over a few advances."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

for name, mk in (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(8)
    acc = [0.0] * 12
    n = 6
    for _ in range(n):
        e.advance(8)
        tl = e.timeline()
        acc = [a + b / n for a, b in zip(acc, tl)]
    e.close()
    s = f"prevFV1end:{acc[1]:.1f} " + " ".join(f"{k}:{acc[3*i]:.1f}-{acc[3*i+2]:.1f}" for i, k in enumerate(("K1", "K2", "K3", "K5")))
    print(os.environ.get("TAG", "?").ljust(28), name, s)
