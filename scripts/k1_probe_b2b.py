"""K1 phase stamps (first / last CTA) of the last step of a back-to-back
advance, config 5 and the wet point: entry (after the PDL wait) -> loads
issued (0), staged (1), level L-1 flags (2), levels done (4), end (5)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

for name, mk in (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(16)
    a = e.debug()
    t0 = min(a[7], a[15])
    out = []
    for c, lab in ((0, "first"), (8, "last")):
        out.append(f"{lab} entry {round((a[c + 7] - t0) / 1e3, 2)} ->" +
                   ",".join(str(round((a[c + i] - a[c + 7]) / 1e3, 2)) if a[c + i] else "-" for i in (0, 1, 2, 4, 5)))
    print(os.environ.get("TAG", "?").ljust(16), name, " | ".join(out))
    e.close()
