"""Stage stamps of the small configs (humps L9, pseudo-2D L8): K1 first/last
CTA (entry -> 0,1,2,4,5), K3 top (entry then 0..6) and its last subtree CTA,
and the step timeline, all of the last step of a back-to-back advance."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

for name, mk in (("humpsL9", lambda: cases.quiescent_humps(L=9, t_end=1e30)),
                 ("p2dL8", lambda: cases.pseudo2d_dambreak(L=8, t_end=1e30))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(16)
    a = e.debug()
    tl = e.timeline()
    t0 = min(a[7], a[15])
    k1 = []
    for c, lab in ((0, "first"), (8, "last")):
        k1.append(f"{lab} entry {round((a[c + 7] - t0) / 1e3, 2)} ->" +
                  ",".join(str(round((a[c + i] - a[c + 7]) / 1e3, 2)) if a[c + i] else "-" for i in (0, 1, 2, 4, 5)))
    t3 = a[16 + 7]
    top = ",".join(str(round((a[16 + i] - t3) / 1e3, 2)) if a[16 + i] else "-" for i in range(7))
    last = ",".join(str(round((a[24 + i] - t3) / 1e3, 2)) if a[24 + i] else "-" for i in (7, 0, 1, 2, 3, 4, 6))
    print(name, "K1:", " | ".join(k1))
    print(name, "K3 top (from entry):", top, "| last subtree (entry,0,1,2,3,4,6):", last,
          f"| K3 entry at {round((t3 - t0) / 1e3, 2)} after K1 entry")
    print(name, "timeline", [round(x, 1) for x in tl[:12]])
    e.close()
