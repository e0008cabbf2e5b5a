"""K3 top-CTA phase stamps (ctl->dbg slots 16..) of the last step of a
back-to-back advance: entry (7) then stamps 0..6, us after entry; and the
last subtree CTA's (slots 24..)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

for name, mk in (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    e.advance(16)
    a = e.debug()
    t0 = a[16 + 7]
    top = ",".join(str(round((a[16 + i] - t0) / 1e3, 2)) if a[16 + i] else "-" for i in range(7))
    last = ",".join(str(round((a[24 + i] - t0) / 1e3, 2)) if a[24 + i] else "-" for i in (7, 0, 1, 2, 3, 4, 6))
    print(os.environ.get("TAG", "?").ljust(10), name, "top:", top, "| last subtree (entry,0,1,2,3,4,6):", last)
    e.close()
