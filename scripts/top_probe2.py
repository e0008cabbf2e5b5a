"""K3 top phases (SWAMP_EXP_TOPPROBE build): entry and stamps 0..6 plus the
fine stamps before the tile listing, the quiet classification, the skip
totals and the offsets (us after entry), config 5, last step of an advance."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu
cfg, h, qx, qy, z = cases.river_flood(L=11)
e = gpu.initialise(cfg, h, qx, qy, z)
for _ in range(3):
    e.advance(16)
    a = e.debug()
    t0 = a[16 + 7]
    st = [round((a[16 + i] - t0) / 1e3, 2) for i in range(7)]
    fine = [round((a[50 + i] - t0) / 1e3, 2) for i in range(4)]
    print("stamps0-6", st, "tiles/qs/sk/offsets", fine)
