"""Print the device stage timeline of a few profiled steps of config 5."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu
L = int(sys.argv[1]) if len(sys.argv) > 1 else 11
cfg, h, qx, qy, z = cases.river_flood(L=L)
e = gpu.initialise(cfg, h, qx, qy, z)
# stage times come from the device timeline (no event nodes)
for k in range(8):
    r = e.step_adaptive()
    if k >= 3:
        tl = e.timeline()
        print("K1 start/last/end", tl[0:3], "K2", tl[3:6], "K3", tl[6:9], "K5", tl[9:12],
              "| ev ms", round(r["ms_encode_flag"], 4), round(r["ms_band_closure"], 4),
              round(r["ms_decode_traverse"], 4), round(r["ms_fv1"], 4))
