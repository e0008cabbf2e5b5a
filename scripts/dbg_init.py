import sys
sys.path.insert(0, '.')
from paper_2206_05761_b200 import cases, gpu
for L in (3, 6, 7):
    cfg, h, qx, qy, z = cases.circular_dambreak(L=L)
    try:
        e = gpu.initialise(cfg, h, qx, qy, z)
        print(L, "ok", e.info())
    except Exception as ex:
        print(L, "fail", ex)
