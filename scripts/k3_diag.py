import os, sys
sys.path.insert(0, os.getcwd())
from paper_2206_05761_b200 import cases, gpu
cfg, h, qx, qy, z = cases.river_flood(L=11)
e = gpu.initialise(cfg, h, qx, qy, z)
e.advance(5)
a0 = list(e.debug())
for k in range(20):
    e.step_adaptive()
a = e.debug()
d = [a[i] - a0[i] for i in range(64)]
print("end-time histogram (us bins from top entry):", d[48:64])
n = max(d[39], 1)
print("late CTAs", d[39], "mean entry", d[41] / n / 1e3, "phases (stage, count, wait, s_top, proj, emit):",
      [round(d[32 + k] / n / 1e3, 2) for k in range(5)] + [round(d[37] / n / 1e3, 2)])
