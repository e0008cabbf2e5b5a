"""One engine of a named case, `warm` steps, then `steps` more (ncu target:
capture the steady-state kernels with -s / -c). Usage:
python scripts/ncu_case.py <case> <L> [warm] [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05761_b200 import cases, gpu

name, L = sys.argv[1], int(sys.argv[2])
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 5
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
cfg, h, qx, qy, z = getattr(cases, name)(L=L)
e = gpu.initialise(cfg, h, qx, qy, z)
e.advance(warm)
for _ in range(steps):
    e.step_adaptive()
print(e.info(), e.work())
