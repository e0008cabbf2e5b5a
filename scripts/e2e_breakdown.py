"""Where the e2e time of bench.py goes (L = 11): create, 50 steps, export."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_05761_b200 import cases, gpu
cfg, h, qx, qy, z = cases.river_flood(L=11)
torch.cuda.init()
h, qx, qy, z = (gpu.pinned_copy(a) for a in (h, qx, qy, z))
outs = [gpu.pinned_empty((2048, 2048)) for _ in range(3)]
e = gpu.initialise(cfg, h, qx, qy, z); del e  # warm (module load)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e = gpu.initialise(cfg, h, qx, qy, z)
    t1 = time.perf_counter()
    for _ in range(50):
        e.step_adaptive()
    t2 = time.perf_counter()
    e.export_finest(out=outs)
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms  50 steps (StepReport each) {1e3*(t2-t1):.2f} ms  export {1e3*(t3-t2):.2f} ms")
    del e
