"""Per-step cost of advance_reports (each step's report written into the
pinned ring by its finalize) against enqueue + one sync (no reports), config
5, wall clock over 64 steps after a warm-up."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_05761_b200 import cases, gpu

cfg, h, qx, qy, z = cases.river_flood(L=11)
e = gpu.initialise(cfg, h, qx, qy, z)
e.advance_reports(16); e.advance(16)
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); e.advance(64); t1 = time.perf_counter()
    t2 = time.perf_counter(); e.advance_reports(64); t3 = time.perf_counter()
    t4 = time.perf_counter()
    for _ in range(64): e.step_adaptive()
    t5 = time.perf_counter()
    print(f"advance {1e6*(t1-t0)/64:.1f} us/step  advance_reports {1e6*(t3-t2)/64:.1f}  step_adaptive {1e6*(t5-t4)/64:.1f}")
