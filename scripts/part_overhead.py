"""Partition overhead on one GPU: config 5 (L = 11) as 1 partition and as
2 / 4 / 8 virtual Morton-subtree partitions (default: each phase of every
partition as a concurrent graph branch, joined between phases; MODE=serial
(SWAMP_PART_CONCURRENT=0): every partition's phase k before phase k + 1 on
one stream), back-to-back step
time from CUDA events on the engine stream; all results bitwise equal
(tests/test_gpu_parity.py). Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_05761_b200 import cases, gpu

L = int(sys.argv[1]) if len(sys.argv) > 1 else 11
cfg, h, qx, qy, z = cases.river_flood(L=L)
if os.environ.get("MODE") == "serial":
    os.environ["SWAMP_PART_CONCURRENT"] = "0"
out = {"workload": f"river_flood_L{L}", "mode": os.environ.get("MODE", "concurrent"), "us_per_step": {}}
ref = None
for G in (1, 2, 4, 8):
    e = gpu.initialise(cfg, h, qx, qy, z) if G == 1 else gpu.initialise_partitioned(cfg, h, qx, qy, z, [0] * G)
    st = torch.cuda.ExternalStream(e.stream_ptr(), device=torch.device("cuda", 0))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e.advance(16)
    torch.cuda.synchronize()
    a.record(st)
    e.enqueue(64)
    b.record(st)
    b.synchronize()
    out["us_per_step"][G] = round(a.elapsed_time(b) / 64 * 1e3, 1)
    f = e.export_finest()[0]
    if ref is None:
        ref = f.copy()
    out.setdefault("bitwise_equal", {})[G] = bool(np.array_equal(f.view(np.uint64), ref.view(np.uint64)))
    e.close()
    gpu.trim_cache()
# the single partition with the one-partition-only features off (split K3,
# quiet split / skip, quadrant marks, FV1 tile phase): the partitions' own
# kernel path, so the ratio to it is the partitioning's overhead alone
os.environ.update({"SWAMP_K3_SPLIT": "0", "SWAMP_QSPLIT": "0", "SWAMP_FV1_TILES": "0"})
e = gpu.initialise(cfg, h, qx, qy, z)
st = torch.cuda.ExternalStream(e.stream_ptr(), device=torch.device("cuda", 0))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e.advance(16)
torch.cuda.synchronize()
a.record(st)
e.enqueue(64)
b.record(st)
b.synchronize()
m1 = a.elapsed_time(b) / 64 * 1e3
out["us_per_step_1_partition_path"] = round(m1, 1)
out["overhead_vs_1_partition_path"] = {G: round(out["us_per_step"][G] / m1, 3) for G in out["us_per_step"]}
e.close()
u = out["us_per_step"]
out["overhead_vs_1"] = {G: round(u[G] / u[1], 3) for G in u}
print(json.dumps(out))
