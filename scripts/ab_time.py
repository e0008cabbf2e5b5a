"""A/B step timing of config 5 and the wet point with the basic API only
(works with older builds of the library: SWAMP_GPU_LIB=<path to .so>)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_05761_b200 import cases, gpu

def run(mk, steps=30, warm=5):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    st = torch.cuda.ExternalStream(e.stream_ptr(), device=torch.device("cuda", 0))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e.advance(warm); torch.cuda.synchronize()
    a.record(st); e.enqueue(steps); b.record(st); b.synchronize()
    b2b = a.elapsed_time(b) / steps * 1e3
    keys = ("ms_encode_flag", "ms_band_closure", "ms_decode_traverse", "ms_fv1")
    acc = [0.0] * 4
    for _ in range(steps):
        r = e.step_adaptive()
        for k, key in enumerate(keys):
            acc[k] += r[key] * 1e3 / steps
    e.close()
    return b2b, acc

out = {}
for name, mk in (("c5", lambda: cases.river_flood(L=11)), ("wet", lambda: cases.monai_runup(L=11))):
    out[name] = run(mk)
print(os.environ.get("TAG", "?").ljust(30), " ".join(f"{k}: step {v[0]:.1f} us K1/K2/K3/FV1 " + "/".join(f"{x:.1f}" for x in v[1]) for k, v in out.items()))
