"""Back-to-back step time of the small / mid configs (humps L9, pseudo-2D L8,
circular L10, Monai L10) with the device stage timeline of the last step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_05761_b200 import cases, gpu

out = []
for name, mk in (("humpsL9", lambda: cases.quiescent_humps(L=9, t_end=1e30)),
                 ("p2dL8", lambda: cases.pseudo2d_dambreak(L=8, t_end=1e30)),
                 ("circL10", lambda: cases.circular_dambreak(L=10, t_end=1e30)),
                 ("monaiL10", lambda: cases.monai_runup(L=10, t_end=1e30))):
    cfg, h, qx, qy, z = mk()
    e = gpu.initialise(cfg, h, qx, qy, z)
    st = torch.cuda.ExternalStream(e.stream_ptr(), device=torch.device("cuda", 0))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e.advance(16); torch.cuda.synchronize()
    a.record(st); e.enqueue(64); b.record(st); b.synchronize()
    us = a.elapsed_time(b) / 64 * 1e3
    tl = e.timeline()
    out.append(f"{name} {us:.1f} us [prev {tl[1]:.1f} K1 {tl[0]:.1f}-{tl[2]:.1f} K2 {tl[3]:.1f}-{tl[5]:.1f} "
               f"K3 {tl[6]:.1f}-{tl[8]:.1f} K5 {tl[9]:.1f}-{tl[11]:.1f}]")
    e.close()
print(os.environ.get("TAG", "?").ljust(12), " | ".join(out))
