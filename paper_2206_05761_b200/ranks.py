"""Host plumbing of the one-process-per-GPU engine (no device code here).

Each torchrun rank owns one Morton-subtree partition: it
creates its partition (gpu.initialise_rank), and the ranks exchange the
CUDA IPC blobs of the arrays their peers read in place. The exchange is an
all-gather of equal-size byte strings in rank order over torch.distributed
(gloo on the host: the blobs are tiny and exchanged once).
"""
from __future__ import annotations


def torch_allgather(blob: bytes) -> list:
    """All-gather one byte string per rank, returned in rank order."""
    import torch
    import torch.distributed as dist

    ws = dist.get_world_size()
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8).clone()
    n = torch.tensor([t.numel()], dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(ws)]
    dist.all_gather(sizes, n)
    if any(int(s.item()) != t.numel() for s in sizes):
        raise ValueError("rank blobs differ in size")
    out = [torch.empty_like(t) for _ in range(ws)]
    dist.all_gather(out, t)
    return [bytes(o.numpy().tobytes()) for o in out]


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar (timings: the slowest rank bounds the step)."""
    import torch
    import torch.distributed as dist

    v = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return float(v.item())
