"""Multi-GPU host logic on CPU: the Morton-subtree partition plan, checked by
a world-size-2 gloo group: ranks agree on the plan, their
ranges tile the domain contiguously, every cell has exactly one owner, and
the concatenation of per-partition leaf slices (by finest Morton range) is
the global leaf list in Morton order — the property the
partitioned engine's exports rely on."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_05761_b200.partition import Plan


def test_plan_properties():
    for L in (7, 8, 9, 11):
        for G in (1, 2, 4, 8):
            p = Plan(L, G)
            if not p.valid():
                assert L - min(L, 6) < 2 and G == 8
                continue
            ranges = [p.finest_range(g) for g in range(G)]
            assert ranges[0][0] == 0 and ranges[-1][1] == 4 ** L
            assert all(ranges[g][1] == ranges[g + 1][0] for g in range(G - 1))
            for n in range(p.R, L + 1):
                for g in range(G):
                    lo, hi = p.level_slice(g, n)
                    assert p.owner(n, lo) == g and p.owner(n, hi - 1) == g
            # cells above R: owner = partition of their first subtree
            for n in range(p.R):
                for m in range(1 << (2 * n)):
                    assert p.owner(n, m) == p.owner(p.R, m << (2 * (p.R - n)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, L, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2206_05761_b200 import cases

    plan = Plan(L, world)
    # every rank computes the same tree (the oracle stands in for the engine
    # state) and keeps only the leaves of its Morton range
    cfg, h, qx, qy, z = cases.circular_dambreak(L=L)
    o = O.Oracle(cfg, h, qx, qy, z)
    o.step(3)
    leaves, _ = o.leaves()
    lv = np.floor(np.log2(3 * leaves.astype(np.int64) + 1)).astype(np.int64) // 2
    first = (leaves.astype(np.int64) - (4 ** lv - 1) // 3) << (2 * (L - lv))
    lo, hi = plan.finest_range(rank)
    mine = leaves[(first >= lo) & (first < hi)]
    gathered = [None] * world
    dist.all_gather_object(gathered, (plan.tile_range(rank), mine.tolist()))
    if rank == 0:
        out.put((gathered, leaves.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("L", [7, 8])
def test_gloo_two_partitions_concatenate_to_global_leaf_list(L):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, L, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    gathered, full = q.get()
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    (r0, l0), (r1, l1) = gathered
    assert r0[1] == r1[0]              # contiguous subtree ranges
    assert l0 + l1 == full             # Morton-order concatenation
    assert len(l0) > 0 and len(l1) > 0


def _blob_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2206_05761_b200.ranks import max_over_ranks, torch_allgather

    # a stand-in for this rank's CUDA IPC blob: fixed size, rank-specific bytes
    blob = bytes([rank]) * 7 + bytes(range(256)) * 4
    got = torch_allgather(blob[:1024])
    slowest = max_over_ranks(0.5 + rank)
    out.put((rank, [g[:8] for g in got], len(got[0]), slowest))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_rank_blob_exchange():
    """The one-process-per-GPU engine's host plumbing (ranks.py) on CPU:
    every rank receives every rank's IPC blob in rank order, and timings
    reduce to the max over ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_blob_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(), q.get()])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    for rank, heads, size, slowest in res:
        assert heads == [bytes([0]) * 7 + b"\x00", bytes([1]) * 7 + b"\x00"]
        assert size == 1024 and slowest == 1.5


def _rebalance_worker(rank, world, port, L, out):
    """One rank of a rebalance: it counts the leaves of its own subtrees (the
    oracle's leaf list stands in for the engine state), the ranks all-gather
    the counts, and each calls the ENGINE's planner (swamp_partition_plan,
    the host code behind swamp_gpu_rebalance) on the cumulative counts."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2206_05761_b200 import cases, gpu

    bounds0 = gpu.partition_plan(L, world)  # creation plan: equal subtree ranges
    R = L - min(L, 6)
    nt = 1 << (2 * R)
    cfg, h, qx, qy, z = cases.circular_dambreak(L=L)
    o = O.Oracle(cfg, h, qx, qy, z)
    o.step(3)
    leaves, _ = o.leaves()
    lv = np.floor(np.log2(3 * leaves.astype(np.int64) + 1)).astype(np.int64) // 2
    first = (leaves.astype(np.int64) - (4 ** lv - 1) // 3) << (2 * (L - lv))
    sub = first >> (2 * (L - R))  # each leaf's (first) subtree
    lo, hi = bounds0[rank], bounds0[rank + 1]
    mine = np.bincount(sub[(sub >= lo) & (sub < hi)], minlength=nt)[lo:hi]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine.tolist())
    counts = np.concatenate([np.asarray(g, dtype=np.uint64) for g in gathered])
    before = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    bounds = gpu.partition_plan(L, world, before)
    owners = [gpu.partition_owner(bounds, L, L, int(m)) for m in range(0, 4 ** L, 4 ** L // 64)]
    out.put((rank, bounds0, bounds, int(before[-1]), [int(before[b]) for b in bounds], owners, len(leaves)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("L,world", [(8, 2), (9, 4)])
def test_gloo_rebalance_plan_uses_engine_code(L, world):
    """Dynamic repartitioning's plan on CPU ranks, computed by the engine's
    own host code through the C-ABI: every rank gets the same contiguous
    boundaries, they cover every subtree, the leaf counts per partition are
    balanced to within the boundary granularity, and the engine's owner
    lookup (swamp_partition_owner, twin of the kernels' owner_of) agrees
    with them."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_rebalance_worker, args=(r, world, port, L, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get() for _ in range(world)])
    for pr in procs:
        pr.join(timeout=180)
        assert pr.exitcode == 0
    plans = {tuple(r[2]) for r in res}
    assert len(plans) == 1, plans  # every rank computed the same plan
    _, bounds0, bounds, total, cum, owners, nleaves = res[0]
    R = L - min(L, 6)
    nt = 1 << (2 * R)
    assert bounds0 == [g * nt // world for g in range(world + 1)]
    assert bounds[0] == 0 and bounds[-1] == nt and all(a < b for a, b in zip(bounds, bounds[1:]))
    assert total == nleaves
    per = [cum[g + 1] - cum[g] for g in range(world)]
    assert max(per) - min(per) <= max(per) * 0.5, per  # balanced (subtree granularity)
    step = 4 ** L // 64
    for k, g in enumerate(owners):
        t = (k * step) >> (2 * (L - R))
        assert bounds[g] <= t < bounds[g + 1]
