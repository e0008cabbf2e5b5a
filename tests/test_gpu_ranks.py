"""One process per partition on the GPU: two processes on one B200 (the box
has one GPU; NVLink peers on a multi-GPU node use the same code path)
exchange CUDA IPC blobs over gloo, step together through the device-side
barriers, repartition once (dynamic rebalance across processes) and
reproduce the one-engine result bitwise."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2206_05761_b200 import cases, gpu
    from paper_2206_05761_b200.ranks import torch_allgather

    cfg, h, qx, qy, z = cases.rect_domain(cases.hump_dambreak, L=7)  # inactive north part: unbalanced halves
    e = gpu.initialise_rank(cfg, h, qx, qy, z, rank, world, 0, torch_allgather)
    e.advance(steps // 2)
    moved = e.rebalance()  # every rank, same step (dynamic repartitioning)
    e.advance(steps - steps // 2)
    info = e.info()
    fin = e.export_finest()[0] if rank == 0 else None
    out.put((rank, info, None if fin is None else fin.tobytes(), moved))
    dist.barrier()
    e.close()
    dist.destroy_process_group()


def test_two_processes_ipc_equal_single():
    from paper_2206_05761_b200 import cases, gpu

    steps = 6
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(), q.get()], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    cfg, h, qx, qy, z = cases.rect_domain(cases.hump_dambreak, L=7)
    one = gpu.initialise(cfg, h, qx, qy, z)
    one.advance(steps)
    assert res[0][3] and res[1][3], "rebalance moved no boundary"
    assert res[0][1] == res[1][1] == one.info()
    np.testing.assert_array_equal(np.frombuffer(res[0][2], np.uint64), one.export_finest()[0].view(np.uint64).ravel())
