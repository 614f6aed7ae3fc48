"""Multi-process host logic on CPU (gloo, world_size 2): the r-slab partition
 tiles the grid, the slab gather reassembles the r-fastest array, the
NCCL id broadcast path, and the deterministic fixed-order dot combination
 the library applies after its all-gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1709_01126_b200 import PC1, PC2, gather_slabs, slab_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nr, nt, np_ = 11, 5, 7
        full = np.arange(nr * nt * np_, dtype=np.float64).reshape(np_, nt, nr)  # r fastest
        out = {}
        for pc, blocks in ((PC1, 1), (PC2, 1), (PC2, 3)):
            i0, i1 = slab_bounds(nr, world, rank, blocks, pc)
            got = gather_slabs(full[:, :, i0:i1].copy(), nr)
            bounds = [None] * world
            dist.all_gather_object(bounds, (i0, i1))
            if rank == 0:
                out[(pc, blocks)] = (np.array_equal(got.numpy(), full), bounds)
        # NCCL-id style broadcast of 128 opaque bytes (the ctypes id path)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ok_bcast = obj[0] == bytes(range(128))
        # fixed-order combination of all-gathered partial sums: bit-identical on all ranks
        rng = np.random.default_rng(rank)
        local = torch.tensor(rng.standard_normal(2))
        gathered = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, local)
        tot = 0.0
        for g in gathered:  # rank order, like k_finalize_* on the device
            tot += float(g[0])
        allt = [None] * world
        dist.all_gather_object(allt, tot)
        q.put((rank, out, ok_bcast, len(set(allt)) == 1))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_two_ranks():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    out = res[0][1]
    for key, (ok, bounds) in out.items():
        assert ok, key
        # contiguous, covering, leading ranks take the remainder
        assert bounds[0][0] == 0 and bounds[-1][1] == 11
        assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))
        widths = [b - a for a, b in bounds]
        assert widths == sorted(widths, reverse=True)
    assert all(r[2] for r in res) and all(r[3] for r in res)


def test_slab_bounds_rules():
    # PC1: 151 shells on 8 ranks -> 19 x7 + 18 (leading remainder)
    w = [slab_bounds(151, 8, r)[1] - slab_bounds(151, 8, r)[0] for r in range(8)]
    assert w == [19] * 7 + [18]
    # PC2 with 2 blocks per rank: rank slab = union of its blocks of the 16-way split
    b = [slab_bounds(151, 8, r, 2, PC2) for r in range(8)]
    assert b[0] == (0, 20) and b[-1][1] == 151
    assert sum(y - x for x, y in b) == 151
