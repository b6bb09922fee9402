"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): pack-group
partitioning and the gather of variable-size shards."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_01253_b200.distributed import _selftest_assemble, gather_packs, group_range


@pytest.mark.parametrize("n,world", [(0, 2), (1, 2), (2, 2), (56, 2), (56, 3), (645, 8), (7, 8)])
def test_group_range_partitions(n, world):
    rs = [group_range(n, r, world) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
        assert a1 == b0
    sizes = [g1 - g0 for g0, g1 in rs]
    assert max(sizes) - min(sizes) <= 1
    assert np.array_equal(_selftest_assemble(world, n), np.arange(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_groups, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g0, g1 = group_range(n_groups, rank, world)
        # each "pack" g is a deterministic (2, 5) block tagged by its group index
        local = torch.stack([torch.full((2, 5), g, dtype=torch.int64) for g in range(g0, g1)]) \
            if g1 > g0 else torch.empty((0, 2, 5), dtype=torch.int64)
        full = gather_packs(local, n_groups, world)
        cnt = torch.tensor([g1 - g0], dtype=torch.int64)
        dist.all_reduce(cnt)
        out_q.put((rank, full.numpy().copy(), int(cnt.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_groups", [(2, 5), (2, 1), (3, 56)])
def test_gather_packs_gloo(world, n_groups):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_groups, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.stack([np.full((2, 5), g, np.int64) for g in range(n_groups)])
    for rank, full, cnt in res:
        assert np.array_equal(full, want), rank
        assert cnt == n_groups
