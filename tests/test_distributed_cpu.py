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


# ---------------------------------------------------------------------------
# DistributedServerEngine.server_round: the protocol checks and session state of
# ServerEngine.server_round (reference protocol.py:219-280) on every rank.  The
# device round is stubbed (deterministic packs per group) so this runs on CPU.

def _stub_engine(extra_noise_std):
    import threading
    from types import SimpleNamespace

    from paper_2509_01253_b200.engine import ServerEngine, _SessionState
    from paper_2509_01253_b200.params import preset_for_bits

    eng = object.__new__(ServerEngine)
    eng.scheme = preset_for_bits(16, 0)
    N, F = eng.scheme.ring.N, eng.scheme.pack_factor
    mk = lambda i, o, final=False: SimpleNamespace(input_len=i, output_len=o, skip_len=0, skip_source=-1,
                                                  final=final)
    eng.model = SimpleNamespace(rounds=[mk(N + 5, 3 * F + 1), mk(3 * F + 1, F), mk(F, 10, True)])
    eng.master_seed = bytes(range(32))
    eng.shuffle_enabled = True
    eng.session_timeout = 300.0
    eng.extra_noise_std = extra_noise_std
    eng._noise_rng = np.random.default_rng(int.from_bytes(eng.master_seed[:8], "little") ^ 0x6E6F6973)
    eng._lock = threading.RLock()
    eng.total_key_switches = 0
    eng.clients = {b"k" * 16: SimpleNamespace(key=None)}
    eng.sessions = {}
    from concurrent.futures import ThreadPoolExecutor
    eng._perm_pool = ThreadPoolExecutor(max_workers=2)
    eng._pending = []
    eng.dev = torch.device("cpu")
    eng._upload_bundles = lambda bundles: (None, [1])

    def round_device(round_no, key, power, exps, im, om, groups=None, **kw):
        g0, g1 = groups
        packs = torch.stack([torch.full((2, N), 1000 * round_no + g, dtype=torch.int64)
                             for g in range(g0, g1)]) if g1 > g0 else torch.empty((0, 2, N), dtype=torch.int64)
        return packs, 7 * (g1 - g0), (0.0, 0.0, 0.0)

    eng.round_device = round_device
    sid = bytes(16)
    eng.sessions[sid] = _SessionState(key_id=b"k" * 16)
    return eng, sid


def _dist_engine_worker(rank, world, port, noise, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_01253_b200.distributed import DistributedServerEngine
        from paper_2509_01253_b200.engine import ERR_MALFORMED, ERR_STALE_ROUND, ProtocolError
        eng, sid = _stub_engine(noise)
        de = DistributedServerEngine(eng)
        codes = []
        for rno, nb in [(2, 2), (0, 2), (1, 1)]:  # out of order, round 0, wrong chunk count
            try:
                de.server_round(sid, rno, [None] * nb)
                codes.append(None)
            except ProtocolError as e:
                codes.append(e.code)
        assert codes == [ERR_STALE_ROUND, ERR_STALE_ROUND, ERR_MALFORMED], codes
        results = []
        for rno, nb in [(1, 2), (2, 1), (3, 1)]:
            packed, st = de.server_round(sid, rno, [None] * nb)
            results.append((np.stack(packed).copy(), st.key_switches))
            if rno < 3:
                assert eng.sessions[sid].next_round == rno + 1
        assert sid not in eng.sessions
        try:
            de.server_round(sid, 1, [None] * 2)
            stale = None
        except ProtocolError as e:
            stale = e.code
        out_q.put((rank, results, eng.total_key_switches, stale))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("noise", [0.0, 1e-9])
def test_distributed_server_round_protocol_gloo(noise):
    from paper_2509_01253_b200.engine import ERR_BAD_SESSION
    from paper_2509_01253_b200.params import preset_for_bits
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_dist_engine_worker, args=(r, world, port, noise, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sch = preset_for_bits(16, 0)
    F, N = sch.pack_factor, sch.ring.N
    groups = [4, 1, 1]
    for rank, results, total, stale in res:
        assert stale == ERR_BAD_SESSION
        assert total == 7 * sum(groups)
        for (packs, nks), rno, G in zip(results, (1, 2, 3), groups):
            assert packs.shape == (G, 2, N) and nks == 7 * G
            want = np.stack([np.full((2, N), 1000 * rno + g, np.uint64) for g in range(G)])
            assert np.array_equal(packs[:, 0], want[:, 0])
            if noise == 0.0:
                assert np.array_equal(packs, want)
            else:
                assert not np.array_equal(packs[:, 1], want[:, 1])
    # both ranks return identical packs (noise included)
    for (pa, _), (pb, _) in zip(res[0][1], res[1][1]):
        assert np.array_equal(pa, pb)
