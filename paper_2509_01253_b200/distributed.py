"""Multi-GPU server rounds: pack groups sharded over ranks, one gather.

Partitioning per round (reference protocol.py:296-321 runs
the same pack groups on a host thread pool):

  1. every rank receives the round's uploads (the caller passes the same
     bundles on each rank, or rank 0's are broadcast) and the key set;
  2. every rank extracts all rows and evaluates the round map (replicated:
     under a random sigma_r each 16-row group of the linear map holds rows
     destined to every rank, so restricting it would not save work);
  3. rank g packs only its contiguous range of pack groups [g0, g1);
  4. one collective: the packed ciphertexts are gathered to every rank
     (all_gather, NCCL over NVLink) in group order; key-switch counts are
     summed with an all_reduce.

Packing is independent per group and every row is computed
deterministically, so the gathered result is bit-identical to one GPU's.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def group_range(n_groups: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous split of n_groups over world ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_groups, world)
    g0 = rank * base + min(rank, extra)
    return g0, g0 + base + (1 if rank < extra else 0)


def gather_packs(local: torch.Tensor, n_groups: int, world: int, group=None) -> torch.Tensor:
    """All-gather variable-size (g_r, 2, N) shards into the full (n_groups, 2, N) tensor."""
    shards = [group_range(n_groups, r, world) for r in range(world)]
    width = max(g1 - g0 for g0, g1 in shards)
    tail = tuple(local.shape[1:])
    padded = torch.zeros((width,) + tail, dtype=local.dtype, device=local.device)
    if local.shape[0]:
        padded[:local.shape[0]] = local
    out = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(out, padded, group=group)
    return torch.cat([o[:g1 - g0] for o, (g0, g1) in zip(out, shards)], dim=0)


class DistributedServerEngine:
    """SPMD wrapper: every rank calls server_round with the same arguments.

    Wraps one ``ServerEngine`` per rank (one process per GPU, torch.distributed
    initialised by the caller with backend "nccl").  Returns the full list of
    packed ciphertexts and RoundStats on every rank.
    """

    def __init__(self, engine, group=None):
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def register_client(self, ksk) -> bytes:
        return self.engine.register_client(ksk)

    def open_session(self, session_id: bytes, key_id: bytes):
        return self.engine.open_session(session_id, key_id)

    def server_round(self, session_id: bytes, round_no: int, bundles):
        """ServerEngine.server_round semantics (protocol checks, session state, extra
        noise, counters; reference protocol.py:219-280) with the pack groups sharded."""
        from .device import to_host_u64
        eng = self.engine
        with eng._lock:
            state = eng._check_round(session_id, round_no, len(bundles))
            rnd = eng.model.rounds[round_no - 1]
            F = eng.scheme.pack_factor
            G = -(-rnd.output_len // F)
            power, exps = eng._upload_bundles(bundles)
            eng._prefetch_perms(state, session_id, round_no + 1)
            in_map, out_map = eng.round_maps(state, session_id, round_no)
            im = torch.from_numpy(in_map).to(eng.dev)
            om = None if out_map is None else torch.from_numpy(out_map).to(eng.dev)
            g0, g1 = group_range(G, self.rank, self.world)
            key = eng.clients[state.key_id].key
            local, nks, times = eng.round_device(round_no, key, power, exps, im, om, groups=(g0, g1))
            full = gather_packs(local, G, self.world, self.group)
            cnt = torch.tensor([nks], dtype=torch.int64, device=local.device)
            dist.all_reduce(cnt, group=self.group)
            total = int(cnt.item())
            eng._finish_round(session_id, state, round_no, total)
            host = to_host_u64(full)
            packed = [host[i] for i in range(G)]
            # every rank's noise generator is seeded from the same master seed and advanced by
            # the same calls, so the noisy packs agree across ranks
            eng._apply_extra_noise(packed)
            return packed, eng._stats(total, times, len(bundles), G)


def _selftest_assemble(world: int, n_groups: int) -> np.ndarray:
    """Host-side model of the shard/gather assembly (used by the CPU gloo tests)."""
    parts = []
    for r in range(world):
        g0, g1 = group_range(n_groups, r, world)
        parts.append(np.arange(g0, g1))
    return np.concatenate(parts)
