"""Oracle: server round, client half, keyed permutations.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates:
  * _PrfStream / derive_permutation / invert     reference confidentiality.py:27-82
  * required_ksk_indices                          reference protocol.py:46-59
  * ServerEngine.server_round/_extract/_pack      reference protocol.py:219-321
  * Client.prepare_round / finish_round           reference protocol.py:324-396
  * run_inference                                 reference protocol.py:407-431

The oracle server takes the round matrix from ``lowering.round_matrix``
(dense; for small models) or a caller-supplied (W, bias) list, exactly as
the reference's engine consumes ``_round_mats``.
"""

from __future__ import annotations

import hashlib
import time
from dataclasses import dataclass

import numpy as np

from . import lowering, pack
from .keyswitch import (Ct, KsEngine, encrypt_batch, keygen, lift, make_ksk,
                        phase_batch)
from .scheme import U64, Scheme, dual_for


# ---------------------------------------------------------------------------
# keyed permutation (blake2b counter-mode PRF + descending Fisher-Yates)


class PrfStream:
    def __init__(self, key: bytes):
        self.key, self.ctr, self.buf = key, 0, b""

    def next_u64(self) -> int:
        while len(self.buf) < 8:
            self.buf += hashlib.blake2b(self.ctr.to_bytes(8, "little"), key=self.key,
                                        digest_size=64).digest()
            self.ctr += 1
        w, self.buf = self.buf[:8], self.buf[8:]
        return int.from_bytes(w, "little")

    def uniform_int(self, bound: int) -> int:
        span = bound + 1
        limit = (1 << 64) - ((1 << 64) % span)
        while True:
            u = self.next_u64()
            if u < limit:
                return u % span


def derive_permutation(master_seed: bytes, session_id: bytes, round_no: int, size: int):
    if size < 1:
        raise ValueError("permutation size must be >= 1")
    if round_no == 0:
        return np.arange(size, dtype=np.int64)
    sk = hashlib.blake2b(session_id, key=master_seed, digest_size=32).digest()
    rk = hashlib.blake2b(round_no.to_bytes(4, "little"), key=sk, digest_size=32).digest()
    s = PrfStream(rk)
    perm = np.arange(size, dtype=np.int64)
    for i in range(size - 1, 0, -1):
        j = s.uniform_int(i)
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def invert_permutation(perm):
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm), dtype=perm.dtype)
    return inv


def required_ksk_indices(scheme: Scheme) -> list[int]:
    R = scheme.ring
    idx = set()
    for j in range(max(scheme.gamma, 1), R.alpha):
        idx.update(pack.stage_reps_above(j, R)[1:])
    if scheme.gamma == 0:
        for ch in pack.stage0_chains(R):
            idx.update(ch[1:])
    return sorted(idx)


# ---------------------------------------------------------------------------
# server


@dataclass
class Stats:
    extract_s: float = 0.0
    linear_s: float = 0.0
    pack_s: float = 0.0
    key_switches: int = 0
    packed_coefficients: int = 0


class OracleServer:
    """Single-session CPU restatement of ServerEngine's round pipeline."""

    def __init__(self, model, scheme: Scheme, ksk, master_seed=bytes(32),
                 session_id=bytes(16), shuffle=True, ks_mode="exact",
                 round_mats=None, threads=1):
        self.model, self.scheme = model, scheme
        self.rounds = lowering.build_rounds(model.layers)
        self.seed, self.sid, self.shuffle = master_seed, session_id, shuffle
        self.engine = KsEngine(ksk, mode=ks_mode)
        self.counter = pack.Counter()
        self.unit = pack.bias_unit(scheme.gamma, scheme.ring)
        self.mats = round_mats if round_mats is not None else \
            [lowering.round_matrix(model.layers, r) for r in self.rounds]
        # thread pool over chunks / pack groups, as the reference engine (protocol.py:175-178)
        from concurrent.futures import ThreadPoolExecutor
        self.pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None

    def perm(self, r, size):
        if not self.shuffle:
            return np.arange(size, dtype=np.int64)
        return derive_permutation(self.seed, self.sid, r, size)

    def extract_all(self, bundles, total):
        R = self.scheme.ring
        jobs = [(b, min(R.N, total - j * R.N)) for j, b in enumerate(bundles)]
        one = lambda a: pack.extract(a[0], a[1], R)  # noqa: E731
        parts = list(self.pool.map(one, jobs)) if self.pool and len(jobs) > 1 else [one(a) for a in jobs]
        return np.concatenate(parts, axis=0)

    def pack_groups(self, out, max_groups=None):
        """ServerEngine._pack over (a prefix of) the pack groups (protocol.py:296-321)."""
        groups = pack.pad_groups(out, self.scheme.pack_factor, self.scheme.ring.N)
        if max_groups is not None:
            groups = groups[:max_groups]
        one = lambda g: pack.fast_pack(g, self.scheme, self.engine, counter=self.counter,  # noqa: E731
                                       skip_zero=True)
        if self.pool and len(groups) > 1:
            return list(self.pool.map(one, groups))
        return [one(g) for g in groups]

    def linear_rows(self, round_no, rows):
        """Unshuffle -> W -> shuffle (protocol.py:243-263)."""
        rnd = self.rounds[round_no - 1]
        main = rnd.input_len - rnd.skip_len
        canon = rows[:main][self.perm(round_no - 1, main)]
        if rnd.skip_len:
            sk = rows[main:rnd.input_len][self.perm(rnd.skip_source + 1, rnd.skip_len)]
            canon = np.concatenate([canon, sk], axis=0)
        W, bias = self.mats[round_no - 1]
        out = lowering.encrypted_linear(W, bias, canon, self.unit)
        if not rnd.final:
            out = out[invert_permutation(self.perm(round_no, rnd.output_len))]
        return out

    def server_round(self, round_no, bundles):
        st = Stats()
        t0 = time.perf_counter()
        rows = self.extract_all(bundles, self.rounds[round_no - 1].input_len)
        t1 = time.perf_counter()
        out = self.linear_rows(round_no, rows)
        t2 = time.perf_counter()
        before = self.counter.total_key_switches
        packs = self.pack_groups(out)
        t3 = time.perf_counter()
        st.extract_s, st.linear_s, st.pack_s = t1 - t0, t2 - t1, t3 - t2
        st.key_switches = self.counter.total_key_switches - before
        st.packed_coefficients = len(packs) * self.scheme.pack_factor
        return packs, st


# ---------------------------------------------------------------------------
# client


class OracleClient:
    """Client half with the reference's RNG draw order (protocol.py:324-390)."""

    def __init__(self, scheme: Scheme, seed: int = 1234):
        self.scheme, self.R = scheme, scheme.ring
        self.dual = dual_for(self.R.t, self.R.alpha, self.R.p_bits)
        self.rng = np.random.default_rng(seed)
        self.sk = keygen(self.R, scheme.key_dist, seed=int(self.rng.integers(0, 2 ** 62)))
        self.ksk = None

    def make_ksk(self):
        if self.ksk is None:
            self.ksk = make_ksk(self.sk, required_ksk_indices(self.scheme), self.scheme.gadget,
                                self.scheme.delta, self.rng, self.dual)
        return self.ksk

    def new_session_id(self) -> bytes:
        return self.rng.integers(0, 256, 16, dtype=np.uint8).tobytes()

    def prepare_round(self, v_signed, expected_len):
        R, p = self.R, self.R.p
        v = np.asarray(v_signed, np.int64).reshape(-1)
        if len(v) != expected_len:
            raise ValueError(f"round input length {len(v)} != expected {expected_len}")
        vm = v % p
        out = []
        for lo in range(0, expected_len, R.N):
            chunk = np.zeros(R.N, np.int64)
            piece = vm[lo:lo + R.N]
            chunk[:len(piece)] = piece
            if self.scheme.gamma == 0:
                exps, polys = [1], [chunk]
            else:
                pr = pack.client_powers(chunk, self.scheme.gamma, R)
                exps, polys = [d for d, _ in pr], [q for _, q in pr]
            payloads = np.stack([lift(q, R) for q in polys])
            batch = encrypt_batch(payloads, self.sk, self.scheme.delta, self.rng, self.dual)
            cts = {d: Ct(batch[i, 0], batch[i, 1], self.scheme.delta) for i, d in enumerate(exps)}
            out.append(pack.Bundle(self.scheme.gamma, cts))
        return out

    def finish_round(self, packed, rnd):
        F = self.scheme.pack_factor
        need = -(-rnd.output_len // F)
        if len(packed) != need:
            raise ValueError(f"expected {need} packed ciphertexts, got {len(packed)}")
        ph = phase_batch(np.stack(packed), self.sk)
        sh = 53 - self.R.p_bits
        res = (((ph + U64(1 << (sh - 1))) >> U64(sh)) & U64(self.R.p - 1)).astype(np.int64)
        vals = pack.read_packed_values(res, rnd.output_len, self.scheme)
        signed = np.where(vals >= self.R.p // 2, vals - self.R.p, vals)
        if rnd.final:
            return signed
        return lowering.requantize(lowering.activation(signed, rnd.activation), rnd.eta, rnd.clip)


def run_rounds(client: OracleClient, server_round, rounds, x):
    """Drive one inference: server_round(round_no, bundles) -> (packs, stats)."""
    v = np.asarray(x, np.int64).reshape(-1)
    hist, stats = [], []
    for rno, rnd in enumerate(rounds, start=1):
        if rnd.skip_len:
            skip = hist[rnd.skip_source] if rnd.skip_source >= 0 else np.asarray(x, np.int64).reshape(-1)
            v = np.concatenate([v, skip])
        bundles = client.prepare_round(v, rnd.input_len)
        packs, st = server_round(rno, bundles)
        stats.append(st)
        out = client.finish_round(packs, rnd)
        if rnd.final:
            return out, stats
        hist.append(out)
        v = out
    raise ValueError("model has no final round")
