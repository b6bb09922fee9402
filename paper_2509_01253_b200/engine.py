"""ServerEngine drop-in: the reference's server round, on one B200.

Keeps the public surface of reference pkg/src/sfhr/protocol.py:145-321 —
``ServerEngine(model, scheme, master_seed, threads, shuffle_enabled,
ks_mode, session_timeout, extra_noise_std)``, ``register_client``,
``open_session``, ``server_round(session_id, round_no, bundles) ->
(packed, RoundStats)`` — and the protocol errors, so the client / wire /
session loop around it is unchanged.

Per round, on the device (one stream, no host round trips in between):
  1. H2D of the uploaded power bundles (k, npow, 2, N)
  2. partial extraction of all E_in rows            (extract_kernel)
  3. unshuffle sigma_{r-1} -> W_r -> shuffle sigma_r  (linear passes; the
     permutations are index maps inside the first/last pass)
  4. fast packing of all pack groups, level-synchronous (merge + fused
     key-switch stage kernels)
  5. D2H of the packed ciphertexts and the live key-switch count.
sigma_r comes from the C++ port of derive_permutation; round r+1's permutations
are derived on a host thread while round r runs on the GPU.
"""

from __future__ import annotations

import concurrent.futures
import functools
import hashlib
import json
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _native as nat
from .device import DeviceKey, RingContext, to_dev, to_host_u64
from .linear import DevicePass, run_round
from .model import QuantModel, lower_round
from .params import SchemeParams
from .tracepack import (extract_device, extraction_payload_for_one, pack_device,
                        power_exponents, stack_bundles, stage0_chains, stage_reps_above)

# wire error codes (reference wire.py:41-46)
ERR_STALE_ROUND = 1
ERR_BAD_SESSION = 2
ERR_BAD_TYPE = 3
ERR_MALFORMED = 4
ERR_PARAM_MISMATCH = 5
ERR_INTERNAL = 6
HEADER_SIZE = 35  # reference wire.py:29-32


class ProtocolError(Exception):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def required_ksk_indices(scheme: SchemeParams) -> list:
    """Automorphism indices the server needs (reference protocol.py:46-59)."""
    R = scheme.ring
    idx = set()
    for j in range(max(scheme.gamma, 1), R.alpha):
        idx.update(stage_reps_above(j, R)[1:])
    if scheme.gamma == 0:
        for ch in stage0_chains(R):
            idx.update(ch[1:])
    return sorted(idx)


def _block_size(m: int, count: int) -> int:
    return 4 + 4 + count * 2 * m * 8 + 1


def round_req_size(scheme: SchemeParams, k_chunks: int) -> int:
    """Analytic upload bytes (reference wire.py:265-268)."""
    npow = len(power_exponents(scheme.gamma, scheme.ring))
    per = 4 + 4 * npow + _block_size(scheme.ring.M, npow)
    return HEADER_SIZE + 4 + k_chunks * per


def round_resp_size(scheme: SchemeParams, n_packs: int) -> int:
    return HEADER_SIZE + 4 + _block_size(scheme.ring.M, n_packs)


@dataclass
class RoundMeta:
    input_len: int
    output_len: int
    activation: Optional[str]
    eta: int
    clip: tuple
    skip_source: int
    skip_len: int
    final: bool


@dataclass
class ModelMetadata:
    rounds: list
    input_shape: tuple
    input_clip: tuple
    num_classes: int
    t: int
    alpha: int
    p_bits: int
    gamma: int
    beta: int

    def to_json(self) -> str:
        return json.dumps({
            "rounds": [vars(r) | {"clip": list(r.clip)} for r in self.rounds],
            "input_shape": list(self.input_shape), "input_clip": list(self.input_clip),
            "num_classes": self.num_classes, "t": self.t, "alpha": self.alpha,
            "p_bits": self.p_bits, "gamma": self.gamma, "beta": self.beta}, sort_keys=True)


def metadata_for(model, scheme: SchemeParams) -> ModelMetadata:
    rounds = [RoundMeta(r.input_len, r.output_len, r.activation, r.eta, tuple(r.clip), r.skip_source,
                        r.skip_len, r.final) for r in model.rounds]
    return ModelMetadata(rounds, tuple(model.input_shape), tuple(model.input_clip), model.num_classes,
                         scheme.ring.t, scheme.ring.alpha, scheme.ring.p_bits, scheme.gamma,
                         scheme.beta_eff)


@dataclass
class RoundStats:
    extract_s: float = 0.0
    linear_s: float = 0.0
    pack_s: float = 0.0
    key_switches: int = 0
    packed_coefficients: int = 0
    bytes_up: int = 0
    bytes_down: int = 0


@dataclass
class _SessionState:
    key_id: bytes
    next_round: int = 1
    last_seen: float = field(default_factory=time.monotonic)
    perms: dict = field(default_factory=dict)   # (round, size) -> Future[np.ndarray]


@dataclass
class _ClientKeys:
    ksk: object
    key: DeviceKey
    scheme: SchemeParams


def _serialized(fn):
    """Run an engine entry point under the engine lock (see ServerEngine.__init__)."""
    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        with self._lock:
            return fn(self, *args, **kwargs)
    return wrapper


class ServerEngine:
    """Holds the model and per-client key material; executes server rounds on a B200."""

    MAX_QUEUED_PERMS = 64  # engine-wide cap on prefetched permutation derivations

    def __init__(self, model: QuantModel, scheme: SchemeParams, master_seed: bytes = b"\x00" * 32,
                 threads: int = 1, shuffle_enabled: bool = True, ks_mode: str = "cuda",
                 session_timeout: float = 300.0, extra_noise_std: float = 0.0, device: int = 0):
        if len(master_seed) != 32:
            raise ValueError("master seed must be 32 bytes")
        if model.acc_bits != scheme.ring.p_bits:
            raise ProtocolError(ERR_PARAM_MISMATCH,
                                "model accumulator width does not match plaintext modulus")
        if ks_mode not in ("cuda", "fft", "exact"):
            raise ValueError(f"unknown key-switch mode {ks_mode!r}")
        self.model = model
        self.scheme = scheme
        self.master_seed = master_seed
        self.threads = max(1, threads)
        self.shuffle_enabled = shuffle_enabled
        self.ks_mode = ks_mode
        self.session_timeout = session_timeout
        self.extra_noise_std = extra_noise_std
        self._noise_rng = np.random.default_rng(int.from_bytes(master_seed[:8], "little") ^ 0x6E6F6973)
        self.ctx = RingContext.for_scheme(scheme, device)
        self.dev = self.ctx.dev
        self.clients: dict = {}
        self.sessions: dict = {}
        R = scheme.ring
        unit = extraction_payload_for_one(int(self.ctx.e1[0]), int(self.ctx.e2[0]), scheme.gamma, R,
                                          self.ctx.inv_m_mod_p)
        self._bias_unit_host = unit
        self._bias_unit = to_dev(unit, self.dev)
        self._passes = [[DevicePass(p, self.dev) for p in lower_round(model, r)]
                        for r in range(len(model.rounds))]
        self._perm_pool = ThreadPoolExecutor(max_workers=4)
        self._pending: list = []  # queued / running permutation derivations (all sessions)
        # The reference serves one TCP connection per thread (transport.py:136-156), so
        # calls on different sessions may be concurrent; they share this engine's device
        # buffers, pinned staging and stream, so they run one at a time.
        self._lock = threading.RLock()
        self.total_key_switches = 0

    # -- setup ---------------------------------------------------------------

    @_serialized
    def register_client(self, ksk) -> bytes:
        needed = set(required_ksk_indices(self.scheme))
        have = set(ksk.indices())
        if not needed <= have:
            raise ProtocolError(ERR_PARAM_MISMATCH, f"key-switch keys missing indices {sorted(needed - have)}")
        key_id = hashlib.blake2b(repr(sorted(have)).encode() + np.asarray(ksk.keys[min(have)][0].a).tobytes(),
                                 digest_size=16).digest()
        if key_id not in self.clients:
            self.clients[key_id] = _ClientKeys(ksk=ksk, key=DeviceKey(self.ctx, ksk), scheme=self.scheme)
        return key_id

    def _round_perm_keys(self, round_no: int) -> list:
        """(round, size) keys of the permutations round round_no consumes (protocol.py:243-263)."""
        if not 1 <= round_no <= len(self.model.rounds):
            return []
        rnd = self.model.rounds[round_no - 1]
        keys = [(round_no - 1, rnd.input_len - rnd.skip_len)]
        if rnd.skip_len:
            keys.append((rnd.skip_source + 1, rnd.skip_len))
        if not rnd.final:
            keys.append((round_no, rnd.output_len))
        return keys

    def _prefetch_perms(self, state: _SessionState, session_id: bytes, round_no: int):
        """Queue the derivations of round round_no's permutations on the pool (C++, GIL
        released), so they run while the current round is on the GPU.

        Only one round ahead is prefetched per session (the reference derives each
        permutation lazily when its round runs, protocol.py:212-217), and nothing is
        queued once the engine already has MAX_QUEUED_PERMS derivations pending: a burst
        of opened or abandoned sessions cannot make later rounds wait behind them."""
        for key in self._round_perm_keys(round_no):
            if key in state.perms:
                continue
            self._pending = [f for f in self._pending if not f.done()]
            if len(self._pending) >= self.MAX_QUEUED_PERMS:
                return  # derived lazily by _perm when the round needs it
            fut = self._perm_pool.submit(self._perm_now, session_id, *key)
            self._pending.append(fut)
            state.perms[key] = fut

    @staticmethod
    def _cancel_perms(state: _SessionState):
        for fut in state.perms.values():
            fut.cancel()
        state.perms.clear()

    def _perm_now(self, session_id, round_no, size):
        if not self.shuffle_enabled or round_no == 0:
            return np.arange(size, dtype=np.int64)
        return nat.derive_permutation(self.master_seed, session_id, round_no, size)

    @_serialized
    def open_session(self, session_id: bytes, key_id: bytes) -> ModelMetadata:
        if key_id not in self.clients:
            raise ProtocolError(ERR_BAD_SESSION, "unknown key id")
        self._reap()
        if session_id in self.sessions:
            raise ProtocolError(ERR_BAD_SESSION, "session id already in use")
        st = _SessionState(key_id=key_id)
        self.sessions[session_id] = st
        self._prefetch_perms(st, session_id, 1)
        return metadata_for(self.model, self.scheme)

    def _reap(self):
        now = time.monotonic()
        for sid in [s for s, st in self.sessions.items() if now - st.last_seen > self.session_timeout]:
            self._cancel_perms(self.sessions.pop(sid))

    def _perm(self, state: _SessionState, session_id: bytes, round_no: int, size: int) -> np.ndarray:
        fut = state.perms.get((round_no, size))
        if fut is None or fut.cancelled():
            fut = concurrent.futures.Future()
            fut.set_result(self._perm_now(session_id, round_no, size))
            state.perms[(round_no, size)] = fut  # sigma_r is used again by round r+1 (unshuffle)
        return fut.result()

    def _finish_round(self, session_id: bytes, state: _SessionState, round_no: int, nks: int):
        """Session bookkeeping after a round (reference protocol.py:265-270)."""
        state.next_round += 1
        state.last_seen = time.monotonic()
        if round_no == len(self.model.rounds):
            self._cancel_perms(state)
            self.sessions.pop(session_id, None)
        else:  # keep only the permutations a later round still consumes (residual skips reach back)
            later = {k for q in range(round_no + 1, len(self.model.rounds) + 1) for k in self._round_perm_keys(q)}
            for k in [k for k in state.perms if k not in later]:
                state.perms.pop(k).cancel()
        self.total_key_switches += nks

    # -- round processing ------------------------------------------------------

    def _check_bundle_exponents(self, gammas, exps_per_bundle):
        """One rule for both entry points: every bundle must carry the engine's extraction
        level (the bias unit and the pack schedule are built for scheme.gamma; the
        reference checks each bundle against its own gamma only, tracepack.py:108-111,
        and would then combine mismatched rows) and exactly its power exponents."""
        want = sorted(power_exponents(self.scheme.gamma, self.scheme.ring))
        for g, exps in zip(gammas, exps_per_bundle):
            if g != self.scheme.gamma:
                raise ProtocolError(ERR_MALFORMED, f"bundle gamma {g} != engine gamma {self.scheme.gamma}")
            if list(exps) != want:
                raise ValueError(f"bundle exponents {list(exps)} != required {want}")

    def _upload_bundles(self, bundles):
        """Stage the uploads in pinned host memory and copy them to the device."""
        R = self.scheme.ring
        exps = sorted(bundles[0].power_cts)
        self._check_bundle_exponents([b.gamma for b in bundles], [sorted(b.power_cts) for b in bundles])
        shape = (len(bundles), len(exps), 2, R.N)
        n = int(np.prod(shape))
        if getattr(self, "_pinned", None) is None or self._pinned.numel() < n:
            self._pinned = torch.empty(n, dtype=torch.int64, pin_memory=True)
        host = self._pinned[:n].numpy().view(np.uint64).reshape(shape)
        for j, b in enumerate(bundles):
            for q, d in enumerate(exps):
                ct = b.power_cts[d]
                host[j, q, 0] = ct.a
                host[j, q, 1] = ct.b
        dev = self._pinned[:n].view(shape).to(self.dev, non_blocking=True)
        return dev, exps

    def round_maps(self, state, session_id, round_no):
        """(in_map, out_map) host int64 arrays for round round_no (protocol.py:243-263)."""
        rnd = self.model.rounds[round_no - 1]
        main = rnd.input_len - rnd.skip_len
        in_map = self._perm(state, session_id, round_no - 1, main)
        if rnd.skip_len:
            sk = self._perm(state, session_id, rnd.skip_source + 1, rnd.skip_len) + main
            in_map = np.concatenate([in_map, sk])
        out_map = None if rnd.final else self._perm(state, session_id, round_no, rnd.output_len)
        return in_map, out_map

    def _stage_to_host(self, t: torch.Tensor) -> torch.Tensor:
        """Enqueue device -> grow-only pinned staging buffer (valid after the next sync)."""
        n = t.numel()
        if getattr(self, "_pinned_out", None) is None or self._pinned_out.numel() < n:
            self._pinned_out = torch.empty(max(n, 1 << 17), dtype=torch.int64, pin_memory=True)
        stage = self._pinned_out[:n].view(t.shape)
        stage.copy_(t, non_blocking=True)
        return stage

    def _to_host_pinned(self, t: torch.Tensor) -> np.ndarray:
        """Device -> host through the pinned staging buffer (one DMA, one memcpy)."""
        stage = self._stage_to_host(t)
        torch.cuda.current_stream(self.dev).synchronize()
        return stage.numpy().view(np.uint64).copy()

    def _check_round(self, session_id: bytes, round_no: int, n_chunks: int):
        state = self.sessions.get(session_id)
        if state is None:
            raise ProtocolError(ERR_BAD_SESSION, "unknown or expired session")
        if round_no != state.next_round:
            raise ProtocolError(ERR_STALE_ROUND, f"expected round {state.next_round}, got {round_no}")
        if not (1 <= round_no <= len(self.model.rounds)):
            raise ProtocolError(ERR_STALE_ROUND, "round beyond model depth")
        rnd = self.model.rounds[round_no - 1]
        k_expected = -(-rnd.input_len // self.scheme.ring.N)
        if n_chunks != k_expected:
            raise ProtocolError(ERR_MALFORMED, f"expected {k_expected} chunks, got {n_chunks}")
        return state

    def _run_round(self, state, session_id: bytes, round_no: int, power, exps, fetch=None):
        keys = self.clients[state.key_id]

        def maps():
            in_map, out_map = self.round_maps(state, session_id, round_no)
            im = torch.from_numpy(in_map).to(self.dev, non_blocking=True)
            om = None if out_map is None else torch.from_numpy(out_map).to(self.dev, non_blocking=True)
            return im, om

        self._prefetch_perms(state, session_id, round_no + 1)  # derived while this round runs
        packs_dev, nks, times = self.round_device(round_no, keys.key, power, exps, maps, None, fetch=fetch)
        self._finish_round(session_id, state, round_no, nks)
        return packs_dev, nks, times

    def _stats(self, nks, times, n_chunks, n_packs):
        return RoundStats(extract_s=times[0], linear_s=times[1], pack_s=times[2], key_switches=nks,
                          packed_coefficients=n_packs * self.scheme.pack_factor,
                          bytes_up=round_req_size(self.scheme, n_chunks),
                          bytes_down=round_resp_size(self.scheme, n_packs))

    @_serialized
    def server_round(self, session_id: bytes, round_no: int, bundles: list):
        """Reference ServerEngine.server_round (protocol.py:219-280): bundles in, packed cts out."""
        state = self._check_round(session_id, round_no, len(bundles))
        power, exps = self._upload_bundles(bundles)
        # packs are copied into a fresh pinned block (torch's caching host allocator, so no
        # cudaHostAlloc per round) before the round's single sync; the returned arrays are
        # views that keep the block alive, so there is no host-side copy
        staged = []

        def fetch(p):
            host = torch.empty(p.shape, dtype=p.dtype, pin_memory=True)
            host.copy_(p, non_blocking=True)
            staged.append(host)

        packs_dev, nks, times = self._run_round(state, session_id, round_no, power, exps, fetch=fetch)
        packs_host = staged[0].numpy().view(np.uint64)
        packed = [packs_host[i] for i in range(packs_host.shape[0])]
        self._apply_extra_noise(packed)
        return packed, self._stats(nks, times, len(bundles), len(packed))

    def _apply_extra_noise(self, packed):
        """Optional host-side extra noise on the packed bodies (reference protocol.py:314-320)."""
        if self.extra_noise_std <= 0:
            return
        q = float(1 << 53)
        for pk in packed:
            extra = np.rint(self._noise_rng.normal(0.0, self.extra_noise_std, pk.shape[-1]) * q)
            pk[1] = (pk[1] + extra.astype(np.int64).astype(np.uint64)) & np.uint64((1 << 53) - 1)

    @_serialized
    def server_round_wire(self, session_id: bytes, round_no: int, payload) -> tuple:
        """ROUND_REQ payload bytes -> (ROUND_RESP payload bytes, RoundStats).

        The transport-facing form of server_round (reference ServerFrontend._round,
        transport.py:82-89, decode_round_req -> server_round -> encode_round_resp):
        the uploads are unpacked and range-checked on the GPU and the packed
        outputs are encoded from device memory (wire.py:99-124, 208-254).
        """
        from .wire import WireError, decode_round_req_device, encode_round_resp_device
        R = self.scheme.ring
        try:
            power, exps, gammas = decode_round_req_device(payload, R.N, self.dev)
        except WireError as e:
            raise ProtocolError(ERR_MALFORMED, e.reason) from e
        state = self._check_round(session_id, round_no, int(power.shape[0]))
        try:
            self._check_bundle_exponents(gammas, [exps] * len(gammas))
        except ValueError as e:
            raise ProtocolError(ERR_MALFORMED, str(e)) from e
        if self.extra_noise_std > 0:
            packed, st = self._round_from_device_with_noise(state, session_id, round_no, power, exps)
            noisy = torch.from_numpy(np.stack(packed).view(np.int64)).to(self.dev)
            return encode_round_resp_device(noisy, R.M, self.scheme.gamma), st
        packs_dev, nks, times = self._run_round(state, session_id, round_no, power, exps)
        resp = encode_round_resp_device(packs_dev, R.M, self.scheme.gamma)
        return resp, self._stats(nks, times, int(power.shape[0]), int(packs_dev.shape[0]))

    def _round_from_device_with_noise(self, state, session_id, round_no, power, exps):
        packs_dev, nks, times = self._run_round(state, session_id, round_no, power, exps)
        packs_host = to_host_u64(packs_dev)
        packed = [packs_host[i] for i in range(packs_host.shape[0])]
        self._apply_extra_noise(packed)
        return packed, self._stats(nks, times, int(power.shape[0]), len(packed))

    def round_device(self, round_no: int, key: DeviceKey, power, exps, in_map, out_map,
                     timed: bool = True, groups: Optional[tuple] = None, counter=None, fetch=None):
        """Device part of one round. power: host (k, npow, 2, N) uint64 or device tensor;
        in_map / out_map: device int64 tensors (out_map None for the final round), or
        in_map a callable returning both, called once the extraction is launched.

        groups=(g0, g1) packs only that range of pack groups (multi-GPU sharding,
        SURVEY §8(e)); extraction and the linear map are computed in full.
        counter: optional device int64 accumulator; when given the call does not
        synchronise and returns key_switches=None (the caller reads the counter).
        fetch: optional callable run on the packs after the last launch, before the sync.
        Returns (packs_dev, key_switches, (extract_s, linear_s, pack_s)).
        """
        rnd = self.model.rounds[round_no - 1]
        ctx = self.ctx
        F = self.scheme.pack_factor
        stream = torch.cuda.current_stream(self.dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timed else None
        if ev:
            ev[0].record(stream)
        pw = power if isinstance(power, torch.Tensor) else to_dev(power, self.dev)
        rows = extract_device(ctx, pw, exps, rnd.input_len)
        if ev:
            ev[1].record(stream)
        if callable(in_map):  # lazy maps: derived / uploaded while the extraction runs
            in_map, out_map = in_map()
        G = -(-rnd.output_len // F)
        buf = torch.empty((G * F, 2, ctx.N), dtype=torch.int64, device=self.dev)
        if G * F > rnd.output_len:
            buf[rnd.output_len:].zero_()  # zero padding of the last group (protocol.py:300-303)
        run_round(ctx, self._passes[round_no - 1], rows, in_map, buf, out_map, self._bias_unit)
        if ev:
            ev[2].record(stream)
        cnt = ctx.counter() if counter is None else counter
        g0, g1 = (0, G) if groups is None else groups
        packs = pack_device(ctx, key, buf[g0 * F:g1 * F], g1 - g0, cnt, skip_zero=True)
        if ev:
            ev[3].record(stream)
        if fetch is not None:  # e.g. enqueue the D2H of the packs ahead of the sync below
            fetch(packs)
        if counter is not None:
            return packs, None, (0.0, 0.0, 0.0)
        nks = int(cnt.item())  # synchronises the stream
        times = (0.0, 0.0, 0.0)
        if ev:
            times = tuple(ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(3))
        return packs, nks, times
