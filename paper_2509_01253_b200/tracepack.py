"""Partial extraction and fast packing on the GPU (operator-level API).

Mirrors the operator seams of reference pkg/src/sfhr/tracepack.py:
``partial_extract`` (:118-154), ``extraction_payload_for_one`` (:157-172),
``fast_pack`` (:288-326) and ``pack_rows`` (:336-348), plus the schedule
helpers and ``KsCounter``.  The pack schedule (stage0 chains, per-level
merges, hoisted stages) runs on the device in one ``sfhr_pack`` call over
all pack groups at once, level-synchronously; each stage is one launch of the
fused key-switch kernel over every live row of every group.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .device import RingContext, to_dev, to_host_u64
from .params import Q_MASK, RingParams, SchemeParams, prime_factors_with_multiplicity, primitive_root


class KsCounter:
    """Thread-safe counters (reference tracepack.py:37-54)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.total_key_switches = 0
        self.packed_coefficients = 0

    def add_switches(self, n: int):
        with self._lock:
            self.total_key_switches += n

    def add_packed(self, n: int):
        with self._lock:
            self.packed_coefficients += n

    def per_coefficient(self) -> float:
        return self.total_key_switches / max(1, self.packed_coefficients)


def power_exponents(gamma: int, params: RingParams) -> list:
    """Client substitution exponents (reference tracepack.py:61-74)."""
    t, M = params.t, params.M
    if gamma == 0:
        return [1]
    if gamma == 1:
        return list(range(1, t))
    if gamma == 2:
        return sorted({(k * (j * t + 1)) % M for j in range(t) for k in range(1, t)})
    raise ValueError("extraction level gamma must be 0, 1 or 2")


@dataclass
class PowerBundle:
    """Encrypted chunk plus its encrypted automorphism powers (reference tracepack.py:93-111)."""
    gamma: int
    power_cts: dict

    def __post_init__(self):
        if self.gamma == 0 and set(self.power_cts) != {1}:
            raise ValueError("gamma=0 bundle carries only the base ciphertext")

    @property
    def base(self):
        return self.power_cts[1]

    def check(self, params: RingParams):
        want = set(power_exponents(self.gamma, params))
        if set(self.power_cts) != want:
            raise ValueError(f"bundle exponents {sorted(self.power_cts)} != required {sorted(want)}")


def check_bundle(bundle, params: RingParams):
    want = set(power_exponents(bundle.gamma, params))
    if set(bundle.power_cts) != want:
        raise ValueError(f"bundle exponents {sorted(bundle.power_cts)} != required {sorted(want)}")


def stack_bundles(bundles, params: RingParams) -> tuple[np.ndarray, list]:
    """(k, npow, 2, N) uint64 host array in ascending exponent order."""
    exps = sorted(bundles[0].power_cts)
    out = np.empty((len(bundles), len(exps), 2, params.N), np.uint64)
    for j, b in enumerate(bundles):
        check_bundle(b, params)
        for q, d in enumerate(exps):
            ct = b.power_cts[d]
            out[j, q, 0] = ct.a
            out[j, q, 1] = ct.b
    return out, exps


def extract_device(ctx: RingContext, power: torch.Tensor, exps, E: int) -> torch.Tensor:
    k = power.shape[0]
    rows = torch.empty((E, 2, ctx.N), dtype=torch.int64, device=ctx.dev)
    ex = np.asarray(exps, np.uint32)
    nat.check(nat.lib.sfhr_extract(ctx.h, nat.ptr(power), ex.ctypes.data, len(ex), k, E, nat.ptr(rows),
                                   ctx.stream()))
    return rows


def partial_extract(bundle, dual, count: int, params: RingParams, device: int = 0) -> np.ndarray:
    """Rows (count, 2, N) of the bottom-tower trace (reference tracepack.py:118-154).

    ``dual`` is accepted for signature parity; the device context derives the
    same two-term dual basis natively.
    """
    check_bundle(bundle, params)
    if count > params.N:
        raise ValueError(f"cannot extract {count} coefficients from a ring of degree {params.N}")
    ctx = RingContext.get(params.t, params.alpha, params.p_bits, 512, 3, 0, 0, device)
    power, exps = stack_bundles([bundle], params)
    rows = extract_device(ctx, to_dev(power, ctx.dev), exps, count)
    return to_host_u64(rows)


def extraction_payload_for_one(e1_0: int, e2_0: int, gamma: int, params: RingParams,
                               inv_m_mod_p: int) -> np.ndarray:
    """Body payload of a noiseless extracted '1' (reference tracepack.py:157-172)."""
    p, M, N, n1 = params.p, params.M, params.N, params.n1
    c = inv_m_mod_p - p if inv_m_mod_p > p // 2 else inv_m_mod_p
    step = 1 << (53 - params.p_bits)
    vec = np.zeros(M, np.int64)
    for d in power_exponents(gamma, params):
        vec[(e1_0 * d) % M] += c * step
        vec[(e2_0 * d) % M] -= c * step
    v = vec.astype(np.uint64) & np.uint64(Q_MASK)
    k = np.arange(N)
    return (v[:N] - v[N + k % n1]) & np.uint64(Q_MASK)


def stage0_chains(params: RingParams) -> list:
    g = primitive_root(params.t)
    out, stride = [], 1
    for ell in prime_factors_with_multiplicity(params.t - 1):
        out.append([pow(g, stride * u, params.M) for u in range(ell)])
        stride *= ell
    return out


def stage_reps_above(level_j: int, params: RingParams) -> list:
    return [(1 + i * params.t ** level_j) % params.M for i in range(params.t)]


def expected_pack_switches(t: int, alpha: int, beta: int, gamma: int) -> int:
    """Key switches per full pack group (reference tracepack.py:254-265)."""
    base = sum(l - 1 for l in prime_factors_with_multiplicity(t - 1))
    F = t ** (beta - 1) * (t - 1)
    tot = F * base if gamma == 0 else 0
    tot += sum(t ** (beta - j) * (t - 1) for j in range(1, beta) if j >= max(gamma, 1))
    tot += sum(t - 1 for j in range(beta, alpha) if j >= max(gamma, 1))
    return tot


def slot_positions(scheme: SchemeParams) -> np.ndarray:
    R = scheme.ring
    return np.arange(scheme.pack_factor) * (R.M // R.t ** scheme.beta_eff)


def pack_device(ctx: RingContext, key, rows: torch.Tensor, G: int, counter_dev, skip_zero=True):
    """Run the whole pack schedule for G groups; `rows` (G*F rows) is clobbered."""
    packs = torch.empty((G, 2, ctx.N), dtype=torch.int64, device=ctx.dev)
    ws_bytes = nat.lib.sfhr_pack_workspace_bytes(ctx.h, G)
    ws = torch.empty(max(1, ws_bytes // 8), dtype=torch.int64, device=ctx.dev)
    nat.check(nat.lib.sfhr_pack(ctx.h, key.h, nat.ptr(rows), G, nat.ptr(packs), nat.ptr(ws), ws_bytes,
                                int(skip_zero), nat.ptr(counter_dev), ctx.stream()))
    return packs


def _engine_ctx(engine, scheme: SchemeParams) -> RingContext:
    R = scheme.ring
    g = engine.ksk.gadget
    return RingContext.get(R.t, R.alpha, R.p_bits, g.D, g.l, scheme.gamma, scheme.beta,
                           engine.ctx.dev.index)


def _engine_key(engine, ctx):
    if engine.ctx is ctx:
        return engine.key
    cache = engine.__dict__.setdefault("_scheme_keys", {})
    if id(ctx) not in cache:
        from .device import DeviceKey
        cache[id(ctx)] = DeviceKey(ctx, engine.ksk)
    return cache[id(ctx)]


def fast_pack(cts, scheme: SchemeParams, engine, counter=None, skip_zero: bool = False):
    """Pack F extracted rows into one ciphertext (reference tracepack.py:288-326)."""
    R = scheme.ring
    F = scheme.pack_factor
    if tuple(cts.shape) != (F, 2, R.N):
        raise ValueError(f"fast_pack expects exactly {F} rows of shape (2, {R.N})")
    return pack_rows(cts, scheme, engine, counter=counter, skip_zero=skip_zero)[0]


def pack_rows(rows, scheme: SchemeParams, engine, counter=None, skip_zero: bool = True):
    """Pack E' rows into ceil(E'/F) ciphertexts, zero-padding the last group (tracepack.py:336-348)."""
    ctx = _engine_ctx(engine, scheme)
    key = _engine_key(engine, ctx)
    F = scheme.pack_factor
    host = not isinstance(rows, torch.Tensor)
    e = rows.shape[0]
    G = -(-e // F)
    buf = torch.zeros((G * F, 2, ctx.N), dtype=torch.int64, device=ctx.dev)
    if e:
        buf[:e] = to_dev(np.asarray(rows, np.uint64), ctx.dev) if host else rows
    cnt = ctx.counter()
    packs = pack_device(ctx, key, buf, G, cnt, skip_zero)
    if counter is not None:
        counter.add_switches(int(cnt.item()))
        counter.add_packed(F * G)
    if host:
        out = to_host_u64(packs)
        return [out[i] for i in range(G)]
    return [packs[i] for i in range(G)]
