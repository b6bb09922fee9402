"""Oracle: partial-trace extraction, tower stages, fast packing.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates:
  * KsCounter                                   reference tracepack.py:37-54
  * power_exponents / client_powers / bundles   reference tracepack.py:61-111
  * partial_extract                             reference tracepack.py:118-154
  * extraction_payload_for_one (bias unit)      reference tracepack.py:157-172
  * stage0_chains / stage_reps_above / counts   reference tracepack.py:179-265
  * fast trace (message-level test helper)      reference tracepack.py:217-242
  * _apply_stage_batch / fast_pack / pack_rows  reference tracepack.py:268-348
  * slot_positions / read_packed_values         reference tracepack.py:329-358
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from .scheme import (U64, UMASK, Ring, Scheme, automorph, centered_inv_m,
                     dual_for, factor_multiset, fold, mono_shift,
                     smallest_generator)


class Counter:
    def __init__(self):
        self._lk = threading.Lock()
        self.total_key_switches = 0
        self.packed_coefficients = 0

    def add_switches(self, n):
        with self._lk:
            self.total_key_switches += n

    def add_packed(self, n):
        with self._lk:
            self.packed_coefficients += n

    def per_coefficient(self):
        return self.total_key_switches / max(1, self.packed_coefficients)


def power_exponents(gamma: int, R: Ring) -> list[int]:
    t, M = R.t, R.M
    if gamma == 0:
        return [1]
    if gamma == 1:
        return list(range(1, t))
    if gamma == 2:
        return sorted({(k * (j * t + 1)) % M for j in range(t) for k in range(1, t)})
    raise ValueError("extraction level gamma must be 0, 1 or 2")


def client_powers(m, gamma: int, R: Ring):
    if gamma == 0:
        return []
    m = np.asarray(m, dtype=np.int64)
    return [(d, automorph(m, d, R) % R.p) for d in power_exponents(gamma, R)]


@dataclass
class Bundle:
    gamma: int
    power_cts: dict

    def __post_init__(self):
        if self.gamma == 0 and set(self.power_cts) != {1}:
            raise ValueError("gamma=0 bundle carries only the base ciphertext")

    @property
    def base(self):
        return self.power_cts[1]

    def check(self, R: Ring):
        want = set(power_exponents(self.gamma, R))
        if set(self.power_cts) != want:
            raise ValueError(f"bundle exponents {sorted(self.power_cts)} != required {sorted(want)}")


def extract(bundle, count: int, R: Ring) -> np.ndarray:
    """Rows (count, 2, N) of the bottom-tower trace of m*conj(dual_i).

    Row i, before the fold, is  sum_d cu * (ct_d[(x)] - ct_d[(x - c_i n1 d)])
    read at x = (i*d + m) mod M (tracepack.py:138-154), with ct_d zero-padded
    to length M and c_i = ratio_len[i].
    """
    Bundle.check(bundle, R)
    if count > R.N:
        raise ValueError(f"cannot extract {count} coefficients from a ring of degree {R.N}")
    M, N, n1 = R.M, R.N, R.n1
    dual = dual_for(R.t, R.alpha, R.p_bits)
    cu = U64(centered_inv_m(R) % (1 << 64))
    i = np.arange(count)
    c = dual.c[:count]
    m = np.arange(M)
    acc = np.zeros((count, 2, M), U64)
    for d, ct in bundle.power_cts.items():
        pw = np.zeros((2, M), U64)
        pw[0, :N] = ct.a
        pw[1, :N] = ct.b
        pw = (pw * cu) & UMASK
        x = (i[:, None] * d + m[None, :]) % M
        y = (x - (c[:, None] * n1 * d)) % M
        acc += (pw[:, x] - pw[:, y]).transpose(1, 0, 2)
    acc &= UMASK
    return fold(acc, R)


def bias_unit(gamma: int, R: Ring) -> np.ndarray:
    """Body payload of a noiseless extracted '1' (tracepack.py:157-172)."""
    dual = dual_for(R.t, R.alpha, R.p_bits)
    c = centered_inv_m(R)
    step = 1 << (53 - R.p_bits)
    vec = np.zeros(R.M, np.int64)
    for d in power_exponents(gamma, R):
        vec[(int(dual.e1[0]) * d) % R.M] += c * step
        vec[(int(dual.e2[0]) * d) % R.M] -= c * step
    return fold(vec.astype(U64) & UMASK, R)


def stage0_chains(R: Ring) -> list[list[int]]:
    g = smallest_generator(R.t)
    out, stride = [], 1
    for ell in factor_multiset(R.t - 1):
        out.append([pow(g, stride * u, R.M) for u in range(ell)])
        stride *= ell
    return out


def stage_reps_above(j: int, R: Ring) -> list[int]:
    return [(1 + i * R.t ** j) % R.M for i in range(R.t)]


def expected_pack_switches(t, alpha, beta, gamma) -> int:
    base = sum(l - 1 for l in factor_multiset(t - 1))
    F = t ** (beta - 1) * (t - 1)
    tot = F * base if gamma == 0 else 0
    tot += sum(t ** (beta - j) * (t - 1) for j in range(1, beta) if j >= max(gamma, 1))
    tot += sum(t - 1 for j in range(beta, alpha) if j >= max(gamma, 1))
    return tot


def expected_trace_switches(R: Ring, from_level=None, to_level=0) -> int:
    fr = R.alpha if from_level is None else from_level
    tot = 0
    for lv in range(fr, to_level, -1):
        tot += (R.t - 1) if lv >= 2 else sum(l - 1 for l in factor_multiset(R.t - 1))
    return tot


def fast_trace(ct, engine, from_level, to_level, counter=None):
    """Homomorphic partial trace along the tower (tracepack.py:217-242)."""
    from .keyswitch import Ct
    R = engine.params
    cur = ct
    for lv in range(from_level, to_level, -1):
        groups = [stage_reps_above(lv - 1, R)] if lv >= 2 else stage0_chains(R)
        for reps in groups:
            acc = cur
            for rep in reps[1:]:
                sw = engine.homomorphic_automorphism(cur, rep, counter)
                acc = Ct((acc.a + sw.a) & UMASK, (acc.b + sw.b) & UMASK)
            cur = acc
    return cur


def apply_stage(x, reps, engine, counter, skip_zero):
    """acc = x + sum_{rep != 1} KS_rep(aut_rep(x)) (tracepack.py:268-285)."""
    acc = x.copy()
    live = None
    if skip_zero:
        live = np.flatnonzero(x.reshape(x.shape[0], -1).any(axis=1))
        if live.size == 0:
            return acc
        if live.size < x.shape[0]:
            x = x[live]
    for rep in reps[1:]:
        sw = engine.switch_batch(engine.automorphism_batch(x, rep), rep, counter=counter)
        if live is not None and live.size < acc.shape[0]:
            acc[live] += sw
        else:
            acc += sw
        acc &= UMASK
    return acc


def merge(cur, members, stride, R: Ring):
    """Level merge: sum_a X^(a*stride) * rows[a*rest + r] (tracepack.py:307-316)."""
    rest = cur.shape[0] // members
    grp = cur.reshape(members, rest, 2, R.N)
    out = np.zeros((rest, 2, R.N), U64)
    for a in range(members):
        part = grp[a] if a == 0 else mono_shift(grp[a], a * stride, R)
        out = (out + part) & UMASK
    return out


def fast_pack(cts, scheme: Scheme, engine, counter=None, skip_zero=False):
    """Pack F extracted rows into one ciphertext (tracepack.py:288-326)."""
    R = scheme.ring
    t, alpha, beta, gamma = R.t, R.alpha, scheme.beta_eff, scheme.gamma
    F = scheme.pack_factor
    if cts.shape != (F, 2, R.N):
        raise ValueError(f"fast_pack expects exactly {F} rows of shape (2, {R.N})")
    cur = cts
    if gamma == 0:
        for chain in stage0_chains(R):
            cur = apply_stage(cur, chain, engine, counter, skip_zero)
    for j in range(1, beta + 1):
        cur = merge(cur, (t - 1) if j == 1 else t, R.M // t ** j, R)
        if max(gamma, 1) <= j <= beta - 1:
            cur = apply_stage(cur, stage_reps_above(j, R), engine, counter, skip_zero)
    for j in range(beta, alpha):
        if j >= max(gamma, 1):
            cur = apply_stage(cur, stage_reps_above(j, R), engine, counter, skip_zero)
    if counter is not None:
        counter.add_packed(F)
    return cur[0]


def pad_groups(rows, F, N):
    e = rows.shape[0]
    G = -(-e // F)
    out = np.zeros((G * F, 2, N), U64)
    out[:e] = rows
    return out.reshape(G, F, 2, N)


def pack_rows(rows, scheme: Scheme, engine, counter=None, skip_zero=True):
    """tracepack.py:336-348."""
    groups = pad_groups(rows, scheme.pack_factor, scheme.ring.N)
    return [fast_pack(g, scheme, engine, counter=counter, skip_zero=skip_zero)
            for g in groups]


def slot_positions(scheme: Scheme):
    R = scheme.ring
    return np.arange(scheme.pack_factor) * (R.M // R.t ** scheme.beta_eff)


def read_packed_values(phases, count, scheme: Scheme):
    pos = slot_positions(scheme)
    F = scheme.pack_factor
    return np.array([phases[i // F][pos[i % F]] for i in range(count)], dtype=np.int64)
