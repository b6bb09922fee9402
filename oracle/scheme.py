"""Oracle: scheme parameters, ring arithmetic mod (2^53, Phi_M), dual basis.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates:
  * parameter rows / gadget / presets      reference pkg/src/sfhr/params.py:14-164
  * fold, automorphism, monomial shift      reference pkg/src/sfhr/ring.py:29-130
  * two-term dual basis (e1, e2, c, M^-1)    reference pkg/src/sfhr/dual.py:71-166
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

QB = 53
Q = 1 << QB
MASK = Q - 1
U64 = np.uint64
UMASK = np.uint64(MASK)


def _is_prime_small(n: int) -> bool:
    if n < 2:
        return False
    f = 2
    while f * f <= n:
        if n % f == 0:
            return False
        f += 1
    return True


def factor_multiset(n: int) -> list[int]:
    """Prime factors with multiplicity, ascending (params.py:28-38)."""
    out, f = [], 2
    while f * f <= n:
        while n % f == 0:
            out.append(f)
            n //= f
        f += 1
    if n > 1:
        out.append(n)
    return out


def smallest_generator(t: int) -> int:
    """Least primitive root of the prime t (params.py:41-47)."""
    fs = set(factor_multiset(t - 1))
    for g in range(2, t):
        if all(pow(g, (t - 1) // f, t) != 1 for f in fs):
            return g
    raise ValueError(f"no primitive root mod {t}")


@dataclass(frozen=True)
class Ring:
    """Z_q[X]/Phi_M, M = t^alpha (params.py:50-92)."""
    t: int
    alpha: int
    p_bits: int

    def __post_init__(self):
        if self.t < 3 or not _is_prime_small(self.t):
            raise ValueError(f"t must be an odd prime >= 3, got {self.t}")
        if self.alpha < 1:
            raise ValueError("alpha must be >= 1")
        if not 8 <= self.p_bits <= 16:
            raise ValueError("p must be a power of two between 2^8 and 2^16")

    @property
    def M(self):
        return self.t ** self.alpha

    @property
    def n1(self):
        return self.t ** (self.alpha - 1)

    @property
    def N(self):
        return self.n1 * (self.t - 1)

    @property
    def p(self):
        return 1 << self.p_bits


@dataclass(frozen=True)
class Gadget:
    """Balanced base-D depth-l gadget (params.py:95-114)."""
    D: int
    l: int

    def __post_init__(self):
        if self.D < 2 or self.l < 1:
            raise ValueError("need D >= 2 and l >= 1")
        if self.D ** self.l > Q:
            raise ValueError("D^l must not exceed q")
        if (self.D & (self.D - 1)) and self.D > 1024:
            raise ValueError("non-power-of-two base must be <= 1024")


@dataclass(frozen=True)
class Scheme:
    """Ring + noise + gadget + (gamma, beta) (params.py:117-142)."""
    ring: Ring
    delta: float
    gadget: Gadget
    gamma: int = 0
    beta: int = 0
    key_dist: str = "binary"

    def __post_init__(self):
        if self.gamma not in (0, 1, 2):
            raise ValueError("extraction level gamma must be 0, 1 or 2")
        b = self.beta or self.ring.alpha - 1
        if not 1 <= b <= self.ring.alpha - 1:
            raise ValueError("packing level beta must satisfy 1 <= beta <= alpha-1")

    @property
    def beta_eff(self):
        return self.beta or self.ring.alpha - 1

    @property
    def pack_factor(self):
        return self.ring.t ** (self.beta_eff - 1) * (self.ring.t - 1)


# (t, alpha, delta, {gamma: (D, l)}) per accumulator width  (params.py:147-151)
PRESET_ROWS = {
    8: (3, 7, 2.0 ** -36, {0: (512, 3), 1: (512, 3), 2: (512, 3)}),
    12: (7, 4, 2.0 ** -51, {0: (4096, 3), 1: (65536, 2), 2: (65536, 2)}),
    16: (5, 5, 2.0 ** -51, {0: (310, 5), 1: (310, 4), 2: (310, 4)}),
}


def preset(b: int, gamma: int = 0, beta: int = 0) -> Scheme:
    """preset_for_bits (params.py:154-164)."""
    if b not in PRESET_ROWS:
        raise ValueError(f"no parameter preset for b={b}")
    if gamma not in (0, 1, 2):
        raise ValueError("extraction level gamma must be 0, 1 or 2")
    t, alpha, delta, gad = PRESET_ROWS[b]
    D, l = gad[gamma]
    return Scheme(Ring(t, alpha, b), delta, Gadget(D, l), gamma, beta)


# ---------------------------------------------------------------------------
# ring arithmetic on (..., N) uint64 numerators


def fold(buf: np.ndarray, R: Ring) -> np.ndarray:
    """Length-M representative -> canonical length-N (ring.py:29-40, 61-67).

    out[k] = buf[k] - buf[N + (k mod n1)] because X^(N+r) = -sum_j X^(r+j n1).
    """
    N, n1 = R.N, R.n1
    k = np.arange(N)
    out = buf[..., :N] - buf[..., N + (k % n1)]
    if out.dtype == U64:
        out &= UMASK
    return out


def reduce_cyclo(raw: np.ndarray, R: Ring) -> np.ndarray:
    """Canonical rep mod Phi_M of a vector of length < 2M (ring.py:43-58)."""
    M, N = R.M, R.N
    raw = np.asarray(raw)
    L = raw.shape[-1]
    if L >= 2 * M:
        raise ValueError("degree too large")
    buf = np.zeros(raw.shape[:-1] + (M,), dtype=raw.dtype)
    h = min(L, M)
    buf[..., :h] = raw[..., :h]
    if L > M:
        buf[..., :L - M] += raw[..., M:]
    if L <= N:
        out = buf[..., :N].copy()
        if out.dtype == U64:
            out &= UMASK
        return out
    return fold(buf, R)


def embed(v: np.ndarray, R: Ring) -> np.ndarray:
    out = np.zeros(v.shape[:-1] + (R.M,), dtype=v.dtype)
    out[..., :R.N] = v
    return out


def scatter_fold(v: np.ndarray, pos: np.ndarray, R: Ring) -> np.ndarray:
    """buf[pos[n]] = v[n] (pos injective into [0,M)), then fold."""
    buf = np.zeros(v.shape[:-1] + (R.M,), dtype=v.dtype)
    buf[..., pos] = v
    return fold(buf, R)


def mono_shift(v: np.ndarray, e: int, R: Ring) -> np.ndarray:
    """v * X^e mod Phi_M (ring.py:77-84)."""
    e %= R.M
    return scatter_fold(v, (np.arange(R.N) + e) % R.M, R)


def automorph(v: np.ndarray, d: int, R: Ring) -> np.ndarray:
    """P(X) -> P(X^d) for gcd(d, M) = 1 (ring.py:87-95)."""
    if math.gcd(d, R.M) != 1:
        raise ValueError(f"automorphism index {d} not coprime with M={R.M}")
    return scatter_fold(v, (np.arange(R.N) * (d % R.M)) % R.M, R)


@lru_cache(maxsize=None)
def automorph_gather(t: int, alpha: int, d: int):
    """Two masked gathers realising automorphism+fold (ring.py:101-121)."""
    R = Ring(t, alpha, 8)
    M, N, n1 = R.M, R.N, R.n1
    where = np.full(M, -1, dtype=np.int64)
    where[(np.arange(N) * (d % M)) % M] = np.arange(N)
    k = np.arange(N)
    s1, s2 = where[k], where[N + k % n1]
    return (np.maximum(s1, 0), (s1 >= 0).astype(U64),
            np.maximum(s2, 0), (s2 >= 0).astype(U64))


def automorph_u64(v: np.ndarray, d: int, R: Ring) -> np.ndarray:
    """Table form for uint64 batches (ring.py:124-130)."""
    g1, m1, g2, m2 = automorph_gather(R.t, R.alpha, d % R.M)
    out = v[..., g1] * m1 - v[..., g2] * m2
    return out & UMASK


# ---------------------------------------------------------------------------
# dual basis (two-term form of M * conj(dual_i))


@dataclass
class Dual:
    e1: np.ndarray
    e2: np.ndarray
    c: np.ndarray            # ratio_len
    inv_m_mod_p: int
    scatter_idx: np.ndarray
    scatter_coef: np.ndarray


def _tr_zeta(k: int, t: int, alpha: int) -> int:
    """Tr(zeta_M^k) (dual.py:18-27)."""
    M, n1 = t ** alpha, t ** (alpha - 1)
    k %= M
    if k == 0:
        return n1 * (t - 1)
    return -n1 if k % n1 == 0 else 0


@lru_cache(maxsize=None)
def dual_for(t: int, alpha: int, p_bits: int) -> Dual:
    """Construct and verify the two-term dual basis (dual.py:108-166)."""
    R = Ring(t, alpha, p_bits)
    M, N, n1 = R.M, R.N, R.n1
    e1 = np.zeros(N, np.int64)
    e2 = np.zeros(N, np.int64)
    cc = np.zeros(N, np.int64)
    for i in range(N):
        a = (-i) % M
        first = i // n1 + 1
        for c in [first] + [c for c in range(1, t) if c != first]:
            b = (a + c * n1) % M
            ok = all(_tr_zeta(j + a, t, alpha) - _tr_zeta(j + b, t, alpha)
                     == (M if j == i else 0) for j in range(i % n1, N, n1))
            if ok:
                e1[i], e2[i], cc[i] = a, b, c
                break
        else:
            raise ValueError(f"dual basis index {i} has no two-term form")
    width = int(cc.max()) * (t - 1)
    sidx = np.zeros((N, width), np.int64)
    scoef = np.zeros((N, width), np.int64)
    for i in range(N):
        acc: dict[int, int] = {}
        for k in range(int(cc[i])):
            g = (-(int(e1[i]) + k * n1)) % M
            if g < N:
                acc[g] = acc.get(g, 0) + 1
            else:
                for j in range(t - 1):
                    pos = g - N + j * n1
                    acc[pos] = acc.get(pos, 0) - 1
        items = [(p, s) for p, s in acc.items() if s != 0]
        for k, (p, s) in enumerate(items):
            sidx[i, k], scoef[i, k] = p, s
    return Dual(e1, e2, cc, pow(M, -1, R.p), sidx, scoef)


def centered_inv_m(R: Ring) -> int:
    """Centered M^-1 mod p used by extraction (tracepack.py:135-136)."""
    u = dual_for(R.t, R.alpha, R.p_bits).inv_m_mod_p
    return u - R.p if u > R.p // 2 else u
