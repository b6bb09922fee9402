"""Oracle: gadget decomposition, key switching, and the client-side crypto.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates:
  * gadget_decompose (both digit algorithms)   reference crypto.py:288-323
  * KeySwitchKeySet / keygen_ksk                reference crypto.py:72-81, 340-357
  * KeySwitchEngine exact + fft backends        reference crypto.py:360-474
  * keygen / encrypt / decrypt (client half)    reference crypto.py:84-235

The client half reproduces the reference's numpy PCG64 draw order exactly so
that keys and uploads generated here are bit-identical to the reference's
for the same seeds (pinned by tests/golden).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .scheme import (Q, QB, U64, UMASK, Dual, Gadget, Ring, automorph,
                     automorph_u64, embed, fold, reduce_cyclo)

# ---------------------------------------------------------------------------
# containers (duck-type compatible with the reference's dataclasses)


@dataclass
class Ct:
    a: np.ndarray
    b: np.ndarray
    noise_hint: float = 0.0


@dataclass
class KskSet:
    keys: dict           # d -> list of l Ct
    gadget: Gadget
    delta: float
    params: Ring

    def indices(self):
        return sorted(self.keys)


@dataclass
class SecretKey:
    s: np.ndarray
    params: Ring
    _mat: object = field(default=None, repr=False)


# ---------------------------------------------------------------------------
# gadget


def decompose(v: np.ndarray, g: Gadget) -> np.ndarray:
    """Balanced base-D digits, shape (l, ...) int64 (crypto.py:288-323)."""
    v = np.asarray(v, dtype=U64)
    D, l = g.D, g.l
    if D & (D - 1) == 0:
        w = D.bit_length() - 1
        sh = QB - w * l
        u = ((v + U64(1 << (sh - 1))) >> U64(sh)).astype(np.int64)
        raw = np.empty((l,) + v.shape, np.int64)
        for i in reversed(range(l)):
            raw[i] = u & (D - 1)
            u >>= w
        out = np.empty_like(raw)
        carry = np.zeros(v.shape, np.int64)
        for i in reversed(range(l)):
            x = raw[i] + carry
            big = x > D // 2
            out[i] = np.where(big, x - D, x)
            carry = big.astype(np.int64)
        return out
    half = 1 << (QB - 1)
    r = v.astype(np.int64)
    r = np.where(v > U64(half), r - Q, r)
    out = np.empty((l,) + v.shape, np.int64)
    for i in range(l):
        prod = r * D
        d = (prod + half) >> QB
        out[i] = d
        r = prod - d * Q
    return out


# ---------------------------------------------------------------------------
# key switching


class KsEngine:
    """Automorphism + gadget key switch (crypto.py:360-474).

    mode='exact' is the formal oracle (uint64 schoolbook); mode='fft'
    restates the reference's default float backend (27-bit key limbs,
    length-M real FFTs) and is used as the timed CPU baseline.
    """

    LIMB = 27

    def __init__(self, ksk: KskSet, mode: str = "exact", max_chunk: int = 128):
        if mode not in ("fft", "exact"):
            raise ValueError(f"unknown key-switch mode {mode!r}")
        self.ksk, self.params, self.mode, self.max_chunk = ksk, ksk.params, mode, max_chunk
        self._spec: dict = {}

    def automorphism_batch(self, cts, d):
        return automorph_u64(cts, d, self.params)

    def switch_batch(self, cts, d, counter=None, skip_zero=False):
        B = cts.shape[0]
        if skip_zero:
            live = np.flatnonzero(cts.reshape(B, -1).any(axis=1))
            out = np.zeros_like(cts)
            if live.size:
                out[live] = self.switch_batch(cts[live], d, counter=counter)
            return out
        if counter is not None:
            counter.add_switches(B)
        out = np.empty_like(cts)
        for s in range(0, B, self.max_chunk):
            out[s:s + self.max_chunk] = self._chunk(cts[s:s + self.max_chunk], d)
        return out

    def _keys(self, d):
        if d not in self.ksk.keys:
            raise KeyError(f"key-switch key set has no index {d}")
        return self.ksk.keys[d]

    def _chunk(self, cts, d):
        keys = self._keys(d)
        digs = decompose(cts[:, 0, :], self.ksk.gadget)
        if self.mode == "exact":
            acc = self._exact(digs, keys)
        else:
            acc = self._fft(digs, d)
        out = np.empty_like(cts)
        out[:, 0] = (U64(0) - acc[:, 0]) & UMASK
        out[:, 1] = (cts[:, 1] - acc[:, 1]) & UMASK
        return out

    def _exact(self, digs, keys):
        l, B, N = digs.shape
        R = self.params
        acc = np.zeros((B, 2, N), U64)
        for r in range(B):
            for i, ct in enumerate(keys):
                dg = digs[i, r].astype(U64)
                for c, comp in enumerate((ct.a, ct.b)):
                    acc[r, c] += reduce_cyclo(np.convolve(dg, comp), R)
        return acc & UMASK

    def _fft(self, digs, d):
        R = self.params
        M = R.M
        if d not in self._spec:
            keys = self._keys(d)
            l = len(keys)
            hi = np.empty((l, 2, M // 2 + 1), np.complex128)
            lo = np.empty_like(hi)
            for i, ct in enumerate(keys):
                for c, comp in enumerate((ct.a, ct.b)):
                    full = embed(comp, R)
                    hi[i, c] = np.fft.rfft((full >> U64(self.LIMB)).astype(np.float64))
                    lo[i, c] = np.fft.rfft((full & U64((1 << self.LIMB) - 1)).astype(np.float64))
            self._spec[d] = (hi, lo)
        hi, lo = self._spec[d]
        l, B, N = digs.shape
        padded = np.zeros((l, B, M))
        padded[:, :, :N] = digs
        sp = np.fft.rfft(padded, axis=2)
        ahi = sum(sp[i][:, None, :] * hi[i][None] for i in range(l))
        alo = sum(sp[i][:, None, :] * lo[i][None] for i in range(l))
        vhi = np.rint(np.fft.irfft(ahi, n=M, axis=2)).astype(np.int64).astype(U64)
        vlo = np.rint(np.fft.irfft(alo, n=M, axis=2)).astype(np.int64).astype(U64)
        return fold((vhi << U64(self.LIMB)) + vlo, R)

    def homomorphic_automorphism(self, ct: Ct, d: int, counter=None) -> Ct:
        if d % self.params.M == 1:
            return ct
        batch = np.stack([ct.a, ct.b])[None]
        sw = self.switch_batch(self.automorphism_batch(batch, d), d, counter=counter)
        return Ct(sw[0, 0], sw[0, 1], ct.noise_hint)


# ---------------------------------------------------------------------------
# client half: keys, encryption, decryption


def keygen(R: Ring, key_dist: str = "binary", seed=0) -> SecretKey:
    """crypto.py:84-92."""
    rng = np.random.default_rng(seed)
    if key_dist == "binary":
        s = rng.integers(0, 2, R.N, dtype=np.int8)
    elif key_dist == "ternary":
        s = rng.integers(-1, 2, R.N, dtype=np.int8)
    else:
        raise ValueError(f"unknown key distribution {key_dist!r}")
    return SecretKey(s, R)


def _key_matrix(sk: SecretKey) -> np.ndarray:
    """Negacyclic-like Toeplitz of s mod Phi_M as float64 (crypto.py:116-129)."""
    if sk._mat is None:
        R = sk.params
        M, N = R.M, R.N
        big = np.zeros((M, N), np.int64)
        rows = (np.arange(N)[:, None] + np.arange(N)[None, :]) % M
        np.add.at(big, (rows, np.broadcast_to(np.arange(N), (N, N))),
                  sk.s.astype(np.int64)[:, None])
        k = np.arange(N)
        mat = big[:N] - big[N + k % R.n1]
        sk._mat = mat.astype(np.float64)
    return sk._mat


def key_times(sk: SecretKey, v: np.ndarray) -> np.ndarray:
    """s * v mod Phi_M exactly, via three 18-bit float64 limbs (crypto.py:131-150)."""
    mat = _key_matrix(sk)
    flat = v.reshape(-1, v.shape[-1]).T
    acc = np.zeros_like(flat)
    for k in range(3):
        limb = ((flat >> U64(18 * k)) & U64((1 << 18) - 1)).astype(np.float64)
        acc += np.rint(mat @ limb).astype(np.int64).astype(U64) << U64(18 * k)
    return (acc.T.reshape(v.shape)) & UMASK


def lift(msg, R: Ring) -> np.ndarray:
    """crypto.py:153-156."""
    return (np.asarray(msg, dtype=np.int64).astype(U64) * U64(Q >> R.p_bits)) & UMASK


def project(phase, R: Ring) -> np.ndarray:
    """crypto.py:159-163."""
    sh = QB - R.p_bits
    return (((phase + U64(1 << (sh - 1))) >> U64(sh)) & U64(R.p - 1)).astype(np.int64)


def encrypt_batch(payloads, sk: SecretKey, delta, rng, dual: Dual) -> np.ndarray:
    """Dual-weighted RLWE encryption of (B, N) payloads (crypto.py:166-199)."""
    payloads = np.atleast_2d(np.asarray(payloads, dtype=U64))
    B, N = payloads.shape
    a_star = rng.integers(0, Q, (B, N), dtype=U64)
    e_star = rng.normal(0.0, delta, (B, N)) if delta > 0 else np.zeros((B, N))
    a_t = np.zeros((N, B), U64)
    e_t = np.zeros((N, B))
    for k in range(dual.scatter_idx.shape[1]):
        idx = dual.scatter_idx[:, k]
        coef = dual.scatter_coef[:, k]
        np.add.at(a_t, idx, (a_star * coef.astype(U64)[None, :]).T)
        np.add.at(e_t, idx, (e_star * coef[None, :]).T)
    a = a_t.T & UMASK
    e_num = np.rint(e_t.T * float(Q)).astype(np.int64).astype(U64)
    out = np.empty((B, 2, N), U64)
    out[:, 0] = a
    out[:, 1] = (key_times(sk, a) + payloads + e_num) & UMASK
    return out


def phase_batch(cts, sk: SecretKey) -> np.ndarray:
    """b - s*a of a (B, 2, N) batch (crypto.py:228-230)."""
    return (cts[:, 1] - key_times(sk, cts[:, 0])) & UMASK


def make_ksk(sk: SecretKey, d_list, g: Gadget, delta, rng, dual: Dual) -> KskSet:
    """RLWE_s(s(X^d) * round(q/D^i)), i=1..l (crypto.py:340-357)."""
    R = sk.params
    keys = {}
    s_int = sk.s.astype(np.int64)
    for d in d_list:
        d = int(d) % R.M
        if np.gcd(d, R.M) != 1:
            raise ValueError(f"key-switch index {d} not coprime with M")
        s_d = automorph(s_int, d, R)
        row = []
        for i in range(1, g.l + 1):
            scale = (2 * Q + g.D ** i) // (2 * g.D ** i)
            payload = (s_d * scale).astype(U64) & UMASK
            ct = encrypt_batch(payload, sk, delta, rng, dual)
            row.append(Ct(ct[0, 0], ct[0, 1], delta))
        keys[d] = row
    return KskSet(keys, g, delta, R)
