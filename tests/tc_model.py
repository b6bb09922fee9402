"""Bit-level numpy model of the tensor-core forward key switch (test-only).

The forward Phi_M-NTT of the digit polynomials is evaluated as two batched
small matrix products over Z_p, each an exact int8 GEMM over byte planes
(csrc/keyswitch_tc.cu):

  coefficient c = j*n1 + m1*SB + m0            (j < t-1, m1 < t^a, m0 < SB = t^b)
  output (o, k1), o = (r-1)*t^a + k0           evaluation point omega^e,
  e = r + t*(k0 + t^a*k1)                      (r in 1..t-1, k0 < t^a, k1 < SB)

  pass A  z[o | m0]  = sum_q W_A[o][q] d[q*SB + m0]   q = j*t^a + m1,
          W_A[o][q]  = omega^(n1 r j + SB m1 (r + t k0))
  twiddle y[o | m0]  = z[o | m0] * omega^((r + t k0) m0)
  pass B  A[o, k1]   = sum_m0 omega^(t^(a+1) k1 m0) y[o | m0]

which is a(omega^e) = sum_c a_c omega^(e c).  On the tensor cores each pass is
D[b] = sum_kk X[kk] * byte_b(C[kk]) with the data planes X folded into K
(C[plane*S + q] = 256^plane W mod p), so the four s32 accumulators combine as
l + 2^16 h (l = D0 + 256 D1, h = D2 + 256 D3) and one Montgomery REDC against
(x, 2^16 x) constants reduces and multiplies in one step.  Digits enter with
an offset (D/2 - 1 for power-of-two D, else D//2) so both planes are unsigned; an extra
K row of ones carries the offset correction.

This model replays exactly that integer arithmetic with range assertions and
is checked against tests/kernel_sim.py (the CUDA-core kernel's model) in
tests/test_tc_model.py.
"""

from __future__ import annotations

import numpy as np

U = np.uint64
M32 = (1 << 32) - 1


def geometry(t: int) -> tuple[int, int]:
    """(a, b): pass A covers (t-1) t^a points, pass B t^b points (a + b = alpha - 1)."""
    return {7: (1, 2), 5: (2, 2), 3: (3, 3)}[t]


def digit_offset(D: int) -> int:
    """Balanced digits lie in [-D/2 + 1, D/2] for power-of-two D (carry chain) and in
    [-D//2, D//2] otherwise (rounded remainders); the offset makes them non-negative."""
    return D // 2 - 1 if D & (D - 1) == 0 else D // 2


class TcTables:
    """Constant operands of one (ring, prime); the same numbers the library builds."""

    def __init__(self, t: int, alpha: int, p: int, omega: int, D: int):
        a, b = geometry(t)
        assert a + b == alpha - 1
        self.t, self.alpha, self.p, self.omega = t, alpha, p, omega
        M = t ** alpha
        n1 = M // t
        ta, SB = t ** a, t ** b
        SA = (t - 1) * ta
        self.M, self.n1, self.ta, self.SA, self.SB = M, n1, ta, SA, SB
        self.N = (t - 1) * n1
        self.off = digit_offset(D)
        pw = [pow(omega, e, p) for e in range(M)]
        o = np.arange(SA)
        r = o // ta + 1
        k0 = o % ta
        q = np.arange(SA)
        j = q // ta
        m1 = q % ta
        eA = (n1 * np.outer(r, j) + SB * np.outer(r + t * k0, m1)) % M
        self.WA = np.array([[pw[e] for e in row] for row in eA], dtype=object)          # [o][q]
        m0 = np.arange(SB)
        self.TW = np.array([[pw[e] for e in row] for row in (np.outer(r + t * k0, m0) % M)], dtype=object)
        k1 = np.arange(SB)
        self.WB = np.array([[pw[e] for e in row] for row in (t ** (a + 1) * np.outer(k1, m0) % M)],
                           dtype=object)                                               # [k1][m0]
        self.e = (r[:, None] + t * (k0[:, None] + ta * k1[None, :])) % M                # [o][k1]
        L = alpha - 1

        def drev(k):
            out = 0
            for _ in range(L):
                out = out * t + k % t
                k //= t
            return out
        kk = k0[:, None] + ta * k1[None, :]
        self.old_idx = (r[:, None] - 1) * n1 + np.vectorize(drev)(kk)                  # [o][k1]
        # folded constant operands: rows kk, value < p (plus the ones row of pass A)
        CA = np.zeros((2 * SA + 1, SA), dtype=object)
        for plane in range(2):
            CA[plane * SA:(plane + 1) * SA] = (self.WA.T * pow(256, plane, p)) % p
        CA[2 * SA] = (-self.off * self.WA.sum(axis=1)) % p
        self.CA = CA
        CB = np.zeros((4 * SB, SB), dtype=object)
        for plane in range(4):
            CB[plane * SB:(plane + 1) * SB] = (self.WB.T * pow(256, plane, p)) % p
        self.CB = CB
        R = (1 << 32) % p
        self.TWm = (self.TW * R) % p                      # [o][m0]
        self.TWm2 = (self.TWm * (1 << 16)) % p
        self.pinv = (-pow(p, -1, 1 << 32)) % (1 << 32)    # -p^-1 mod 2^32 (REDC: x + m p)

    # -- exact integer pieces -------------------------------------------------
    def redc(self, x):
        x = np.asarray(x, dtype=object)
        assert np.all(x < self.p * (1 << 32)) and np.all(x >= 0), "REDC input out of range"
        m = ((x & M32) * self.pinv) & M32
        r = (x + m * self.p) >> 32
        assert np.all(r < 2 * self.p)
        return r

    @staticmethod
    def planes(C, nplanes=4):
        C = np.asarray(C, dtype=object)
        return [(C >> (8 * b)) & 255 for b in range(nplanes)]

    def gemm_planes(self, X, C):
        """X: [seq][K] bytes, C: [K][N] values < 2^32 -> 4 accumulators [seq][N] (exact, < 2^32)."""
        X = np.asarray(X, dtype=np.int64)
        outs = []
        for cb in self.planes(C):
            w = X @ np.asarray(cb, dtype=np.int64)
            assert np.all(w >= 0) and np.all(w < (1 << 31)), "s32 accumulator overflow"
            outs.append(w.astype(object))
        return outs

    def combine(self, w):
        lo = w[0] + 256 * w[1]
        hi = w[2] + 256 * w[3]
        assert np.all(lo < (1 << 32)) and np.all(hi < (1 << 32))
        return lo, hi

    def forward_digit(self, dg):
        """dg: (N,) balanced digits -> (SA, SB) NTT values (lazy, < 2p), o-major."""
        t, SA, SB, ta = self.t, self.SA, self.SB, self.ta
        ev = np.asarray(dg, dtype=np.int64) + self.off
        assert np.all(ev >= 0) and np.all(ev < 65536)
        # coefficient c = j n1 + m1 SB + m0 = q SB + m0 (q = j t^a + m1)
        E = ev.reshape(SA, SB)                  # [q][m0]
        X = np.zeros((SB, 2 * SA + 1), np.int64)  # sequences m0, K = (plane, q) + ones
        X[:, :SA] = (E & 255).T
        X[:, SA:2 * SA] = (E >> 8).T
        X[:, 2 * SA] = 1
        wA = self.gemm_planes(X, self.CA)       # [m0][o]
        lo, hi = self.combine(wA)
        y = self.redc(lo * self.TWm.T + hi * self.TWm2.T)   # [m0][o]  < 2p
        Y = np.asarray(y, dtype=np.int64)
        XB = np.concatenate([(Y.T >> (8 * b)) & 255 for b in range(4)], axis=1)  # [o][(plane, m0)]
        wB = self.gemm_planes(XB, self.CB)      # [o][k1]
        return self.combine(wB)                 # (lo, hi): value = lo + 2^16 hi (times nothing)

    def mac(self, lohi, Km):
        """REDC(lo Km + hi 2^16 Km) with Km = K^ R mod p: (value * K^) mod p, lazy."""
        lo, hi = lohi
        Km = np.asarray(Km, dtype=object)
        Km2 = (Km * (1 << 16)) % self.p
        x = lo * Km + hi * Km2
        assert np.all(x < (1 << 64))
        m = ((x & M32) * self.pinv) & M32
        r = (x + m * self.p) >> 32
        assert np.all(r < (1 << 32))
        return r
