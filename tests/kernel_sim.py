"""Bit-level numpy model of the device key-switch stage kernel (test-only).

Replays, with the library's own constant tables (planning-only context, no
GPU), exactly the arithmetic of ks_stage_kernel / ks_spectra_kernel in
paper_2509_01253_b200/csrc/keyswitch.cu: Montgomery REDC with lazy [0, 2p)
ranges, the radix-t DFTs (Rader/Winograd dft_wino7 / dft_wino5 for t = 7 / 5, symmetric-pair
dft_sym for t = 3; lazy outputs before twiddles), the fused automorphism+decomposition first step, radix-t DIF/DIT
stages, NTT-domain accumulation over reps, and explicit CRT mod 2^53.
Every REDC input is range-checked, so an overflow in the kernel's bound
reasoning fails here on CPU before any GPU time is spent.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2509_01253_b200 import _native as nat

U = np.uint64
M32 = U(0xFFFFFFFF)


class SimPlan:
    def __init__(self, t, alpha, p_bits, D, l, gamma=0, beta=0):
        h = C.c_void_p()
        nat.check(nat.lib.sfhr_ctx_create(t, alpha, p_bits, D, l, gamma, beta, -1, C.byref(h)))
        self.h = h
        rc = nat.RingConst()
        self.M = t ** alpha
        npr = rc_np = None  # noqa
        info = (C.c_int64 * 32)()
        k = nat.lib.sfhr_ctx_info(h, info, 32)
        self.info = list(info[:k])
        np_ = self.info[3]
        stride = (self.M + 4) & ~3  # csrc/sfhr_common.cuh twid_stride
        n1 = self.M // t
        sstride = (2 * (n1 + 1) + 3) & ~3  # shoup_stride
        tw = np.zeros(np_ * (stride + sstride), np.uint32)
        nat.check(nat.lib.sfhr_ctx_debug_tables(h, C.byref(rc), C.sizeof(rc), tw.ctypes.data, tw.size))
        self.rc = rc
        self.tw = tw[:np_ * stride].reshape(np_, stride)[:, :self.M + 1].astype(U)
        self.sh = tw[np_ * stride:].reshape(np_, sstride).astype(U)
        self.t, self.alpha, self.N, self.n1 = t, alpha, rc.N, rc.n1
        self.np, self.l = rc.np, rc.l
        self.nitems = rc.nitems

    def close(self):
        nat.lib.sfhr_ctx_destroy(self.h)


class Prime:
    def __init__(self, sp: SimPlan, i: int):
        pc = sp.rc.pc[i]
        self.p, self.pinv, self.mu = U(pc.p), U(pc.pinv), U(pc.mu)
        self.bc = U(pc.bc)
        assert int(self.bc) == (1 << 33) // int(self.p)
        self.r2, self.rmod = U(pc.r2), U(pc.rmod)
        T = sp.t
        self.z = np.array([[pc.z[k][m] for m in range(T)] for k in range(T)], dtype=U)
        self.zi = np.array([[pc.zi[k][m] for m in range(T)] for k in range(T)], dtype=U)
        self.g = np.array([[pc.g[j][r] for r in range(T - 1)] for j in range(T - 1)], dtype=U)
        H = (T - 1) // 2
        self.hc = np.array([[pc.hc[k][m] for m in range(H)] for k in range(H)], dtype=U)
        self.hs = np.array([[pc.hs[k][m] for m in range(H)] for k in range(H)], dtype=U)
        self.wino = [pc.wino[0], pc.wino[1], pc.wino[2]]
        self.q_mod64 = U(pc.q_mod64)
        self.inv_p = pc.inv_p
        self.wt = sp.tw[i]
        self.t = T
        sh = sp.sh[i]
        self.sh_w, self.sh_q = sh[0::2][:sp.n1 + 1], sh[1::2][:sp.n1 + 1]
        # the table is the plain omega^(t i) and floor(w 2^32 / p) (plan.cpp)
        rinv = pow(1 << 32, -1, int(self.p))
        assert all(int(self.sh_w[k]) == int(self.wt[T * k]) * rinv % int(self.p) for k in (0, 1, sp.n1))
        assert all(int(self.sh_q[k]) == (int(self.sh_w[k]) << 32) // int(self.p) for k in (0, 1, sp.n1))

    def redc(self, x):
        x = np.asarray(x, dtype=U)
        hi = x >> U(32)
        assert np.all(hi < self.p), "REDC input >= p * 2^32"
        m = ((x & M32) * self.pinv) & M32
        r = hi + self.p - ((m * self.p) >> U(32))
        assert np.all((r > 0) & (r < U(2) * self.p))
        return r

    def redc_wide(self, x):
        x = np.asarray(x, dtype=U)
        assert np.all(x < U(1 << 63)), "wide accumulator overflow"
        hi = x >> U(32)
        m = ((x & M32) * self.pinv) & M32
        r = hi + self.p - ((m * self.p) >> U(32))
        q = (r * self.mu) >> U(32)
        r = r - q * self.p
        assert np.all(r < U(2) * self.p)
        return r

    def redc_lazy(self, x, l):
        """REDC of a lazy key-MAC sum (< l p 2^32), then one Barrett step -> [0, 2p)."""
        x = np.asarray(x, dtype=U)
        hi = x >> U(32)
        assert np.all(hi < U(l) * self.p), "lazy MAC sum >= l p 2^32"
        m = ((x & M32) * self.pinv) & M32
        r = hi + self.p - ((m * self.p) >> U(32))
        assert np.all(r < U(1 << 32))
        return self.barrett(r)

    def shoup(self, a, e):
        """shoup_mul (sfhr_common.cuh) by omega^e from the Shoup pair table (e a multiple of t):
        any a < 2^32 -> [0, 2p)."""
        a = np.asarray(a, dtype=U)
        assert np.all(a < U(1 << 32))
        w = self.sh_w[np.asarray(e) // self.t]
        wq = self.sh_q[np.asarray(e) // self.t]
        q = (a * wq) >> U(32)
        r = (a * w - q * self.p) & M32
        assert np.all(r < U(2) * self.p), "Shoup product out of [0, 2p)"
        return r

    def mont(self, a, bm):
        a = np.asarray(a, dtype=U)
        assert np.all(a < U(2) * self.p)
        return self.redc(a * np.asarray(bm, dtype=U))

    def dft(self, xs, Z):
        """xs: list of T arrays; returns T arrays (sum over m of x_m Z[k][m], REDC)."""
        T = len(xs)
        out = []
        for k in range(T):
            s = np.zeros_like(xs[0], dtype=U)
            for m in range(T):
                s = s + xs[m] * Z[k][m]
            out.append(self.redc(s))
        return out

    def barrett(self, v):
        """keyswitch.cu bar(): bred (32-bit multiplies) under SFHR_BRED, else umulhi by mu."""
        v = np.asarray(v, dtype=U)
        assert np.all(v < U(1 << 32))
        if BRED:
            q = (((v >> U(16)) * self.bc) & M32) >> U(17)
            assert np.all(((v >> U(16)) * self.bc) < U(1 << 32))
            r = (v - q * self.p) & M32
        else:
            r = v - ((v * self.mu) >> U(32)) * self.p
        assert np.all(r < U(2) * self.p)
        return r

    def dft_sym(self, xs, inv=False, red=False):
        """keyswitch.cu dft_sym: symmetric-pair radix-t DFT with its lazy ranges."""
        T = len(xs)
        H = (T - 1) // 2
        p2 = U(2) * self.p
        xs = [np.asarray(x, dtype=U) for x in xs]
        for x in xs:
            assert np.all(x < p2), "DFT input >= 2p"
        a = [xs[m] + xs[T - m] for m in range(1, H + 1)]
        b = [xs[m] + p2 - xs[T - m] for m in range(1, H + 1)]
        y0 = xs[0] + sum(a)
        out = [None] * T
        out[0] = self.barrett(y0)
        for k in range(1, H + 1):
            sp = sum(a[m] * self.hc[k - 1][m] for m in range(H))
            sq = sum(b[m] * self.hs[k - 1][m] for m in range(H))
            P, Q = self.redc(sp), self.redc(sq)
            u, v = xs[0] + P + Q, xs[0] + P + p2 - Q
            assert np.all(u < U(1 << 32)) and np.all(v < U(1 << 32))
            if red:
                u, v = self.barrett(u), self.barrett(v)
            out[k], out[T - k] = (v, u) if inv else (u, v)
        return out

    def shoup_c(self, x, cw, cq):
        """shoup_mul by a constant (plain c, floor(c 2^32 / p)): x < 2^32 -> [0, 2p)."""
        x = np.asarray(x, dtype=U)
        assert np.all(x < U(1 << 32))
        q = (x * U(cq)) >> U(32)
        r = (x * U(cw) - q * self.p) & M32
        assert np.all(r < U(2) * self.p)
        return r

    def wino_m0(self, S, w, acc):
        """keyswitch.cu wino_m0: S mu (Shoup under SFHR_WINO_SHOUP, else Montgomery)."""
        if WINO_SHOUP:
            return self.shoup_c(np.asarray(S).astype(U), w.mu_w, w.mu_q)
        return self.redc(np.asarray(S).astype(U) * U(w.mu))

    def wino_r2(self, Tm, w, acc):
        """keyswitch.cu wino_r2: Tm rho with Tm offset by toff (a multiple of p) for Shoup."""
        if WINO_SHOUP:
            x = np.asarray(Tm, dtype=np.int64) + int(w.toff)
            assert np.all(x >= 0), "negative Shoup operand"
            assert int(w.toff) % int(self.p) == 0
            return self.shoup_c(x.astype(U), w.rho_w, w.rho_q)
        return self.redc(acc(w.kT, (Tm, w.rho)))

    def wino_g(self, A0, A1, w, acc):
        """keyswitch.cu wino_g: [[a00, a01], [a10, a00]] (A0, A1), Karatsuba under SFHR_WINO_KARA."""
        if WINO_KARA:
            D = A0 - A1
            assert np.all(np.abs(D) < (1 << 31)), "Karatsuba operand overflow"
            return (self.redc(acc(w.kG, (D, w.a00), (A1, w.ka01))),
                    self.redc(acc(w.kG, (-D, w.a00), (A0, w.ka10))))
        return self.redc(acc(w.kG, (A0, w.a00), (A1, w.a01))), self.redc(acc(w.kG, (A0, w.a10), (A1, w.a00)))

    def wino_h(self, C0, C1, w, acc):
        """keyswitch.cu wino_h: [[b00, b01], [b10, b00]] (C0, C1), Karatsuba under SFHR_WINO_KARA."""
        if WINO_KARA:
            S = C0 + C1
            assert np.all(np.abs(S) < (1 << 31)), "Karatsuba operand overflow"
            return (self.redc(acc(w.kG, (S, w.b00), (C1, w.kb01))),
                    self.redc(acc(w.kG, (S, w.b00), (C0, w.kb10))))
        return self.redc(acc(w.kG, (C0, w.b00), (C1, w.b01))), self.redc(acc(w.kG, (C0, w.b10), (C1, w.b00)))

    def dft_wino7(self, xs, inv=False, red=False):
        """keyswitch.cu dft_wino7: Rader/Winograd radix-7 DFT, signed operands, its offsets."""
        w = self.wino[1 if inv else 0]
        p = int(self.p)
        x = [np.asarray(v, dtype=U) for v in xs]
        for v in x:
            assert np.all(v < U(2 * p)), "DFT input >= 2p"
        I = np.int64
        v0, v1, v2, v3, v4, v5 = (x[i].astype(I) for i in (1, 5, 4, 6, 2, 3))
        p03, p14, p25 = v0 + v3, v1 + v4, v2 + v5
        d03, d14, d25 = v0 - v3, v1 - v4, v2 - v5
        S = p03 + p14 + p25
        Tm = d03 - d14 + d25
        A0, A1 = p03 - p25, p14 - p25
        C0, C1 = d03 - d25, d14 + d25
        for a in (d03, d14, d25, Tm, A0, A1, C0, C1):
            assert np.all(np.abs(a) < (1 << 31)), "signed 32-bit operand overflow"

        def acc(off, *terms):
            r = np.full(S.shape, off, dtype=I)
            for a, c in terms:
                r = r + a * I(c)
            assert np.all(r >= 0), "negative REDC input"
            return r.astype(U)
        M0 = self.wino_m0(S, w, acc)
        R2 = self.wino_r2(Tm, w, acc)
        g0, g1 = self.wino_g(A0, A1, w, acc)
        h0, h1 = self.wino_h(C0, C1, w, acc)
        X0 = x[0].astype(I) + M0.astype(I)
        R2, g0, g1, h0, h1 = (a.astype(I) for a in (R2, g0, g1, h0, h1))
        gs, hd = g0 + g1, h1 - h0
        z = [X0 + R2 + g0 + h0, X0 - R2 + w.k1p + g1 + h1, X0 + R2 + w.k3p - gs + hd,
             X0 - R2 + w.k2p + g0 - h0, X0 + R2 + w.k4p + g1 - h1, X0 - R2 + w.k5p - gs - hd]
        for a in z:
            assert np.all(a >= 0) and np.all(a < (1 << 32)), "output sum out of [0, 2^32)"
        out = [None] * 7
        out[0] = self.barrett((x[0].astype(I) + S).astype(U))
        for i, k in enumerate((1, 3, 2, 6, 4, 5)):
            out[k] = self.barrett(z[i].astype(U)) if red else z[i].astype(U)
        return out

    def dft_wino5(self, xs, inv=False, red=False):
        """keyswitch.cu dft_wino5: Rader radix-5 DFT, signed operands, its offsets."""
        w = self.wino[1 if inv else 0]
        p = int(self.p)
        x = [np.asarray(v, dtype=U) for v in xs]
        for v in x:
            assert np.all(v < U(2 * p)), "DFT input >= 2p"
        I = np.int64
        v0, v1, v2, v3 = (x[i].astype(I) for i in (1, 3, 4, 2))
        S = v0 + v1 + v2 + v3
        Tm = v0 - v1 + v2 - v3
        A0, A1 = v0 - v2, v1 - v3

        def acc(off, *terms):
            r = np.full(S.shape, off, dtype=I)
            for a, c in terms:
                r = r + a * I(c)
            assert np.all(r >= 0), "negative REDC input"
            return r.astype(U)
        M0 = self.wino_m0(S, w, acc).astype(I)
        R2 = self.wino_r2(Tm, w, acc).astype(I)
        g0, g1 = (v.astype(I) for v in self.wino_g(A0, A1, w, acc))
        X0 = x[0].astype(I) + M0
        z = [X0 + R2 + g0, X0 - R2 + w.k1p + g1, X0 + R2 + w.k2p - g0, X0 - R2 + w.k3p - g1]
        for a in z:
            assert np.all(a >= 0) and np.all(a < (1 << 32)), "output sum out of [0, 2^32)"
        out = [None] * 5
        out[0] = self.barrett((x[0].astype(I) + S).astype(U))
        for i, k in enumerate((1, 2, 4, 3)):
            out[k] = self.barrett(z[i].astype(U)) if red else z[i].astype(U)
        return out

    def inv_first7(self, Cs):
        """keyswitch.cu inv_first7: the t = 7 inverse first step in Winograd form -> [0, p)."""
        w = self.wino[2]
        p = int(self.p)
        I = np.int64
        for c in Cs:
            assert np.all(np.asarray(c) < U(2 * p))
        c = [np.asarray(x, dtype=U).astype(I) for x in Cs]
        v0, v1, v2, v3, v4, v5 = c[0], c[4], c[3], c[5], c[1], c[2]
        p03, p14, p25 = v0 + v3, v1 + v4, v2 + v5
        d03, d14, d25 = v0 - v3, v1 - v4, v2 - v5
        S = p03 + p14 + p25
        Tm = d03 - d14 + d25
        A0, A1, C0, C1 = p03 - p25, p14 - p25, d03 - d25, d14 + d25

        def acc(off, *terms):
            r = np.full(S.shape, off, dtype=I)
            for a, k in terms:
                r = r + a * I(k)
            assert np.all(r >= 0)
            return r.astype(U)
        S7 = self.wino_m0(S, w, acc).astype(I)
        R2 = self.wino_r2(Tm, w, acc).astype(I)
        g0, g1 = (v.astype(I) for v in self.wino_g(A0, A1, w, acc))
        h0, h1 = (v.astype(I) for v in self.wino_h(C0, C1, w, acc))
        z = [S7 + R2 + h0 + w.k1p - g0, 2 * (R2 + h0), 2 * R2 + h1 + w.k2p - 2 * g0 - g1,
             g1 + h1 + h0 + w.k3p - g0, 2 * R2 + g1 + h0 + w.k4p - h1 - g0, 2 * h0 + w.k5p - 2 * g0 - g1 - h1]
        out = []
        for a in z:
            assert np.all(a >= 0) and np.all(a < (1 << 32)), "inverse first step sum out of range"
            r = self.barrett(a.astype(U))
            out.append(np.where(r >= self.p, r - self.p, r))
        return np.stack(out)

    def dft_k(self, xs, inv=False, red=False):
        """The radix-t DFT the stage kernel uses for this ring (dft_fwd_tw / _red, dft_inv_red)."""
        if len(xs) == 7:
            return self.dft_wino7(xs, inv, red)
        if len(xs) == 5:
            return self.dft_wino5(xs, inv, red)
        return self.dft_sym(xs, inv, red)

    def mont6(self, a, bm):
        """mont_mul with a lazy operand (twiddle after a DFT: < 6p symmetric, < 2^32 Winograd)."""
        a = np.asarray(a, dtype=U)
        assert np.all(a < U(1 << 32))
        return self.redc(a * np.asarray(bm, dtype=U))


LAZY_INV = True   # keyswitch.cu SFHR_LAZY_INV
LAZY_MAC = True   # keyswitch.cu SFHR_LAZY_MAC (applies from l >= 3)
SHOUP_MID = True  # keyswitch.cu SFHR_SHOUP_MID (mid-stage twiddles as Shoup products)
WINO_SHOUP = True  # keyswitch.cu SFHR_WINO_SHOUP (Rader M0 / R2 terms as Shoup products)
BRED = True        # keyswitch.cu SFHR_BRED (Barrett step with 32-bit multiplies)
WINO_KARA = False  # keyswitch.cu SFHR_WINO_KARA (Karatsuba 2x2 blocks)


def forward(sp: SimPlan, pr: Prime, vals, red=True):
    """vals: (N,) residues < 2p (coefficient domain) -> (nitems, T) last-stage outputs
    (in [0, 2p) when red, else the lazy last stage: < 2^32)."""
    T, n1, M = sp.t, sp.n1, sp.M
    A = np.asarray(vals, dtype=U).reshape(T - 1, n1)
    m = np.arange(n1)
    buf = np.zeros((T - 1, n1), U)
    ys = pr.dft_k([A[j] for j in range(T - 1)] + [np.zeros(n1, U)])
    for q in range(1, T):
        buf[q - 1] = pr.mont6(ys[q], pr.wt[q * m])
    buf = buf.reshape(-1)
    nsub = n1 // T
    L = nsub
    for s_ in range(sp.alpha - 2):
        blocks = T ** s_
        v = buf.reshape(T - 1, blocks, T, L)
        step = M // (T * L)
        j = np.arange(L)
        xs = [v[:, :, mm, :] for mm in range(T)]
        ys = pr.dft_k(xs)
        nv = np.empty_like(v)
        nv[:, :, 0, :] = ys[0]
        for k in range(1, T):
            if SHOUP_MID:
                nv[:, :, k, :] = pr.shoup(ys[k], (step * j * k)[None, None, :])
            else:
                nv[:, :, k, :] = pr.mont6(ys[k], pr.wt[step * j * k][None, None, :])
        buf = nv.reshape(-1)
        L //= T
    x = buf.reshape(sp.nitems, T)
    ys = pr.dft_k([x[:, mm] for mm in range(T)], red=red)
    return np.stack(ys, axis=1)  # (nitems, T)


def inverse(sp: SimPlan, pr: Prime, y):
    """y: (nitems, T) in [0,2p) -> (N,) CRT-weighted residues y_i in [0, p)."""
    T, n1, M = sp.t, sp.n1, sp.M
    lazy = LAZY_INV
    xs = pr.dft_k([y[:, k] for k in range(T)], inv=True, red=not lazy)
    buf = np.stack(xs, axis=1).reshape(-1)
    L = T
    mul = pr.mont6 if lazy else pr.mont   # twiddle multiply of a lazy (< 2^32) operand
    for s_ in range(sp.alpha - 3, -1, -1):
        blocks = T ** s_
        v = buf.reshape(T - 1, blocks, T, L)
        step = M // (T * L)
        j = np.arange(L)
        z0 = pr.barrett(v[:, :, 0, :]) if lazy else v[:, :, 0, :]
        if SHOUP_MID:
            zs = [z0] + [pr.shoup(v[:, :, k, :], (M - step * j * k)[None, None, :]) for k in range(1, T)]
        else:
            zs = [z0] + [mul(v[:, :, k, :], pr.wt[M - step * j * k][None, None, :]) for k in range(1, T)]
        xs = pr.dft_k(zs, inv=True, red=not lazy)
        buf = np.stack(xs, axis=2).reshape(-1)
        L *= T
    v = buf.reshape(T - 1, n1)
    m = np.arange(n1)
    Cs = [mul(v[r - 1], pr.wt[M - r * m]) for r in range(1, T)]
    if T == 7:
        return pr.inv_first7(Cs).reshape(-1)
    out = np.zeros((T - 1, n1), U)
    for j in range(T - 1):
        s = np.zeros(n1, U)
        for r in range(T - 1):
            s = s + Cs[r] * pr.g[j][r]
        a = pr.redc(s)
        out[j] = np.where(a >= pr.p, a - pr.p, a)
    return out.reshape(-1)


def key_spectrum(sp: SimPlan, pr: Prime, key_poly):
    v = np.asarray(key_poly, dtype=U) & U((1 << 53) - 1)
    c = v.astype(np.int64)
    c = np.where(v >= U(1 << 52), c - (1 << 53), c)
    vals = (c % int(pr.p)).astype(U)
    y = forward(sp, pr, vals)
    z = pr.mont(y, pr.r2)
    return np.where(z >= pr.p, z - pr.p, z)  # (nitems, T)


def stage_row(sp: SimPlan, x, reps_dinv_keys, identity, decompose, automorph_u64):
    """Model of stage_body for one row.  reps_dinv_keys: list of (d, keys[l][2] polys)."""
    N = sp.N
    Q = (1 << 53) - 1
    ys = {}
    for i in range(sp.np):
        pr = Prime(sp, i)
        accA = np.zeros((sp.nitems, sp.t), U)
        accB = np.zeros((sp.nitems, sp.t), U)
        for d, keys in reps_dinv_keys:
            y = automorph_u64(x[0], d) if identity else x[0]
            digs = decompose(y)
            ta = np.zeros((sp.nitems, sp.t), U)
            tb = np.zeros((sp.nitems, sp.t), U)
            lazy = LAZY_MAC and sp.l >= 3
            for li in range(sp.l):
                dm = np.where(digs[li] < 0, digs[li] + int(pr.p), digs[li]).astype(U)
                out = forward(sp, pr, dm, red=not lazy)
                pa, pb = ta, tb
                ta = ta + out * key_spectrum(sp, pr, keys[li][0])
                tb = tb + out * key_spectrum(sp, pr, keys[li][1])
                assert np.all(ta >= pa) and np.all(tb >= pb), "MAC accumulator wrapped"
            if lazy:   # REDC of a sum < l p 2^32 lands in (0, (l + 1) p); one Barrett step
                ra, rb = pr.redc_lazy(ta, sp.l), pr.redc_lazy(tb, sp.l)
            else:      # one REDC per rep into a u32 accumulator
                ra, rb = pr.redc(ta), pr.redc(tb)
            accA = accA + ra
            accB = accB + rb
            assert np.all(accA < U(1 << 32)) and np.all(accB < U(1 << 32))
        za, zb = pr.barrett(accA), pr.barrett(accB)
        assert np.all(za < U(2) * pr.p) and np.all(zb < U(2) * pr.p)
        ya = inverse(sp, pr, za)
        yb = inverse(sp, pr, zb)
        ys[i] = (ya, yb)
    A = np.zeros(N, U)
    B = np.zeros(N, U)
    fa = np.zeros(N)
    fb = np.zeros(N)
    for i in range(sp.np):
        pc = sp.rc.pc[i]
        A = A + ys[i][0] * U(pc.q_mod64)
        B = B + ys[i][1] * U(pc.q_mod64)
        fa = fa + ys[i][0].astype(np.float64) * pc.inv_p
        fb = fb + ys[i][1].astype(np.float64) * pc.inv_p
    Pm = U(sp.rc.P_mod64)
    A = A - np.rint(fa).astype(np.int64).astype(U) * Pm
    B = B - np.rint(fb).astype(np.int64).astype(U) * Pm
    bsum = x[1].copy() if identity else np.zeros(N, U)
    for d, _ in reps_dinv_keys:
        bsum = bsum + (automorph_u64(x[1], d) if identity else x[1])
    out = np.empty((2, N), U)
    out[0] = ((x[0] if identity else U(0)) - A) & U(Q)
    out[1] = (bsum - B) & U(Q)
    return out
