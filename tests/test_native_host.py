"""CPU tests of the native library's host side (no GPU): symbols, planning,
dual basis, permutations, and a bit-level simulation of the key-switch
kernel arithmetic against the oracle."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, u53
from oracle import keyswitch as oks
from oracle import pack as opk
from oracle import protocol as opr
from oracle import scheme as osc

nat = pytest.importorskip("paper_2509_01253_b200._native")


def test_library_exports_every_header_symbol():
    hdr = (ROOT / "include" / "sfhr_b200.h").read_text()
    names = set(re.findall(r"\b(sfhr_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 15
    for n in sorted(names):
        assert hasattr(nat.lib, n), n


@pytest.mark.parametrize("b,gamma", [(8, 0), (8, 2), (12, 0), (12, 1), (16, 0), (16, 1)])
def test_plan_matches_oracle_dual_and_bounds(b, gamma):
    sch = osc.preset(b, gamma)
    R = sch.ring
    h = C.c_void_p()
    nat.check(nat.lib.sfhr_ctx_create(R.t, R.alpha, R.p_bits, sch.gadget.D, sch.gadget.l, gamma, 0, -1,
                                      C.byref(h)))
    try:
        info = (C.c_int64 * 32)()
        k = nat.lib.sfhr_ctx_info(h, info, 32)
        M, N, n1, npr, F = info[0], info[1], info[2], info[3], info[4]
        assert (M, N, n1, F) == (R.M, R.N, R.n1, sch.pack_factor)
        primes = info[9:9 + npr]
        for p in primes:
            assert (p - 1) % M == 0 and p < (1 << 31) // max(R.t, sch.gadget.l)
        bound, crt = info[9 + npr] / 1000, info[10 + npr] / 1000
        assert crt >= bound + 1.5
        e1 = np.zeros(N, np.int32)
        e2 = np.zeros(N, np.int32)
        c = np.zeros(N, np.int32)
        nat.check(nat.lib.sfhr_ctx_dual(h, e1.ctypes.data, e2.ctypes.data, c.ctypes.data))
        d = osc.dual_for(R.t, R.alpha, R.p_bits)
        assert np.array_equal(e1, d.e1) and np.array_equal(e2, d.e2) and np.array_equal(c, d.c)
        assert info[7] == d.inv_m_mod_p
        assert info[8] == osc.centered_inv_m(R)
        # compute entry points refuse a planning-only context
        with pytest.raises(ValueError):
            nat.check(nat.lib.sfhr_automorphism_batch(h, 2, None, None, 0, None))
    finally:
        nat.lib.sfhr_ctx_destroy(h)


def test_ctx_rejects_bad_parameters():
    h = C.c_void_p()
    with pytest.raises(ValueError):
        nat.check(nat.lib.sfhr_ctx_create(4, 3, 8, 512, 3, 0, 0, -1, C.byref(h)))
    with pytest.raises(ValueError):
        nat.check(nat.lib.sfhr_ctx_create(3, 3, 8, 1025 * 2 + 1, 3, 0, 0, -1, C.byref(h)))
    with pytest.raises(ValueError):
        nat.check(nat.lib.sfhr_ctx_create(3, 3, 8, 512, 3, 3, 0, -1, C.byref(h)))
    with pytest.raises(ValueError):
        nat.check(nat.lib.sfhr_ctx_create(3, 3, 8, 512, 3, 0, 3, -1, C.byref(h)))


def test_permutation_matches_oracle_and_golden(golden):
    for c in golden["perms"]:
        pm = nat.derive_permutation(bytes(range(32)), bytes(range(16, 32)), c["round"], c["size"])
        assert pm[:16].tolist() == c["head"]
        ref = opr.derive_permutation(bytes(range(32)), bytes(range(16, 32)), c["round"], c["size"])
        assert np.array_equal(pm, ref)
    rng = np.random.default_rng(5)
    for _ in range(5):
        seed = rng.integers(0, 256, 32, dtype=np.uint8).tobytes()
        sid = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        n = int(rng.integers(1, 3000))
        r = int(rng.integers(0, 40))
        assert np.array_equal(nat.derive_permutation(seed, sid, r, n),
                              opr.derive_permutation(seed, sid, r, n))
    with pytest.raises(ValueError):
        nat.derive_permutation(bytes(32), bytes(16), 1, 0)


@pytest.mark.parametrize("t,alpha,b,gamma,D,l", [
    (3, 3, 8, 0, 512, 3),      # reference tests' M = 27 ring
    (3, 2, 8, 0, 512, 3),      # M = 9
    (5, 2, 8, 0, 310, 4),      # M = 25, odd gadget
    (7, 4, 12, 1, 65536, 2),   # b = 12 row, widest CRT bound
    (7, 4, 12, 0, 4096, 3),
    (5, 5, 16, 0, 310, 5),
    (3, 7, 8, 0, 512, 3),
])
def test_stage_kernel_arithmetic_simulation(t, alpha, b, gamma, D, l):
    """Replay the kernel's Montgomery/CRT arithmetic exactly; compare with the oracle."""
    import kernel_sim as ks
    sp = ks.SimPlan(t, alpha, b, D, l, gamma)
    try:
        R = osc.Ring(t, alpha, b)
        g = osc.Gadget(D, l)
        rng = np.random.default_rng(t * 100 + alpha)
        reps = [1] + [(1 + i * t ** (alpha - 1)) % R.M for i in range(1, t)]
        keys = {d: [oks.Ct(u53(1000 + d * 10 + i, R.N), u53(2000 + d * 10 + i, R.N)) for i in range(l)]
                for d in reps[1:]}
        ksk = oks.KskSet(keys, g, 0.0, R)
        eng = oks.KsEngine(ksk, "exact")
        x = u53(int(rng.integers(1 << 30)), (1, 2, R.N))
        # adversarial row: values that maximise digit magnitudes
        x2 = np.full((1, 2, R.N), (1 << 53) - 1, np.uint64)
        for row in (x, x2):
            want = opk.apply_stage(row, reps, eng, None, False)[0]
            got = ks.stage_row(sp, row[0], [(d, [(kk.a, kk.b) for kk in keys[d]]) for d in reps[1:]], True,
                               lambda y: oks.decompose(y, g), lambda v, d: osc.automorph_u64(v, d, R))
            assert np.array_equal(got, want)
        # plain switch mode (one rep, no automorphism, no identity term)
        d = reps[1]
        want = eng.switch_batch(x, d)[0]
        got = ks.stage_row(sp, x[0], [(d, [(kk.a, kk.b) for kk in keys[d]])], False,
                           lambda y: oks.decompose(y, g), None)
        assert np.array_equal(got, want)
    finally:
        sp.close()


@pytest.mark.parametrize("t,alpha,b,gamma,D,l", [(7, 4, 12, 0, 4096, 3), (7, 4, 12, 1, 65536, 2),
                                                  (5, 5, 16, 0, 310, 5), (5, 5, 16, 1, 310, 4)])
def test_rader_dft_exact_with_ranges(t, alpha, b, gamma, D, l):
    """dft_wino7 / dft_wino5 (keyswitch.cu) with the library's constants: every output congruent
    to the direct DFT, every REDC input / output sum inside the bounds the planner proved, for
    random and extreme inputs < 2p, forward and inverse, lazy and reduced."""
    import kernel_sim as ks
    sp = ks.SimPlan(t, alpha, b, D, l, gamma)
    try:
        rng = np.random.default_rng(7)
        for i in range(sp.np):
            pr = ks.Prime(sp, i)
            p = int(pr.p)
            zeta = pow(_omega(p, sp.M, t), sp.M // t, p)
            xs = rng.integers(0, 2 * p, size=(t, 4096), dtype=np.int64).astype(np.uint64)
            xs[:, :128] = rng.choice([0, 2 * p - 1], size=(t, 128)).astype(np.uint64)
            xs[t - 1, 128:256] = 0  # the fused first step's zero input
            for inv in (False, True):
                z = pow(zeta, -1, p) if inv else zeta
                for red in (False, True):
                    ys = pr.dft_k(list(xs), inv=inv, red=red)
                    X = xs.astype(object)
                    for k in range(t):
                        want = sum(X[n] * pow(z, n * k, p) for n in range(t)) % p
                        got = ys[k].astype(object) % p
                        assert np.array_equal(got, want), (i, inv, red, k)
                        if red or k == 0:
                            assert np.all(ys[k] < 2 * p)
    finally:
        sp.close()


@pytest.mark.parametrize("gamma,D,l", [(0, 4096, 3), (1, 65536, 2)])
def test_winograd_inverse_first_step_matches_matrix(gamma, D, l):
    """inv_first7 (keyswitch.cu, t = 7) equals the (t-1)x(t-1) CRT-weighted solve sum_r C_r g[j][r]
    it replaces, fully reduced, for random and extreme inputs < 2p."""
    import kernel_sim as ks
    sp = ks.SimPlan(7, 4, 12, D, l, gamma)
    try:
        rng = np.random.default_rng(11)
        for i in range(sp.np):
            pr = ks.Prime(sp, i)
            p = int(pr.p)
            Cs = rng.integers(0, 2 * p, size=(6, 2048), dtype=np.int64).astype(np.uint64)
            Cs[:, :64] = rng.choice([0, 2 * p - 1], size=(6, 64)).astype(np.uint64)
            got = pr.inv_first7(list(Cs))
            R_inv = pow(1 << 32, -1, p)
            G = pr.g.astype(object)
            X = Cs.astype(object)
            for j in range(6):
                want = sum(X[r] * G[j][r] for r in range(6)) * R_inv % p
                assert np.array_equal(got[j].astype(object), want), (i, j)
    finally:
        sp.close()


def _omega(p, M, t):
    """The planner's primitive M-th root (plan.cpp: first x whose (p-1)/M power has order M)."""
    for x in range(2, p):
        w = pow(x, (p - 1) // M, p)
        if pow(w, M // t, p) != 1:
            return w


@pytest.mark.parametrize("b,gamma", [(8, 0), (12, 0), (12, 1), (16, 0), (16, 1)])
def test_closed_form_digits_match_reference_decomposition(b, gamma):
    """The device's per-digit closed forms (keyswitch.cu digit_i) with the library's
    decM / decDp tables reproduce reference crypto.gadget_decompose exactly."""
    import kernel_sim as ks
    sch = osc.preset(b, gamma)
    R, g = sch.ring, sch.gadget
    sp = ks.SimPlan(R.t, R.alpha, R.p_bits, g.D, g.l, gamma)
    try:
        rc = sp.rc
        v = u53(9, 3000)
        v[:6] = [0, 1, (1 << 53) - 1, 1 << 52, (1 << 52) + 1, (1 << 53) // g.D]
        want = oks.decompose(v, g)

        def digit(y, i):
            y = int(y)
            if rc.dlog2 >= 0:
                u = (y + (1 << (rc.shift - 1))) >> rc.shift
                low = rc.dlog2 * (rc.l - 1 - i)
                x = ((u >> low) & (rc.D - 1)) + (1 if (u & ((1 << low) - 1)) > rc.decM[i] else 0)
                return x - rc.D if x > rc.D // 2 else x
            r = y - (1 << 53) if y > (1 << 52) else y
            F = lambda k: (r * rc.decDp[k] + (1 << 52)) >> 53  # noqa: E731
            return F(i) - (rc.D * F(i - 1) if i else 0)

        got = np.array([[digit(y, i) for y in v] for i in range(g.l)])
        assert np.array_equal(got, want)
    finally:
        sp.close()
