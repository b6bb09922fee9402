"""CPU check of the tensor-core forward key-switch arithmetic (tests/tc_model.py)
against the CUDA-core kernel's bit-level model (tests/kernel_sim.py): the two-pass
byte-plane GEMM formulation gives the same NTT-domain accumulators, mod p, at
the old kernel's positions (old_idx), with every intermediate in range."""

import numpy as np
import pytest

from conftest import u53
from kernel_sim import Prime, SimPlan, forward, key_spectrum
from oracle import keyswitch as oks
from oracle import scheme as osc
from tc_model import TcTables


def _omega(pr):
    p = int(pr.p)
    return int(pr.wt[1]) * pow((1 << 32) % p, -1, p) % p


@pytest.mark.parametrize("b,gamma", [(12, 0), (12, 1), (16, 0), (16, 1), (8, 0)])
def test_tc_forward_mac_matches_kernel_model(b, gamma):
    sch = osc.preset(b, gamma)
    R = sch.ring
    sp = SimPlan(R.t, R.alpha, R.p_bits, sch.gadget.D, sch.gadget.l, gamma, 0)
    try:
        rng = np.random.default_rng(b * 10 + gamma)
        x = u53(b + gamma, (R.N,))
        digs = oks.decompose(x, sch.gadget)                 # (l, N) balanced digits
        keys = [u53(100 + i, (R.N,)) for i in range(sch.gadget.l)]
        for ip in range(sp.np):
            pr = Prime(sp, ip)
            p = int(pr.p)
            tc = TcTables(R.t, R.alpha, p, _omega(pr), sch.gadget.D)
            acc_old = np.zeros(R.N, dtype=object)
            acc_new = np.zeros((tc.SA, tc.SB), dtype=object)
            for li in range(sch.gadget.l):
                dm = np.where(digs[li] < 0, digs[li] + p, digs[li]).astype(np.uint64)
                fo = forward(sp, pr, dm).reshape(-1).astype(object)
                ks = key_spectrum(sp, pr, keys[li]).reshape(-1).astype(object)  # K^ R
                acc_old += fo * ks * pow(1 << 32, -1, p)
                lohi = tc.forward_digit(digs[li])
                acc_new += tc.mac(lohi, ks[tc.old_idx])
            acc_old %= p
            assert np.array_equal(acc_new % p, acc_old[tc.old_idx]), (b, gamma, ip)
            assert sorted(tc.old_idx.reshape(-1).tolist()) == list(range(R.N))
    finally:
        sp.close()


def _kmaj(k, n, ncols):
    return ((k // 16) * (ncols // 8) + n // 8) * 128 + (n % 8) * 16 + (k % 16)


@pytest.mark.parametrize("gamma", [0, 1])
def test_library_tc_tables_match_model(gamma):
    """The constant operands the library builds (canonical UMMA K-major byte layout) are the
    byte planes of tc_model's folded matrices, the twiddle pairs and the NTT-order map."""
    import ctypes as C
    from paper_2509_01253_b200 import _native as nat
    sch = osc.preset(12, gamma)
    R = sch.ring
    sp = SimPlan(R.t, R.alpha, R.p_bits, sch.gadget.D, sch.gadget.l, gamma, 0)
    try:
        nbytes = nat.lib.sfhr_tc_table_bytes(sp.h)
        assert nbytes > 0
        tabs = np.zeros(nbytes, np.uint8)
        oi = np.zeros(42 * 49, np.int32)
        nat.check(nat.lib.sfhr_ctx_tc_tables(sp.h, tabs.ctypes.data, nbytes, oi.ctypes.data))
        per = nbytes // sp.np
        KA, NA, KB, NBH = 96, 176, 224, 112
        BA_B, BB_B = KA * NA, KB * NBH
        for ip in range(sp.np):
            pr = Prime(sp, ip)
            tc = TcTables(R.t, R.alpha, int(pr.p), _omega(pr), sch.gadget.D)
            blob = tabs[ip * per:(ip + 1) * per]
            assert np.array_equal(oi.reshape(42, 49), tc.old_idx)
            kk, oo = np.meshgrid(np.arange(2 * tc.SA + 1), np.arange(tc.SA), indexing="ij")
            for b in range(4):
                got = blob[_kmaj(kk, b * 44 + oo, NA)]
                assert np.array_equal(got, np.asarray((tc.CA >> (8 * b)) & 255, dtype=np.uint8)), b
            kk, k1 = np.meshgrid(np.arange(4 * tc.SB), np.arange(tc.SB), indexing="ij")
            h = (k1 >= 25).astype(int)
            for b in range(4):
                got = blob[BA_B + h * BB_B + _kmaj(kk, b * 28 + k1 - 25 * h, NBH)]
                assert np.array_equal(got, np.asarray((tc.CB >> (8 * b)) & 255, dtype=np.uint8)), b
            tw = blob[BA_B + 2 * BB_B:].view(np.uint32)[:49 * 43 * 2].reshape(49, 43, 2)
            assert np.array_equal(tw[:, :42, 0], np.asarray(tc.TWm.T, dtype=np.uint32))
            assert np.array_equal(tw[:, :42, 1], np.asarray(tc.TWm2.T, dtype=np.uint32))
    finally:
        sp.close()
