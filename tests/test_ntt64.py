"""Standalone RNS negacyclic NTT (BASELINE configs[1]; csrc/ntt64.cu).

No reference oracle exists for power-of-two rings: the C
oracle (oracle/ntt_ref.c) is pinned by self-consistency (round trip and
NTT-convolution = schoolbook), and the CUDA transforms must equal it
bit-for-bit (fully reduced residues, same bit-reversed output order)."""

import numpy as np
import pytest

from conftest import has_cuda
from oracle import ntt as on


@pytest.mark.parametrize("logn", [10, 12])
def test_oracle_roundtrip_and_convolution(logn):
    from paper_2509_01253_b200.ntt import RnsNtt
    pl = RnsNtt(logn, 2, 50, device=-1)
    for p in pl.primes.tolist():
        rng = np.random.default_rng(p & 0xFFFF)
        a = rng.integers(0, p, 1 << logn, dtype=np.uint64)
        b = rng.integers(0, p, 1 << logn, dtype=np.uint64)
        assert np.array_equal(on.inverse(on.forward(a, p), p), a)
        c = on.inverse(on.pointwise(on.forward(a, p), on.forward(b, p), p), p)
        assert np.array_equal(c, on.negacyclic(a, b, p))
    # X * X^(N-1) = -1 in Z_p[X]/(X^N + 1)
    p = int(pl.primes[0])
    n = 1 << logn
    x1 = np.zeros(n, np.uint64)
    x1[1] = 1
    xn = np.zeros(n, np.uint64)
    xn[n - 1] = 1
    c = on.inverse(on.pointwise(on.forward(x1, p), on.forward(xn, p), p), p)
    want = np.zeros(n, np.uint64)
    want[0] = p - 1
    assert np.array_equal(c, want)


@pytest.mark.parametrize("logn,L,bits", [(14, 4, 50), (16, 16, 50), (10, 32, 50), (13, 3, 30)])
def test_plan_primes_and_twiddles(logn, L, bits):
    from paper_2509_01253_b200.ntt import RnsNtt
    pl = RnsNtt(logn, L, bits, device=-1)
    n = 1 << logn
    pr = [int(p) for p in pl.primes]
    assert len(set(pr)) == L and all(p < (1 << bits) and p % (2 * n) == 1 for p in pr)
    assert all(pow(3, p - 1, p) == 1 and pow(5, p - 1, p) == 1 for p in pr)
    w, wi = pl.tables()
    for i in (0, L - 1):
        p = pr[i]
        psi = on.psi(p, logn)
        assert pow(psi, n, p) == p - 1
        for k in (1, 2, 3, n // 2 + 1, n - 1):
            e = int(format(k, f"0{logn}b")[::-1], 2)
            assert int(w[i, k]) == pow(psi, e, p)
            assert int(wi[i, k]) == pow(psi, (2 * n - e) % (2 * n), p)
        assert int(wi[i, 0]) * n % p == 1


def test_plan_rejects_bad_parameters():
    from paper_2509_01253_b200.ntt import RnsNtt
    for args in [(9, 1, 50), (17, 1, 50), (14, 0, 50), (14, 33, 50), (14, 1, 51), (14, 1, 29)]:
        with pytest.raises(ValueError):
            RnsNtt(*args, device=-1)




@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("logn", [10, 11, 12, 13, 14, 15, 16])
def test_gpu_forward_inverse_match_oracle(logn):
    import torch
    from paper_2509_01253_b200.ntt import RnsNtt
    L, B = 3, 2
    pl = RnsNtt(logn, L, 50, device=0)
    rng = np.random.default_rng(logn)
    n = 1 << logn
    x = np.stack([np.stack([rng.integers(0, int(p), n, dtype=np.uint64) for p in pl.primes]) for _ in range(B)])
    d = torch.from_numpy(x.view(np.int64)).cuda()
    pl.forward(d)
    y = d.cpu().numpy().view(np.uint64)
    for b in range(B):
        for i, p in enumerate(pl.primes.tolist()):
            assert np.array_equal(y[b, i], on.forward(x[b, i], p)), (b, i)
    pl.inverse(d)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), x)


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("logn,L,B", [(14, 16, 8), (15, 8, 4), (16, 16, 4), (16, 4, 64)])
def test_gpu_roundtrip_full_size(logn, L, B):
    import torch
    from paper_2509_01253_b200.ntt import RnsNtt
    pl = RnsNtt(logn, L, 50, device=0)
    P = torch.tensor(pl.primes.view(np.int64), device="cuda")
    g = torch.Generator(device="cuda").manual_seed(logn * 1000 + L)
    x = torch.randint(0, 1 << 62, (B, L, 1 << logn), device="cuda", generator=g, dtype=torch.int64)
    x = torch.remainder(x, P[None, :, None])
    y = x.clone()
    pl.forward(y)
    assert not torch.equal(x, y)
    pl.inverse(y)
    assert torch.equal(x, y)


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_gpu_convolution_matches_schoolbook():
    import torch
    from paper_2509_01253_b200.ntt import RnsNtt
    logn = 14
    pl = RnsNtt(logn, 1, 50, device=0)
    p = int(pl.primes[0])
    rng = np.random.default_rng(7)
    a = rng.integers(0, p, 1 << logn, dtype=np.uint64)
    b = rng.integers(0, p, 1 << logn, dtype=np.uint64)
    da = torch.from_numpy(a.view(np.int64).reshape(1, 1, -1).copy()).cuda()
    db = torch.from_numpy(b.view(np.int64).reshape(1, 1, -1).copy()).cuda()
    pl.forward(da)
    pl.forward(db)
    c = on.pointwise(da.cpu().numpy().view(np.uint64).ravel(), db.cpu().numpy().view(np.uint64).ravel(), p)
    dc = torch.from_numpy(c.view(np.int64).reshape(1, 1, -1).copy()).cuda()
    pl.inverse(dc)
    assert np.array_equal(dc.cpu().numpy().view(np.uint64).ravel(), on.negacyclic(a, b, p))
