"""Client-side batch operations with the key product on the GPU:
identical to the oracle client (pinned to the reference's client keys and encryptions,
tests/golden) for the same key, the same generator state and the same inputs."""

import numpy as np
import pytest

from conftest import has_cuda, u53
from oracle import keyswitch as oks
from oracle import scheme as osc


@pytest.mark.parametrize("b,dist", [(8, "binary"), (12, "ternary"), (16, "binary")])
def test_key_matrix_matches_reference_operator(b, dist):
    from paper_2509_01253_b200.client_ops import key_matrix
    from paper_2509_01253_b200.params import RingParams
    R = osc.preset(b, 0).ring
    sk = oks.keygen(R, dist, seed=b)
    mat = key_matrix(sk.s, RingParams(R.t, R.alpha, R.p_bits))
    assert np.array_equal(mat, oks._key_matrix(sk).astype(np.int64))
    assert np.abs(mat).max() <= 2


gpu = pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")


@pytest.mark.gpu
@gpu
@pytest.mark.parametrize("b,dist", [(8, "binary"), (12, "ternary"), (16, "binary")])
def test_gpu_key_product_encrypt_phase_match_oracle(b, dist):
    from paper_2509_01253_b200.client_ops import (KeyMul, encrypt_rlwe_batch, project_p,
                                                  rlwe_phase_batch)
    from paper_2509_01253_b200.params import RingParams
    sch = osc.preset(b, 0)
    R = sch.ring
    Rm = RingParams(R.t, R.alpha, R.p_bits)
    sk = oks.keygen(R, dist, seed=7)
    km = KeyMul(sk.s, Rm)
    for B in (1, 3, 64):
        v = u53(B, (B, R.N))
        assert np.array_equal(km.times(v), oks.key_times(sk, v)), B
    dual = osc.dual_for(R.t, R.alpha, R.p_bits)
    msgs = np.random.default_rng(3).integers(0, R.p, (5, R.N))
    payloads = oks.lift(msgs, R)
    got = encrypt_rlwe_batch(payloads, km, sch.delta, np.random.default_rng(11), dual.scatter_idx,
                             dual.scatter_coef)
    want = oks.encrypt_batch(payloads, sk, sch.delta, np.random.default_rng(11), dual)
    assert np.array_equal(got, want)
    ph = rlwe_phase_batch(got, km)
    assert np.array_equal(ph, oks.phase_batch(want, sk))
    assert np.array_equal(project_p(ph, Rm), msgs)
