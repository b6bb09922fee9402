"""GPU parity of the tensor-core forward key switch (csrc/keyswitch_tc.cu, ring row
b = 12): every stage / switch launch is bit-identical to the CPU oracle and to the
CUDA-core kernel (ks_stage_kernel's own forward, sfhr_ctx_set_tc(ctx, 0)), including
odd batch sizes (a half-empty last row pair), zero rows and multi-chunk launches."""

import numpy as np
import pytest

from conftest import has_cuda, u53
from oracle import keyswitch as oks
from oracle import pack as opk
from oracle import protocol as opr
from oracle import scheme as osc

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


def _engine(sch, ksk):
    from paper_2509_01253_b200.keyswitch import KeySwitchEngine, KeySwitchKeySet
    from paper_2509_01253_b200.params import GadgetParams, RingParams
    R = RingParams(sch.ring.t, sch.ring.alpha, sch.ring.p_bits)
    g = GadgetParams(sch.gadget.D, sch.gadget.l)
    return KeySwitchEngine(KeySwitchKeySet(ksk.keys, g, ksk.delta, R), gamma=sch.gamma)


def _both(eng, fn):
    ctx = eng.ctx
    keep = ctx.tensor_core_min_reps
    try:
        ctx.tensor_core_min_reps = 1  # every stage / switch launch on the tensor-core forward
        got = fn()
        ctx.tensor_core_min_reps = 0  # CUDA-core forward of ks_stage_kernel
        want = fn()
    finally:
        ctx.tensor_core_min_reps = keep
    return got, want


@pytest.mark.parametrize("gamma", [0, 1])
def test_tc_stage_matches_oracle(gamma):
    sch = osc.preset(12, gamma)
    ksk = opr.OracleClient(sch, seed=40 + gamma).make_ksk()
    eng = _engine(sch, ksk)
    keep = eng.ctx.tensor_core_min_reps
    eng.ctx.tensor_core_min_reps = 1
    try:
        _stage_vs_oracle(sch, ksk, eng, gamma)
    finally:
        eng.ctx.tensor_core_min_reps = keep


def _stage_vs_oracle(sch, ksk, eng, gamma):
    ref = oks.KsEngine(ksk, "fft")
    R = sch.ring
    x = u53(500 + gamma, (5, 2, R.N))
    x[3] = 0
    stages = [opk.stage_reps_above(j, R) for j in range(max(gamma, 1), R.alpha)]
    if gamma == 0:
        stages += opk.stage0_chains(R)
    for reps in stages:
        from paper_2509_01253_b200.tracepack import KsCounter
        c1, c2 = KsCounter(), opk.Counter()
        got = eng.stage_batch(x, reps, counter=c1, skip_zero=True)
        want = opk.apply_stage(x, reps, ref, c2, True)
        assert np.array_equal(got, want), reps
        assert c1.total_key_switches == c2.total_key_switches
    for d in opr.required_ksk_indices(sch)[:3]:
        moved = ref.automorphism_batch(x[:3], d)
        assert np.array_equal(eng.switch_batch(moved, d), ref.switch_batch(moved, d)), d


@pytest.mark.parametrize("gamma,B", [(0, 1), (0, 2), (0, 37), (1, 300), (0, 2100)])
def test_tc_matches_cuda_core_kernel(gamma, B):
    import torch
    sch = osc.preset(12, gamma)
    R = sch.ring
    rng = np.random.default_rng(B)
    keys = {d: [oks.Ct(rng.integers(0, 1 << 53, R.N, dtype=np.uint64),
                       rng.integers(0, 1 << 53, R.N, dtype=np.uint64)) for _ in range(sch.gadget.l)]
            for d in opr.required_ksk_indices(sch)}
    eng = _engine(sch, oks.KskSet(keys, sch.gadget, 0.0, R))
    x = torch.from_numpy(u53(B + 7, (B, 2, R.N)).view(np.int64)).cuda()
    if B > 3:
        x[B // 2] = 0
    for reps in [opk.stage_reps_above(j, R) for j in range(max(gamma, 1), R.alpha)][:2]:
        got, want = _both(eng, lambda: eng.stage_batch(x, reps, skip_zero=True))
        assert torch.equal(got, want), reps
    d = opr.required_ksk_indices(sch)[-1]
    got, want = _both(eng, lambda: eng.switch_batch(x, d))
    assert torch.equal(got, want)
