"""GPU edge cases: empty and ragged batches, all-zero rows and the skip_zero
KS counting (reference tracepack.py:268-285, 299-303), extraction at 1 and N
rows, missing key indices, and the RNS NTT on an empty batch.  Bit-exact
against the oracle wherever there is an output."""

import numpy as np
import pytest

from conftest import has_cuda, u53
from oracle import keyswitch as oks
from oracle import pack as opk
from oracle import protocol as opr
from oracle import scheme as osc

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


def _engine(b, gamma, seed=3):
    from paper_2509_01253_b200.keyswitch import KeySwitchEngine, KeySwitchKeySet
    from paper_2509_01253_b200.params import GadgetParams, RingParams
    sch = osc.preset(b, gamma)
    ksk = opr.OracleClient(sch, seed=seed).make_ksk()
    R = RingParams(sch.ring.t, sch.ring.alpha, sch.ring.p_bits)
    g = GadgetParams(sch.gadget.D, sch.gadget.l)
    eng = KeySwitchEngine(KeySwitchKeySet(ksk.keys, g, ksk.delta, R), gamma=gamma)
    return sch, ksk, eng


@pytest.mark.parametrize("b", [8, 12, 16])
def test_empty_batches(b):
    sch, ksk, eng = _engine(b, 1)
    N = sch.ring.N
    d = sorted(ksk.keys)[0]
    empty = np.zeros((0, 2, N), np.uint64)
    assert eng.switch_batch(empty, d).shape == (0, 2, N)
    assert eng.automorphism_batch(empty, d).shape == (0, 2, N)
    assert eng.stage_batch(empty, [1, d]).shape == (0, 2, N)


@pytest.mark.parametrize("b,gamma", [(8, 0), (12, 1), (16, 2)])
def test_zero_rows_skip_zero_counting(b, gamma):
    """Zero rows switch to zero and are not counted with skip_zero (the padding of the
    last pack group); counted otherwise.  Ragged batch sizes (1, 7, 130)."""
    from paper_2509_01253_b200.tracepack import KsCounter
    sch, ksk, eng = _engine(b, gamma)
    ref = oks.KsEngine(ksk, "exact")
    R = sch.ring
    reps = opk.stage_reps_above(R.alpha - 1, R)
    for B in (1, 7, 130):
        x = u53(B, (B, 2, R.N))
        x[::3] = 0
        live = int(np.any(x.reshape(B, -1) != 0, axis=1).sum())
        for skip in (True, False):
            c = KsCounter()
            got = eng.stage_batch(x, reps, counter=c, skip_zero=skip)
            assert c.total_key_switches == (live if skip else B) * (len(reps) - 1)
            assert np.all(got[::3] == 0)
        if B <= 7:  # exact oracle is slow: check the values on the small batches
            assert np.array_equal(got, opk.apply_stage(x, reps, ref, None, False))


@pytest.mark.parametrize("b", [8, 16])
def test_extract_one_and_full_chunk(b):
    from paper_2509_01253_b200.params import RingParams
    from paper_2509_01253_b200.tracepack import PowerBundle, partial_extract, power_exponents
    from paper_2509_01253_b200.keyswitch import RlweCiphertext
    sch = osc.preset(b, 1)
    R = sch.ring
    Rm = RingParams(R.t, R.alpha, R.p_bits)
    exps = power_exponents(1, Rm)
    power = u53(77, (len(exps), 2, R.N))
    bundle = PowerBundle(1, {d: RlweCiphertext(power[q, 0], power[q, 1]) for q, d in enumerate(exps)})
    obundle = opk.Bundle(1, {d: oks.Ct(power[q, 0], power[q, 1]) for q, d in enumerate(exps)})
    full = partial_extract(bundle, None, R.N, Rm)
    one = partial_extract(bundle, None, 1, Rm)
    assert one.shape == (1, 2, R.N) and np.array_equal(one[0], full[0])
    assert np.array_equal(full, opk.extract(obundle, R.N, R))
    with pytest.raises(ValueError):
        partial_extract(bundle, None, R.N + 1, Rm)


@pytest.mark.parametrize("b,gamma", [(8, 0), (12, 0), (16, 0), (8, 1), (12, 1), (16, 1), (8, 2), (12, 2), (16, 2)])
def test_extract_kernels_agree(b, gamma, monkeypatch):
    """The offset-table kernel (< 6 powers; one component at a time when both do not fit), the
    many-power kernel (>= 6 powers), the general kernels and the oracle agree bit for bit."""
    from paper_2509_01253_b200.params import RingParams
    from paper_2509_01253_b200.tracepack import PowerBundle, partial_extract, power_exponents
    from paper_2509_01253_b200.keyswitch import RlweCiphertext
    sch = osc.preset(b, gamma)
    R = sch.ring
    Rm = RingParams(R.t, R.alpha, R.p_bits)
    exps = power_exponents(gamma, Rm)
    power = u53(91 + b, (len(exps), 2, R.N))
    bundle = PowerBundle(gamma, {d: RlweCiphertext(power[q, 0], power[q, 1]) for q, d in enumerate(exps)})
    obundle = opk.Bundle(gamma, {d: oks.Ct(power[q, 0], power[q, 1]) for q, d in enumerate(exps)})
    fast = partial_extract(bundle, None, R.N, Rm)
    monkeypatch.setenv("SFHR_EXTRACT_TILED", "1")
    tiled = partial_extract(bundle, None, R.N, Rm)
    assert np.array_equal(fast, tiled)
    assert np.array_equal(fast, opk.extract(obundle, R.N, R))


def test_missing_key_index_raises():
    sch, ksk, eng = _engine(12, 1)
    N = sch.ring.N
    bad = max(ksk.keys) + 1
    while bad in ksk.keys:
        bad += 1
    with pytest.raises(KeyError):
        eng.switch_batch(np.zeros((2, 2, N), np.uint64), bad)
    with pytest.raises(KeyError):
        eng.stage_batch(np.zeros((2, 2, N), np.uint64), [1, bad])


def test_ntt_empty_batch_and_bad_shapes():
    import torch
    from paper_2509_01253_b200.ntt import RnsNtt
    pl = RnsNtt(12, 2, 50, device=0)
    x = torch.zeros((0, 2, 1 << 12), dtype=torch.int64, device="cuda")
    assert pl.forward(x).shape == (0, 2, 1 << 12)
    with pytest.raises(ValueError):
        pl.forward(torch.zeros((1, 3, 1 << 12), dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        pl.forward(torch.zeros((1, 2, 1 << 12), dtype=torch.int32, device="cuda"))


def test_concurrent_sessions_match_sequential():
    """Three client threads on one engine (the reference's one-thread-per-connection
    server, transport.py:136-156) get exactly the packs of a sequential run."""
    import threading
    from paper_2509_01253_b200.engine import ServerEngine
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet
    from paper_2509_01253_b200.params import GadgetParams, RingParams, SchemeParams
    from paper_2509_01253_b200.workloads import toy_model
    from oracle import lowering as olo
    b, gamma = 12, 1
    sch = osc.preset(b, gamma)
    R = RingParams(sch.ring.t, sch.ring.alpha, sch.ring.p_bits)
    g = GadgetParams(sch.gadget.D, sch.gadget.l)
    mys = SchemeParams(R, sch.delta, g, gamma, sch.beta)
    model = toy_model(b, 5)
    rounds = olo.build_rounds(model.layers)
    ksks, bundles = [], []
    for i in range(3):  # the client RNG draws happen once; both servers see the same uploads
        cl = opr.OracleClient(sch, seed=40 + i)
        ksks.append(cl.make_ksk())
        x = np.random.default_rng(50 + i).integers(0, 4, model.input_shape)
        bundles.append(cl.prepare_round(np.asarray(x).reshape(-1), rounds[0].input_len))

    def run(server, i, out):
        kid = server.register_client(KeySwitchKeySet(ksks[i].keys, g, 0.0, R))
        sid = bytes([i + 1]) * 16
        server.open_session(sid, kid)
        packs, _ = server.server_round(sid, 1, bundles[i])
        out[i] = np.stack(packs)

    seq, par = {}, {}
    s1 = ServerEngine(model, mys, master_seed=bytes(range(32)))
    for i in range(3):
        run(s1, i, seq)
    s2 = ServerEngine(model, mys, master_seed=bytes(range(32)))
    th = [threading.Thread(target=run, args=(s2, i, par)) for i in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(3):
        assert np.array_equal(seq[i], par[i]), i


@pytest.mark.parametrize("b,gamma,E_frac", [(12, 2, 2.4), (16, 2, 1.7), (12, 1, 2.4), (8, 2, 1.3), (16, 1, 2.0)])
def test_extract_multi_chunk_ragged(b, gamma, E_frac):
    """Several chunks and a ragged last one through extract_device (the round path): rows of
    chunk j are extracted from chunk j's powers only, the tail stops at E, bit-exact vs the
    oracle chunk by chunk (many-power and offset-table kernels)."""
    import torch
    from paper_2509_01253_b200.params import RingParams
    from paper_2509_01253_b200.device import RingContext, to_dev, to_host_u64
    from paper_2509_01253_b200.tracepack import extract_device, power_exponents
    sch = osc.preset(b, gamma)
    R = sch.ring
    Rm = RingParams(R.t, R.alpha, R.p_bits)
    exps = power_exponents(gamma, Rm)
    E = int(E_frac * R.N)
    k = -(-E // R.N)
    power = u53(300 + b + gamma, (k, len(exps), 2, R.N))
    ctx = RingContext.get(R.t, R.alpha, R.p_bits, sch.gadget.D, sch.gadget.l, gamma, 0, 0)
    rows = to_host_u64(extract_device(ctx, to_dev(power, ctx.dev), exps, E))
    assert rows.shape == (E, 2, R.N)
    for j in range(k):
        cnt = min(R.N, E - j * R.N)
        ob = opk.Bundle(gamma, {d: oks.Ct(power[j, q, 0], power[j, q, 1]) for q, d in enumerate(exps)})
        assert np.array_equal(rows[j * R.N:j * R.N + cnt], opk.extract(ob, cnt, R)), j


def test_misaligned_rows():
    """The stage kernel bulk-copies rows (16-byte granules): the C-ABI rejects misaligned
    in/out with SFHR_EINVAL, and the Python engine copies a misaligned view first, so its
    result equals the aligned call's."""
    import ctypes
    import torch
    from paper_2509_01253_b200 import _native as nat
    sch, ksk, eng = _engine(12, 1)
    N = sch.ring.N
    d = sorted(k for k in ksk.keys if k != 1)[0]
    x = torch.from_numpy(u53(5, (3, 2, N)).view(np.int64)).cuda()
    big = torch.zeros(3 * 2 * N + 1, dtype=torch.int64, device="cuda")
    big[1:] = x.reshape(-1)
    mis = big[1:].view(3, 2, N)
    assert mis.data_ptr() % 16 == 8
    ref = eng.switch_batch(x, d)
    assert torch.equal(eng.switch_batch(mis, d), ref)
    out = torch.empty_like(x)
    code = nat.lib.sfhr_keyswitch_batch(eng.ctx.h, eng.key.h, d % eng.ctx.M, nat.ptr(mis), nat.ptr(out), 3, 0,
                                        None, eng.ctx.stream())
    assert code == nat.SFHR_EINVAL and "aligned" in nat.last_error()
