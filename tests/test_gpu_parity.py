"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle and the
reference's golden fixtures.  Bit-exact for every integer output."""

import numpy as np
import pytest

from conftest import digest, has_cuda, u53
from oracle import keyswitch as oks
from oracle import lowering as olo
from oracle import pack as opk
from oracle import protocol as opr
from oracle import scheme as osc

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


def _ring(sch):
    from paper_2509_01253_b200.params import GadgetParams, RingParams
    return RingParams(sch.ring.t, sch.ring.alpha, sch.ring.p_bits), \
        GadgetParams(sch.gadget.D, sch.gadget.l)


def _engine_for(ksk, sch, gamma=0):
    from paper_2509_01253_b200.keyswitch import KeySwitchEngine, KeySwitchKeySet
    R, g = _ring(sch)
    mine = KeySwitchKeySet(keys=ksk.keys, gadget=g, delta=ksk.delta, params=R)
    return KeySwitchEngine(mine, mode="cuda", gamma=gamma)


def _scheme(sch):
    from paper_2509_01253_b200.params import SchemeParams
    R, g = _ring(sch)
    return SchemeParams(R, sch.delta, g, sch.gamma, sch.beta)


@pytest.mark.parametrize("row", range(9))
def test_keyswitch_matches_golden_and_oracle(golden, row):
    r = golden["rows"][row]
    sch = osc.preset(r["b"], r["gamma"])
    ksk = opr.OracleClient(sch, seed=r["client_seed"]).make_ksk()
    eng = _engine_for(ksk, sch)
    x = u53(r["ks_input_seed"], (3, 2, sch.ring.N))
    for case in r["ks"]:
        moved = eng.automorphism_batch(x, case["d"])
        assert digest(moved) == case["aut_digest"]
        out = eng.switch_batch(moved, case["d"])
        assert digest(out) == case["exact_digest"]
    # every index of the key set, against the exact oracle on one row
    ref = oks.KsEngine(ksk, "exact")
    for d in r["indices"]:
        moved = ref.automorphism_batch(x[:1], d)
        assert np.array_equal(eng.switch_batch(moved, d), ref.switch_batch(moved, d)), d


@pytest.mark.parametrize("row", [0, 3, 4, 6])
def test_stage_batch_matches_oracle(golden, row):
    r = golden["rows"][row]
    sch = osc.preset(r["b"], r["gamma"])
    ksk = opr.OracleClient(sch, seed=r["client_seed"]).make_ksk()
    eng = _engine_for(ksk, sch)
    ref = oks.KsEngine(ksk, "fft")
    R = sch.ring
    x = u53(77 + row, (5, 2, R.N))
    x[2] = 0  # zero row: skipped and not counted when skip_zero
    stages = [opk.stage_reps_above(j, R) for j in range(max(sch.gamma, 1), R.alpha)]
    if sch.gamma == 0:
        stages += opk.stage0_chains(R)
    for reps in stages:
        from paper_2509_01253_b200.tracepack import KsCounter
        c1, c2 = KsCounter(), opk.Counter()
        got = eng.stage_batch(x, reps, counter=c1, skip_zero=True)
        want = opk.apply_stage(x, reps, ref, c2, True)
        assert np.array_equal(got, want), reps
        assert c1.total_key_switches == c2.total_key_switches == 4 * (len(reps) - 1)


@pytest.mark.parametrize("row", range(9))
def test_extract_matches_golden(golden, row):
    from paper_2509_01253_b200 import tracepack as tp
    r = golden["rows"][row]
    sch = osc.preset(r["b"], r["gamma"])
    R = sch.ring
    cl = opr.OracleClient(sch, seed=r["client_seed"])
    cl.make_ksk()
    v = np.random.default_rng(r["extract"]["msg_seed"]).integers(-3, 4, R.N)
    bundle = cl.prepare_round(v, R.N)[0]
    Rm, _ = _ring(sch)
    assert digest(tp.partial_extract(bundle, None, R.N, Rm)) == r["extract"]["rows_digest"]
    assert digest(tp.partial_extract(bundle, None, 37, Rm)) == r["extract"]["rows37_digest"]


@pytest.mark.parametrize("row", range(9))
def test_fast_pack_matches_golden(golden, row):
    from paper_2509_01253_b200 import tracepack as tp
    r = golden["rows"][row]
    sch = osc.preset(r["b"], r["gamma"])
    ksk = opr.OracleClient(sch, seed=r["client_seed"]).make_ksk()
    eng = _engine_for(ksk, sch, sch.gamma)
    mys = _scheme(sch)
    F = r["pack"]["F"]
    grp = u53(r["pack"]["seed"], (F, 2, sch.ring.N))
    cnt = tp.KsCounter()
    pk = tp.fast_pack(grp, mys, eng, counter=cnt, skip_zero=True)
    assert digest(pk) == r["pack"]["digest"]
    assert cnt.total_key_switches == r["pack"]["ks"]
    grp2 = grp.copy()
    grp2[F // 3:] = 0
    cnt2 = tp.KsCounter()
    pk2 = tp.pack_rows(grp2[:r["pack"]["tail_rows"]], mys, eng, counter=cnt2)
    assert digest(np.stack(pk2)) == r["pack"]["tail_digest"]
    assert cnt2.total_key_switches == r["pack"]["tail_ks"]


def test_m27_pack_matches_golden(golden):
    from paper_2509_01253_b200 import tracepack as tp
    from paper_2509_01253_b200.keyswitch import KeySwitchEngine, KeySwitchKeySet
    from paper_2509_01253_b200.params import GadgetParams, RingParams, SchemeParams
    R = osc.Ring(3, 3, 8)
    for c in golden["m27"]:
        sch = osc.Scheme(R, 2.0 ** -36, osc.Gadget(512, 3), c["gamma"])
        sk = oks.keygen(R, seed=31)
        ksk = oks.make_ksk(sk, c["indices"], sch.gadget, sch.delta, np.random.default_rng(32),
                           osc.dual_for(3, 3, 8))
        Rm, g = RingParams(3, 3, 8), GadgetParams(512, 3)
        eng = KeySwitchEngine(KeySwitchKeySet(ksk.keys, g, ksk.delta, Rm), gamma=c["gamma"])
        mys = SchemeParams(Rm, 2.0 ** -36, g, c["gamma"])
        grp = u53(c["seed"], (mys.pack_factor, 2, R.N))
        cnt = tp.KsCounter()
        pk = tp.fast_pack(grp, mys, eng, counter=cnt)
        assert digest(pk) == c["digest"] and cnt.total_key_switches == c["ks"]


def test_linear_matches_golden(golden):
    from paper_2509_01253_b200 import linear as lin
    c = golden["int_matmul"]
    w = np.random.default_rng(c["w_seed"]).integers(-7, 8, (5, 9))
    rows = u53(c["rows_seed"], (9, 2, 11))
    assert digest(lin.int_matmul_mod_q(w, rows)) == c["digest"]
    c = golden["enc_linear"]
    sch = osc.preset(c["b"], c["gamma"])
    W = np.random.default_rng(c["w_seed"]).integers(-3, 4, (40, 70))
    bias = np.random.default_rng(c["bias_seed"]).integers(-9, 10, 40)
    rows = u53(c["rows_seed"], (70, 2, sch.ring.N))
    unit = opk.bias_unit(c["gamma"], sch.ring)
    assert digest(lin.encrypted_linear(W, bias, rows, unit)) == c["digest"]
    # edge cases: empty output, a single lane, wide weights
    assert lin.int_matmul_mod_q(np.zeros((0, 3), np.int64), rows[:3]).shape == (0, 2, sch.ring.N)
    w2 = np.random.default_rng(1).integers(-1000, 1000, (33, 17))
    r2 = u53(2, (17, 5))
    assert np.array_equal(lin.int_matmul_mod_q(w2, r2), olo.int_matmul_exact_objects(w2, r2))


@pytest.mark.parametrize("case", range(6))
def test_engine_toy_inference_matches_golden(golden, case):
    """Whole server rounds through the drop-in ServerEngine; same uploads -> same packs."""
    from paper_2509_01253_b200.engine import ServerEngine
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet
    from paper_2509_01253_b200.workloads import toy_model
    c = golden["inference"][case]
    sch = osc.preset(c["b"], c["gamma"])
    mys = _scheme(sch)
    toy = toy_model(c["b"], c["toy_seed"])
    client = opr.OracleClient(sch, seed=c["client_seed"])
    ksk = client.make_ksk()
    R, g = _ring(sch)
    server = ServerEngine(toy, mys, master_seed=bytes(range(32)))
    kid = server.register_client(KeySwitchKeySet(ksk.keys, g, ksk.delta, R))
    sid = client.new_session_id()
    assert sid.hex() == c["session_id"]
    server.open_session(sid, kid)
    x = np.random.default_rng(c["x_seed"]).integers(0, 4, toy.input_shape)
    log = []

    def srv(rno, bundles):
        pk, st = server.server_round(sid, rno, bundles)
        log.append((pk, st))
        return pk, st

    logits, _ = opr.run_rounds(client, srv, olo.build_rounds(toy.layers), x)
    assert logits.tolist() == c["logits"]
    for (pk, st), ref in zip(log, c["rounds"]):
        assert digest(np.stack(pk)) == ref["digest"]
        assert st.key_switches == ref["ks"]
        assert st.packed_coefficients == ref["packed"]


def test_engine_protocol_errors():
    from paper_2509_01253_b200.engine import ProtocolError, ServerEngine
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet
    from paper_2509_01253_b200.workloads import toy_model
    sch = osc.preset(8, 1)
    client = opr.OracleClient(sch, seed=5)
    ksk = client.make_ksk()
    R, g = _ring(sch)
    server = ServerEngine(toy_model(8, 3), _scheme(sch), master_seed=bytes(32))
    kid = server.register_client(KeySwitchKeySet(ksk.keys, g, ksk.delta, R))
    with pytest.raises(ProtocolError):
        server.server_round(b"\x01" * 16, 1, [])
    server.open_session(b"\x02" * 16, kid)
    with pytest.raises(ProtocolError):
        server.server_round(b"\x02" * 16, 2, [])
    with pytest.raises(ProtocolError):
        server.server_round(b"\x02" * 16, 1, [])
    with pytest.raises(ProtocolError):
        server.open_session(b"\x02" * 16, kid)
    partial = KeySwitchKeySet({d: ksk.keys[d] for d in list(ksk.keys)[:2]}, g, ksk.delta, R)
    with pytest.raises(ProtocolError):
        server.register_client(partial)
