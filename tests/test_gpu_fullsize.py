"""Full-size checks on the GPU: BASELINE workloads end to end.

* ResNet-20 stem round (3072 -> 16384 rows, 56 pack groups): packs and KS
  count bit-identical to the CPU oracle on the same uploads.
* pack-group sharding (multi-GPU partition) reproduces the single-range packs.
* whole inferences through the oracle client (real keys, encryption noise):
  decrypted logits equal the integer cleartext forward pass exactly
  (ResNet-20 shape b=12 gamma=0; MLP 784-128-10 b=16 gamma=0,1,2).
"""

import numpy as np
import pytest

from conftest import has_cuda
from oracle import keyswitch as oks
from oracle import lowering as olo
from oracle import pack as opk
from oracle import protocol as opr
from oracle import scheme as osc

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")]


def _mine(sch):
    from paper_2509_01253_b200.params import GadgetParams, RingParams, SchemeParams
    R = RingParams(sch.ring.t, sch.ring.alpha, sch.ring.p_bits)
    g = GadgetParams(sch.gadget.D, sch.gadget.l)
    return R, g, SchemeParams(R, sch.delta, g, sch.gamma, sch.beta)


def _uniform_keys(sch, seed):
    rng = np.random.default_rng(seed)
    R = sch.ring
    return {d: [oks.Ct(rng.integers(0, 1 << 53, R.N, dtype=np.uint64),
                       rng.integers(0, 1 << 53, R.N, dtype=np.uint64)) for _ in range(sch.gadget.l)]
            for d in opr.required_ksk_indices(sch)}


@pytest.mark.parametrize("gamma", [1])
def test_resnet20_stem_round_matches_oracle(gamma):
    from paper_2509_01253_b200.engine import ServerEngine
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet
    from paper_2509_01253_b200.workloads import resnet20_model
    sch = osc.preset(12, gamma)
    R, g, mys = _mine(sch)
    model = resnet20_model(12, seed=0)
    keys = _uniform_keys(sch, 5)
    sid = bytes(range(100, 116))
    eng = ServerEngine(model, mys, master_seed=bytes(range(32)))
    kid = eng.register_client(KeySwitchKeySet(keys, g, 0.0, R))
    eng.open_session(sid, kid)
    rnd = model.rounds[0]
    exps = opk.power_exponents(gamma, sch.ring)
    k = -(-rnd.input_len // R.N)
    power = np.random.default_rng(9).integers(0, 1 << 53, (k, len(exps), 2, R.N), dtype=np.uint64)
    from paper_2509_01253_b200.keyswitch import RlweCiphertext
    from paper_2509_01253_b200.tracepack import PowerBundle
    bundles = [PowerBundle(gamma, {d: RlweCiphertext(power[j, q, 0], power[j, q, 1])
                                   for q, d in enumerate(exps)}) for j in range(k)]
    packs, st = eng.server_round(sid, 1, bundles)
    # oracle: same uploads, same sigma, stem round matrix = its layer matrix
    orounds = olo.build_rounds(model.layers)
    W, bias = olo.layer_matrix(model.layers[orounds[0].layers[0]])
    srv = opr.OracleServer(model, sch, oks.KskSet(keys, sch.gadget, 0.0, sch.ring),
                           master_seed=bytes(range(32)), session_id=sid, ks_mode="fft",
                           round_mats=[(W, bias)] + [None] * (len(orounds) - 1), threads=8)
    obund = [opk.Bundle(gamma, {d: oks.Ct(power[j, q, 0], power[j, q, 1]) for q, d in enumerate(exps)})
             for j in range(k)]
    opacks, ost = srv.server_round(1, obund)
    assert len(packs) == len(opacks) == 56
    assert np.array_equal(np.stack(packs), np.stack(opacks))
    assert st.key_switches == ost.key_switches


def test_sharded_pack_ranges_reassemble():
    import torch
    from paper_2509_01253_b200.distributed import group_range
    from paper_2509_01253_b200.engine import ServerEngine
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet
    from paper_2509_01253_b200.workloads import resnet20_model
    sch = osc.preset(12, 2)
    R, g, mys = _mine(sch)
    model = resnet20_model(12, seed=1)
    eng = ServerEngine(model, mys, master_seed=bytes(32))
    kid = eng.register_client(KeySwitchKeySet(_uniform_keys(sch, 6), g, 0.0, R))
    sid = bytes(16)
    eng.open_session(sid, kid)
    st = eng.sessions[sid]
    exps = opk.power_exponents(2, sch.ring)
    rnd = model.rounds[0]
    k = -(-rnd.input_len // R.N)
    power = torch.from_numpy(np.random.default_rng(3).integers(
        0, 1 << 53, (k, len(exps), 2, R.N), dtype=np.uint64).view(np.int64)).cuda()
    im, om = eng.round_maps(st, sid, 1)
    im, om = torch.from_numpy(im).cuda(), torch.from_numpy(om).cuda()
    key = eng.clients[kid].key
    full, nks, _ = eng.round_device(1, key, power, exps, im, om)
    G = full.shape[0]
    for world in (2, 3, 8):
        parts, tot = [], 0
        for r in range(world):
            part, n, _ = eng.round_device(1, key, power, exps, im, om, groups=group_range(G, r, world))
            parts.append(part)
            tot += n
        assert torch.equal(torch.cat(parts), full)
        assert tot == nks


def _client_inference(model, b, gamma, seed, x):
    from paper_2509_01253_b200.engine import ServerEngine
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet
    sch = osc.preset(b, gamma)
    R, g, mys = _mine(sch)
    client = opr.OracleClient(sch, seed=seed)
    ksk = client.make_ksk()
    server = ServerEngine(model, mys, master_seed=bytes(range(32)))
    kid = server.register_client(KeySwitchKeySet(ksk.keys, g, ksk.delta, R))
    sid = client.new_session_id()
    server.open_session(sid, kid)
    logits, stats = opr.run_rounds(client, lambda rno, bd: server.server_round(sid, rno, bd),
                                   olo.build_rounds(model.layers), x)
    return logits, stats


def test_resnet20_exact_logits_end_to_end():
    from paper_2509_01253_b200.workloads import image_input, resnet20_model
    model = resnet20_model(12, seed=0)
    x = image_input(model, seed=4)
    logits, stats = _client_inference(model, 12, 0, 77, x)
    assert logits.tolist() == olo.cleartext_forward(model, x).tolist()
    assert sum(s.key_switches for s in stats) > 700_000


@pytest.mark.parametrize("gamma", [0, 1, 2])
def test_mlp_exact_logits_end_to_end(gamma):
    from paper_2509_01253_b200.workloads import mlp_input, mlp_model
    model = mlp_model(0)
    x = mlp_input(0)
    logits, _ = _client_inference(model, 16, gamma, 1, x)
    assert logits.tolist() == olo.cleartext_forward(model, x).tolist()


def test_distributed_engine_matches_server_round():
    """DistributedServerEngine (NCCL, one rank) == ServerEngine.server_round on the same
    uploads, with the same protocol checks, session state and extra noise."""
    import os
    import socket

    import torch.distributed as dist
    from paper_2509_01253_b200.distributed import DistributedServerEngine
    from paper_2509_01253_b200.engine import ERR_STALE_ROUND, ProtocolError, ServerEngine
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet, RlweCiphertext
    from paper_2509_01253_b200.tracepack import PowerBundle
    from paper_2509_01253_b200.workloads import mlp_model
    sch = osc.preset(16, 1)
    R, g, mys = _mine(sch)
    model = mlp_model(0)
    keys = _uniform_keys(sch, 8)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        engs = [ServerEngine(model, mys, master_seed=bytes(range(32)), extra_noise_std=2.0 ** -40)
                for _ in range(2)]
        kids = [e.register_client(KeySwitchKeySet(keys, g, 0.0, R)) for e in engs]
        sid = bytes(range(16))
        for e, kid in zip(engs, kids):
            e.open_session(sid, kid)
        de = DistributedServerEngine(engs[1])
        exps = opk.power_exponents(1, sch.ring)
        rng = np.random.default_rng(21)
        with pytest.raises(ProtocolError) as ei:
            de.server_round(sid, 2, [])
        assert ei.value.code == ERR_STALE_ROUND
        for rno, rnd in enumerate(model.rounds, start=1):
            k = -(-rnd.input_len // R.N)
            power = rng.integers(0, 1 << 53, (k, len(exps), 2, R.N), dtype=np.uint64)
            bundles = [PowerBundle(1, {d: RlweCiphertext(power[j, q, 0], power[j, q, 1])
                                       for q, d in enumerate(exps)}) for j in range(k)]
            want, st_w = engs[0].server_round(sid, rno, bundles)
            got, st_g = de.server_round(sid, rno, bundles)
            assert np.array_equal(np.stack(got), np.stack(want))
            assert st_g.key_switches == st_w.key_switches
        assert sid not in engs[1].sessions
        assert engs[1].total_key_switches == engs[0].total_key_switches
    finally:
        dist.destroy_process_group()
