"""Ciphertext-block wire codec: oracle pinned to the reference's own payloads
(tests/golden/golden_wire.json), device codec byte-identical to both."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import has_cuda, u53
from oracle import scheme as osc
from oracle import wire as ow

GW = json.loads((Path(__file__).parent / "golden" / "golden_wire.json").read_text())["cases"]


def _case(c):
    sch = osc.preset(c["b"], c["gamma"])
    R = sch.ring
    power = u53(c["seed"], (c["k"], len(c["exps"]), 2, R.N))
    packs = u53(c["seed"] + 1, (c["n_packs"], 2, R.N))
    return sch, R, power, packs


@pytest.mark.parametrize("i", range(len(GW)))
def test_oracle_wire_matches_reference_payloads(i):
    c = GW[i]
    sch, R, power, packs = _case(c)
    req = ow.encode_round_req(power, c["exps"], R.M, c["gamma"])
    assert len(req) == c["req_len"] and hashlib.sha256(req).hexdigest() == c["req_sha256"]
    resp = ow.encode_round_resp(packs, R.M, c["gamma"])
    assert len(resp) == c["resp_len"] and hashlib.sha256(resp).hexdigest() == c["resp_sha256"]
    got, exps, gammas = ow.decode_round_req(req, R.N)
    assert np.array_equal(got, power) and exps == [c["exps"]] * c["k"] and gammas == [c["gamma"]] * c["k"]
    assert np.array_equal(ow.decode_round_resp(resp, R.N), packs)
    bad = bytearray(req)
    off = c["bad_lane_offset"]
    bad[off:off + 8] = (1 << 53).to_bytes(8, "little")
    with pytest.raises(ow.WireError) as e:
        ow.decode_round_req(bytes(bad), R.N)
    assert e.value.reason == c["bad_lane_error"]
    with pytest.raises(ow.WireError) as e:
        ow.decode_round_req(req[:-3], R.N)
    assert e.value.reason == c["truncated_error"]


@pytest.mark.parametrize("i", range(len(GW)))
def test_host_header_parse(i):
    from paper_2509_01253_b200.wire import WireError, parse_round_req
    c = GW[i]
    sch, R, power, packs = _case(c)
    req = ow.encode_round_req(power, c["exps"], R.M, c["gamma"])
    k, exps, m, gammas, offs = parse_round_req(req, R.N)
    assert (k, exps, m, gammas) == (c["k"], c["exps"], R.M, [c["gamma"]] * c["k"])
    per = 4 + 4 * len(c["exps"]) + ow.block_size(R.M, len(c["exps"]))
    assert offs == [4 + j * per + 4 + 4 * len(c["exps"]) + 8 for j in range(k)]
    for cut in (2, 10, len(req) - 3):
        with pytest.raises(WireError):
            parse_round_req(req[:cut], R.N)


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("i", range(len(GW)))
def test_device_codec_matches_reference(i):
    import torch
    from paper_2509_01253_b200.wire import WireError, decode_round_req_device, encode_round_resp_device
    c = GW[i]
    sch, R, power, packs = _case(c)
    req = ow.encode_round_req(power, c["exps"], R.M, c["gamma"])
    got, exps, gammas = decode_round_req_device(req, R.N, "cuda:0")
    assert np.array_equal(got.cpu().numpy().view(np.uint64), power)
    resp = encode_round_resp_device(torch.from_numpy(packs.view(np.int64)).cuda(), R.M, c["gamma"])
    assert hashlib.sha256(resp).hexdigest() == c["resp_sha256"]
    bad = bytearray(req)
    off = c["bad_lane_offset"]
    bad[off:off + 8] = (1 << 53).to_bytes(8, "little")
    with pytest.raises(WireError) as e:
        decode_round_req_device(bytes(bad), R.N, "cuda:0")
    assert e.value.reason == c["bad_lane_error"]
    # a bad lane in the LAST chunk's padding (byte-misaligned block)
    bad = bytearray(req)
    per = 4 + 4 * len(c["exps"]) + ow.block_size(R.M, len(c["exps"]))
    off_last = 4 + (c["k"] - 1) * per + 4 + 4 * len(c["exps"]) + 8 + 8 * (2 * R.M * len(c["exps"]) - 1)
    bad[off_last:off_last + 8] = (1 << 60).to_bytes(8, "little")
    with pytest.raises(WireError):
        decode_round_req_device(bytes(bad), R.N, "cuda:0")


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("b,gamma", [(12, 1), (16, 0)])
def test_wire_inference_exact_logits(b, gamma):
    """A whole toy inference through ServerEngine.server_round_wire (payload bytes in and
    out, reference encoding on the client side) gives the cleartext logits exactly, and
    each response equals the reference encoding of the plain server_round output."""
    from oracle import lowering as olo
    from oracle import protocol as opr
    from paper_2509_01253_b200.engine import ServerEngine
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet
    from paper_2509_01253_b200.params import GadgetParams, RingParams, SchemeParams
    from paper_2509_01253_b200.workloads import toy_model
    sch = osc.preset(b, gamma)
    R0 = sch.ring
    R = RingParams(R0.t, R0.alpha, R0.p_bits)
    g = GadgetParams(sch.gadget.D, sch.gadget.l)
    mys = SchemeParams(R, sch.delta, g, gamma, sch.beta)
    model = toy_model(b, 5)
    client = opr.OracleClient(sch, seed=21)
    ksk = client.make_ksk()
    servers = [ServerEngine(model, mys, master_seed=bytes(range(32))) for _ in range(2)]
    sid = client.new_session_id()
    for srv in servers:
        srv.open_session(sid, srv.register_client(KeySwitchKeySet(ksk.keys, g, ksk.delta, R)))

    def round_fn(rno, bundles):
        exps = sorted(bundles[0].power_cts)
        power = np.stack([np.stack([np.stack([bd.power_cts[d].a, bd.power_cts[d].b]) for d in exps])
                          for bd in bundles])
        resp, st = servers[0].server_round_wire(sid, rno, ow.encode_round_req(power, exps, R.M, gamma))
        packed, st2 = servers[1].server_round(sid, rno, bundles)
        assert resp == ow.encode_round_resp(np.stack(packed), R.M, gamma)
        assert st.key_switches == st2.key_switches and st.bytes_down == st2.bytes_down
        got = ow.decode_round_resp(resp, R.N)
        return [got[i] for i in range(got.shape[0])], st

    x = np.random.default_rng(9).integers(0, 4, model.input_shape)
    logits, _ = opr.run_rounds(client, round_fn, olo.build_rounds(model.layers), x)
    assert logits.tolist() == olo.cleartext_forward(model, x).tolist()
