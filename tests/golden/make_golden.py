"""Generate golden fixtures by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes tests/golden/golden.json: for each case, the seeds/shapes needed to
regenerate the inputs with numpy, plus sha256 digests (and small slices) of
the reference's outputs.  The CPU tests pin oracle/ against these; the GPU
tests pin the CUDA path against both.  /root/reference is read here only;
nothing at test time on the GPU box touches it.

Reference entry points exercised (pkg/src/sfhr/...):
  crypto.gadget_decompose            crypto.py:288
  crypto.KeySwitchEngine (exact/fft)  crypto.py:360-474
  protocol.Client.make_ksk / prepare_round       protocol.py:336-373
  tracepack.partial_extract / fast_pack / pack_rows  tracepack.py:118-348
  model.int_matmul_mod_q / encrypted_linear       model.py:384-429
  confidentiality.derive_permutation            confidentiality.py:57-76
  protocol.ServerEngine.server_round (toy model) protocol.py:219-280
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

from sfhr import crypto, model as mm, tracepack
from sfhr.confidentiality import derive_permutation
from sfhr.dual import dual_basis
from sfhr.params import GadgetParams, RingParams, SchemeParams, preset_for_bits
from sfhr.protocol import Client, ServerEngine, required_ksk_indices, run_inference
from sfhr.testing import make_random_toy_model

OUT = Path(__file__).with_name("golden.json")


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a))
    if a.dtype.kind in "iu":
        a = a.astype("<u8") if a.dtype.kind == "u" else a.astype("<i8")
    return hashlib.sha256(a.tobytes()).hexdigest()


def u53(seed, shape):
    return np.random.default_rng(seed).integers(0, 1 << 53, shape, dtype=np.uint64)


def ksk_digest(ksk):
    parts = []
    for d in ksk.indices():
        for ct in ksk.keys[d]:
            parts.append(ct.a)
            parts.append(ct.b)
    return digest(np.stack(parts))


def main():
    g: dict = {"meta": {"numpy": np.__version__, "generated_by": "tests/golden/make_golden.py"}}
    t0 = time.time()

    # 1. gadget digits
    cases = []
    for D, l in [(512, 3), (4096, 3), (1 << 16, 2), (310, 5), (310, 4)]:
        v = u53(7, 4096)
        v[:4] = [0, (1 << 53) - 1, 1 << 52, (1 << 53) // D]
        dg = crypto.gadget_decompose(v, GadgetParams(D, l))
        cases.append({"D": D, "l": l, "seed": 7, "n": 4096,
                      "head": [0, (1 << 53) - 1, 1 << 52, (1 << 53) // D],
                      "digest": digest(dg), "first_cols": dg[:, :4].tolist()})
    g["gadget"] = cases

    # 2. per preset row: client keys, key switches, extraction, one pack group
    rows = []
    for b in (8, 12, 16):
        for gamma in (0, 1, 2):
            scheme = preset_for_bits(b, gamma)
            P = scheme.ring
            cseed = 500 + 10 * b + gamma
            client = Client(scheme, seed=cseed)
            ksk = client.make_ksk()
            idx = required_ksk_indices(scheme)
            rec = {"b": b, "gamma": gamma, "client_seed": cseed, "indices": idx,
                   "ksk_digest": ksk_digest(ksk), "sk_digest": digest(client.sk.s.astype(np.int64))}
            # key switch: 3 uniform cts through two indices, exact and fft
            x = u53(1000 + b + gamma, (3, 2, P.N))
            eng_x = crypto.KeySwitchEngine(ksk, mode="exact")
            eng_f = crypto.KeySwitchEngine(ksk, mode="fft")
            ks = []
            for d in (idx[0], idx[-1]):
                moved = eng_x.automorphism_batch(x, d)
                out_x = eng_x.switch_batch(moved, d)
                out_f = eng_f.switch_batch(moved, d)
                ks.append({"d": d, "aut_digest": digest(moved), "exact_digest": digest(out_x),
                           "fft_digest": digest(out_f), "fft_equals_exact": bool(np.array_equal(out_x, out_f))})
            rec["ks_input_seed"] = 1000 + b + gamma
            rec["ks"] = ks
            # extraction of one client bundle (message seeded)
            mrng = np.random.default_rng(2000 + b + gamma)
            v = mrng.integers(-3, 4, P.N)
            bundles = client.prepare_round(v, P.N)
            bundle = bundles[0]
            exps = sorted(bundle.power_cts)
            power_cts = np.stack([np.stack([bundle.power_cts[d].a, bundle.power_cts[d].b]) for d in exps])
            dual = dual_basis(P)
            ext = tracepack.partial_extract(bundle, dual, P.N, P)
            ext_part = tracepack.partial_extract(bundle, dual, 37, P)
            rec["extract"] = {"msg_seed": 2000 + b + gamma, "power_digest": digest(power_cts),
                              "exps": exps, "rows_digest": digest(ext), "rows37_digest": digest(ext_part)}
            unit = tracepack.extraction_payload_for_one(dual, gamma, P)
            rec["bias_unit_digest"] = digest(unit)
            # one pack group of uniform rows; a second with a zero tail (skip_zero counting)
            F = scheme.pack_factor
            grp = u53(3000 + b + gamma, (F, 2, P.N))
            cnt = tracepack.KsCounter()
            pk = tracepack.fast_pack(grp, scheme, eng_f, counter=cnt, skip_zero=True)
            grp2 = grp.copy()
            grp2[F // 3:] = 0
            cnt2 = tracepack.KsCounter()
            pk2 = tracepack.pack_rows(grp2[:F // 3 + 1], scheme, eng_f, counter=cnt2)
            rec["pack"] = {"seed": 3000 + b + gamma, "F": F, "digest": digest(pk),
                           "ks": cnt.total_key_switches, "tail_digest": digest(np.stack(pk2)),
                           "tail_rows": F // 3 + 1, "tail_ks": cnt2.total_key_switches}
            rows.append(rec)
            print(f"row b={b} gamma={gamma} done at {time.time() - t0:.1f}s", file=sys.stderr)
    g["rows"] = rows

    # 3. small ring M=27 (reference tests' ring) key switch + pack
    P27 = RingParams(t=3, alpha=3, p_bits=8)
    small = []
    for gamma in (0, 1, 2):
        sch = SchemeParams(ring=P27, delta=2.0 ** -36, gadget=GadgetParams(512, 3), gamma=gamma)
        dual = dual_basis(P27)
        sk = crypto.keygen(P27, seed=31)
        rng = np.random.default_rng(32)
        idx = required_ksk_indices(SchemeParams(ring=P27, delta=2.0 ** -36,
                                                gadget=GadgetParams(512, 3), gamma=0))
        ksk = crypto.keygen_ksk(sk, idx, sch.gadget, sch.delta, rng, dual)
        eng = crypto.KeySwitchEngine(ksk, mode="exact")
        grp = u53(4000 + gamma, (sch.pack_factor, 2, P27.N))
        cnt = tracepack.KsCounter()
        pk = tracepack.fast_pack(grp, sch, eng, counter=cnt)
        small.append({"gamma": gamma, "indices": idx, "ksk_digest": ksk_digest(ksk),
                      "seed": 4000 + gamma, "digest": digest(pk), "ks": cnt.total_key_switches,
                      "packed": pk.tolist()})
    g["m27"] = small

    # 4. encrypted linear
    w = np.random.default_rng(43).integers(-7, 8, (5, 9))
    rws = u53(44, (9, 2, 11))
    g["int_matmul"] = {"w_seed": 43, "rows_seed": 44, "digest": digest(mm.int_matmul_mod_q(w, rws))}
    P = preset_for_bits(12, 1).ring
    W = np.random.default_rng(45).integers(-3, 4, (40, 70))
    bias = np.random.default_rng(46).integers(-9, 10, 40)
    rws = u53(47, (70, 2, P.N))
    unit = tracepack.extraction_payload_for_one(dual_basis(P), 1, P)
    g["enc_linear"] = {"b": 12, "gamma": 1, "w_seed": 45, "bias_seed": 46, "rows_seed": 47,
                       "digest": digest(mm.encrypted_linear(W, bias, rws, unit))}

    # 5. permutations
    perms = []
    for size, rno in [(1, 1), (2, 1), (17, 3), (1000, 2), (5000, 7)]:
        pm = derive_permutation(bytes(range(32)), bytes(range(16, 32)), rno, size)
        perms.append({"size": size, "round": rno, "digest": digest(pm), "head": pm[:16].tolist()})
    g["perms"] = perms

    # 6. whole server rounds on the random toy model (reference make_random_toy_model)
    infer = []
    for b, gamma in [(8, 0), (8, 1), (12, 1), (16, 2), (12, 0), (16, 0)]:
        scheme = preset_for_bits(b, gamma)
        toy = make_random_toy_model(b, seed=3)
        server = ServerEngine(toy, scheme, master_seed=bytes(range(32)), ks_mode="fft")
        client = Client(scheme, seed=11 + b + gamma)
        key_id = server.register_client(client.make_ksk())
        x = np.random.default_rng(7).integers(0, 4, toy.input_shape)
        # capture per-round packs by wrapping server_round
        packs_log = []
        orig = server.server_round

        def wrapped(sid, rno, bundles, _orig=orig):
            pk, st = _orig(sid, rno, bundles)
            packs_log.append({"round": rno, "n": len(pk), "digest": digest(np.stack(pk)),
                              "ks": st.key_switches, "packed": st.packed_coefficients,
                              "bundle_digest": digest(np.stack([np.stack([np.stack([bd.power_cts[d].a, bd.power_cts[d].b]) for d in sorted(bd.power_cts)]) for bd in bundles]))})
            return pk, st

        server.server_round = wrapped
        res = run_inference(client, server, x, key_id=key_id)
        infer.append({"b": b, "gamma": gamma, "toy_seed": 3, "client_seed": 11 + b + gamma,
                      "x_seed": 7, "logits": res.logits.tolist(),
                      "cleartext": mm.cleartext_forward(toy, x).tolist(),
                      "session_id": res.session_id.hex(), "rounds": packs_log})
        print(f"inference b={b} gamma={gamma} done at {time.time() - t0:.1f}s", file=sys.stderr)
    g["inference"] = infer

    OUT.write_text(json.dumps(g, indent=1, sort_keys=True) + "\n")
    print(f"wrote {OUT} in {time.time() - t0:.1f}s", file=sys.stderr)


if __name__ == "__main__":
    main()
