"""Golden fixtures for the ciphertext-block wire codec, from the REAL reference.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_wire.py

Writes tests/golden/golden_wire.json: seeds/shapes plus sha256 digests of the
reference's encode_round_req / encode_round_resp payloads (wire.py:99-124,
208-254) and the messages of its decode errors.  Build container only.
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from sfhr import wire
from sfhr.crypto import RlweCiphertext
from sfhr.params import preset_for_bits
from sfhr.tracepack import PowerBundle, power_exponents

OUT = Path(__file__).with_name("golden_wire.json")


def u53(seed, shape):
    return np.random.default_rng(seed).integers(0, 1 << 53, shape, dtype=np.uint64)


def main():
    cases = []
    for b, gamma, k, n_packs in [(8, 0, 2, 3), (12, 0, 3, 5), (12, 1, 2, 1), (16, 1, 2, 4), (16, 2, 1, 0)]:
        sch = preset_for_bits(b, gamma)
        R = sch.ring
        exps = sorted(power_exponents(gamma, R))
        seed = 1000 * b + 10 * gamma + k
        power = u53(seed, (k, len(exps), 2, R.N))
        bundles = [PowerBundle(gamma=gamma, power_cts={d: RlweCiphertext(a=power[j, q, 0], b=power[j, q, 1])
                                                       for q, d in enumerate(exps)}) for j in range(k)]
        req = wire.encode_round_req(bundles, R.M)
        assert len(wire.encode(wire.WireMessage(wire.ROUND_REQ, bytes(16), 1, req))) == \
            wire.round_req_size(sch, k)
        packs = u53(seed + 1, (n_packs, 2, R.N))
        resp = wire.encode_round_resp([packs[i] for i in range(n_packs)], R.M, gamma)
        assert len(wire.encode(wire.WireMessage(wire.ROUND_RESP, bytes(16), 1, resp))) == \
            wire.round_resp_size(sch, n_packs)
        # decode of a corrupted request: one padding lane set to 2^53
        bad = bytearray(req)
        off = 4 + 4 + 4 * len(exps) + 8 + 8 * R.N  # first chunk, first power, a component, lane N
        bad[off:off + 8] = (1 << 53).to_bytes(8, "little")
        try:
            wire.decode_round_req(bytes(bad), R.N)
            err = None
        except wire.WireError as e:
            err = e.reason
        try:
            wire.decode_round_req(req[:-3], R.N)
            trunc = None
        except (wire.WireError, Exception) as e:  # noqa: BLE001
            trunc = getattr(e, "reason", type(e).__name__)
        cases.append({"b": b, "gamma": gamma, "k": k, "n_packs": n_packs, "seed": seed, "exps": exps,
                      "req_len": len(req), "req_sha256": hashlib.sha256(req).hexdigest(),
                      "resp_len": len(resp), "resp_sha256": hashlib.sha256(resp).hexdigest(),
                      "bad_lane_offset": off, "bad_lane_error": err, "truncated_error": trunc})
    OUT.write_text(json.dumps({"cases": cases}, indent=1))
    print(OUT, len(cases))


if __name__ == "__main__":
    main()
