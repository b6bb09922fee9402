"""Where does the e2e (host API) time of one ResNet-20 server inference go?"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_01253_b200.engine import ServerEngine  # noqa: E402
from paper_2509_01253_b200.keyswitch import KeySwitchKeySet  # noqa: E402
from paper_2509_01253_b200.params import preset_for_bits  # noqa: E402
from paper_2509_01253_b200.device import to_host_u64  # noqa: E402

import os
GAMMA = int(os.environ.get("GAMMA", "0"))
sch = preset_for_bits(12, GAMMA)
model = bench.make_model("resnet20", 12, 0)
eng = ServerEngine(model, sch, master_seed=bytes(32), device=0)
keys = bench.synthetic_ksk(sch, 0)
kid = eng.register_client(KeySwitchKeySet(keys, sch.gadget, 0.0, sch.ring))
powers, exps = bench.synthetic_inputs(model, sch, 1000)
bundles = [bench.as_bundles(p, exps, GAMMA) for p in powers]
acc = {}


def tick(name, t0):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    acc[name] = acc.get(name, 0.0) + (t1 - t0)
    return t1


for it in range(4):
    sid = bytes([9, it]) + bytes(14)
    t0 = time.perf_counter()
    eng.open_session(sid, kid)
    t0 = tick("open_session", t0) if it else time.perf_counter()
    st = eng.sessions[sid]
    for r in range(1, len(model.rounds) + 1):
        state = eng._check_round(sid, r, len(bundles[r - 1]))
        power, ex = eng._upload_bundles(bundles[r - 1])
        t0 = tick("upload", t0)
        in_map, out_map = eng.round_maps(state, sid, r)
        im = torch.from_numpy(in_map).to(eng.dev, non_blocking=True)
        om = None if out_map is None else torch.from_numpy(out_map).to(eng.dev, non_blocking=True)
        t0 = tick("maps", t0)
        packs, nks, times = eng.round_device(r, eng.clients[state.key_id].key, power, ex, im, om, timed=False)
        t0 = tick("device", t0)
        h = to_host_u64(packs)
        t0 = tick("d2h", t0)
        state.next_round += 1
    if it == 0:
        acc.clear()
tot = sum(acc.values())
print({k: round(v / 3 * 1e3, 2) for k, v in acc.items()}, "total ms", round(tot / 3 * 1e3, 2))
