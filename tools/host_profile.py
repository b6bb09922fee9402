"""cProfile of the host side of server_round (e2e path) for a workload: where the per-round
host time goes between GPU launches.

    python tools/host_profile.py [mlp|resnet20] [iterations]
"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_01253_b200.engine import ServerEngine  # noqa: E402
from paper_2509_01253_b200.keyswitch import KeySwitchKeySet  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "mlp"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
b, gamma = bench.WORKLOADS[wl][1], bench.WORKLOADS[wl][2]
from paper_2509_01253_b200.params import preset_for_bits  # noqa: E402
sch = preset_for_bits(b, gamma)
model = bench.make_model(wl, b, 0)
eng = ServerEngine(model, sch, master_seed=bytes(32), device=0)
kid = eng.register_client(KeySwitchKeySet(bench.synthetic_ksk(sch, 0), sch.gadget, 0.0, sch.ring))
powers, exps = bench.synthetic_inputs(model, sch, 1000)
bundles = [bench.as_bundles(p, exps, gamma) for p in powers]


def one(i):
    sid = bytes([3, i % 256, i // 256]) + bytes(13)
    eng.open_session(sid, kid)
    for r in range(1, len(model.rounds) + 1):
        eng.server_round(sid, r, bundles[r - 1])


for i in range(5):
    one(i)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(iters):
    one(1000 + i)
torch.cuda.synchronize()
print(f"{wl}: {(time.perf_counter() - t0) / iters * 1e3:.3f} ms per inference (e2e)")
pr = cProfile.Profile()
pr.enable()
for i in range(iters):
    one(5000 + i)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
