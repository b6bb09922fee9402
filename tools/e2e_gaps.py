"""GPU idle gaps between the rounds of one e2e ResNet-20 inference through server_round:
CUDA events recorded right before each round's first launch and after its last one."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_01253_b200 import engine as E  # noqa: E402
from paper_2509_01253_b200.keyswitch import KeySwitchKeySet  # noqa: E402
from paper_2509_01253_b200.params import preset_for_bits  # noqa: E402

sch = preset_for_bits(12, 0)
model = bench.make_model("resnet20", 12, 0)
eng = E.ServerEngine(model, sch, master_seed=bytes(32), device=0)
keys = bench.synthetic_ksk(sch, 0)
kid = eng.register_client(KeySwitchKeySet(keys, sch.gadget, 0.0, sch.ring))
powers, exps = bench.synthetic_inputs(model, sch, 1000)
bundles = [bench.as_bundles(p, exps, 0) for p in powers]
marks = []
orig_extract, orig_pack = E.extract_device, E.pack_device


def extract(*a, **k):
    ev = torch.cuda.Event(enable_timing=True)
    ev.record()
    marks.append(("start", ev))
    return orig_extract(*a, **k)


def pack(*a, **k):
    out = orig_pack(*a, **k)
    ev = torch.cuda.Event(enable_timing=True)
    ev.record()
    marks.append(("end", ev))
    return out


E.extract_device, E.pack_device = extract, pack
for it in range(3):
    marks.clear()
    sid = bytes([7, it]) + bytes(14)
    eng.open_session(sid, kid)
    for r in range(1, len(model.rounds) + 1):
        eng.server_round(sid, r, bundles[r - 1])
    torch.cuda.synchronize()
busy = sum(marks[i][1].elapsed_time(marks[i + 1][1]) for i in range(0, len(marks), 2))
gaps = [marks[i][1].elapsed_time(marks[i + 1][1]) for i in range(1, len(marks) - 1, 2)]
print(f"device busy {busy:.2f} ms, gaps between rounds {sum(gaps):.2f} ms "
      f"(max {max(gaps):.3f}, mean {sum(gaps) / len(gaps):.3f})")

# host-side split of one round trip (perf_counter): before the first launch / after the sync
import time  # noqa: E402
T = {"pre": 0.0, "post": 0.0}
orig_up = eng._upload_bundles


def up(*a, **k):
    T["t_up0"] = time.perf_counter()
    return orig_up(*a, **k)


def extract2(*a, **k):
    T["pre"] += time.perf_counter() - T["t_round0"]
    return orig_extract(*a, **k)


eng._upload_bundles = up
E.extract_device = extract2
E.pack_device = orig_pack
sid = bytes([7, 9]) + bytes(14)
eng.open_session(sid, kid)
for r in range(1, len(model.rounds) + 1):
    T["t_round0"] = time.perf_counter()
    eng.server_round(sid, r, bundles[r - 1])
print(f"host time before the first launch of a round: {T['pre'] / len(model.rounds) * 1e3:.3f} ms")
