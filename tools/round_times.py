import sys
sys.path.insert(0, ".")
import bench
from paper_2509_01253_b200.engine import ServerEngine
from paper_2509_01253_b200.keyswitch import KeySwitchKeySet
from paper_2509_01253_b200.params import preset_for_bits
sch = preset_for_bits(12, 0)
model = bench.make_model("resnet20", 12, 0)
eng = ServerEngine(model, sch, master_seed=bytes(32), device=0)
kid = eng.register_client(KeySwitchKeySet(bench.synthetic_ksk(sch, 0), sch.gadget, 0.0, sch.ring))
powers, exps = bench.synthetic_inputs(model, sch, 1000)
bundles = [bench.as_bundles(p, exps, 0) for p in powers]
for it in range(2):
    sid = bytes([5, it]) + bytes(14)
    eng.open_session(sid, kid)
    rows = []
    for r in range(1, len(model.rounds) + 1):
        _, st = eng.server_round(sid, r, bundles[r - 1])
        rnd = model.rounds[r - 1]
        rows.append((r, rnd.input_len, rnd.output_len, st.key_switches, st.extract_s * 1e3, st.linear_s * 1e3, st.pack_s * 1e3))
for r in rows:
    print("round %2d in %6d out %6d KS %6d  extract %.2f linear %.2f pack %.2f ms" % r)
