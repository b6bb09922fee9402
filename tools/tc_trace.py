"""Timeline of one tensor-core forward launch (CTA 0), from SFHR_TC_TRACE=1 stderr lines.

    SFHR_TC_TRACE=1 python tools/tc_trace.py   # runs a few stage launches and prints per-role timing
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from oracle import keyswitch as oks  # noqa: E402
from oracle import pack as opk  # noqa: E402
from oracle import protocol as opr  # noqa: E402
from oracle import scheme as osc  # noqa: E402

from paper_2509_01253_b200.keyswitch import KeySwitchEngine, KeySwitchKeySet  # noqa: E402
from paper_2509_01253_b200.params import GadgetParams, RingParams  # noqa: E402

gamma = int(os.environ.get("GAMMA", "0"))
B = int(os.environ.get("ROWS", "2048"))
sch = osc.preset(12, gamma)
R = sch.ring
rng = np.random.default_rng(0)
keys = {d: [oks.Ct(rng.integers(0, 1 << 53, R.N, dtype=np.uint64), rng.integers(0, 1 << 53, R.N, dtype=np.uint64))
            for _ in range(sch.gadget.l)] for d in opr.required_ksk_indices(sch)}
eng = KeySwitchEngine(KeySwitchKeySet(keys, GadgetParams(sch.gadget.D, sch.gadget.l), 0.0,
                                      RingParams(R.t, R.alpha, R.p_bits)), gamma=gamma)
x = torch.from_numpy(rng.integers(0, 1 << 53, (B, 2, R.N), dtype=np.uint64).view(np.int64)).cuda()
for reps in ([1, 3], opk.stage_reps_above(1, R)):
    eng.stage_batch(x, reps)
    torch.cuda.synchronize()
