"""Host-side ServerEngine logic on CPU (no GPU): the bundle validation rule shared by
server_round and server_round_wire, and the per-round permutation prefetch
(one round ahead, engine-wide cap, cancelled on reap / session end)."""

import threading
import time
from concurrent.futures import ThreadPoolExecutor
from types import SimpleNamespace

import numpy as np
import pytest

from paper_2509_01253_b200 import _native as nat
from paper_2509_01253_b200.engine import (ERR_MALFORMED, ProtocolError, ServerEngine, _SessionState)
from paper_2509_01253_b200.params import preset_for_bits
from paper_2509_01253_b200.tracepack import power_exponents


def _engine(gamma=1, rounds=None, workers=2):
    eng = object.__new__(ServerEngine)
    eng.scheme = preset_for_bits(12, gamma)
    mk = lambda i, o, final=False, skip_len=0, skip_source=-1: SimpleNamespace(
        input_len=i, output_len=o, skip_len=skip_len, skip_source=skip_source, final=final)
    eng.model = SimpleNamespace(rounds=rounds or [mk(50, 40), mk(40, 30), mk(70, 30, skip_len=40, skip_source=0),
                                                  mk(30, 10, True)])
    eng.master_seed = bytes(range(32))
    eng.shuffle_enabled = True
    eng.session_timeout = 300.0
    eng._lock = threading.RLock()
    eng.total_key_switches = 0
    eng.sessions = {}
    eng._perm_pool = ThreadPoolExecutor(max_workers=workers)
    eng._pending = []
    return eng


def test_bundle_gamma_and_exponent_rule():
    eng = _engine(gamma=1)
    R = eng.scheme.ring
    want = sorted(power_exponents(1, R))
    eng._check_bundle_exponents([1, 1], [want, want])
    with pytest.raises(ProtocolError) as ei:  # another extraction level, even if self-consistent
        eng._check_bundle_exponents([1, 2], [want, sorted(power_exponents(2, R))])
    assert ei.value.code == ERR_MALFORMED
    with pytest.raises(ValueError) as ve:
        eng._check_bundle_exponents([1], [want[:-1]])
    assert str(want) in str(ve.value)  # the message names the set actually required


def test_perm_prefetch_one_round_ahead_and_reuse():
    eng = _engine()
    sid = bytes(16)
    st = _SessionState(key_id=b"k")
    eng.sessions[sid] = st
    eng._prefetch_perms(st, sid, 1)
    assert set(st.perms) == set(eng._round_perm_keys(1))  # round 1 only, not the whole session
    in_map, out_map = eng.round_maps(st, sid, 1)
    assert np.array_equal(out_map, nat.derive_permutation(eng.master_seed, sid, 1, 40))
    eng._prefetch_perms(st, sid, 2)
    eng._finish_round(sid, st, 1, 5)
    # sigma_1 stays for round 2's unshuffle and round 3's residual skip; identity (0, 50) is dropped
    assert (1, 40) in st.perms and (0, 50) not in st.perms
    in2, _ = eng.round_maps(st, sid, 2)
    assert np.array_equal(in2, out_map)
    assert eng.total_key_switches == 5


def test_perm_prefetch_cap_and_cancel():
    eng = _engine(workers=1)
    eng.MAX_QUEUED_PERMS = 3
    gate = threading.Event()
    eng._perm_pool.submit(gate.wait)  # occupy the single worker
    sids = [bytes([i]) * 16 for i in range(4)]
    for sid in sids:
        st = _SessionState(key_id=b"k")
        eng.sessions[sid] = st
        eng._prefetch_perms(st, sid, 2)
    queued = sum(len(eng.sessions[s].perms) for s in sids)
    assert queued == 3  # engine-wide cap
    # reaping cancels the queued work of expired sessions
    for s in sids:
        eng.sessions[s].last_seen = time.monotonic() - 1e4
    futs = [f for s in sids for f in eng.sessions[s].perms.values()]
    eng._reap()
    assert not eng.sessions and all(f.cancelled() for f in futs)
    gate.set()
    # a round whose prefetch was skipped or cancelled derives its sigma lazily
    st = _SessionState(key_id=b"k")
    eng.sessions[sids[0]] = st
    _, om = eng.round_maps(st, sids[0], 2)
    assert np.array_equal(om, nat.derive_permutation(eng.master_seed, sids[0], 2, 30))
