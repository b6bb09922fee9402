"""B200-native Safhire server hot path (arxiv 2509.01253).

Drop-in for the reference's server-side engine (reference
pkg/src/sfhr/protocol.py:145-321): ``ServerEngine.server_round`` keeps its
signature, while partial extraction, the encrypted linear map, shuffling
and fast packing run as hand-written sm_100a kernels behind the C-ABI in
``include/sfhr_b200.h`` (``libsfhr_b200.so``).

Heavy modules (torch, the native library) load lazily on first use.
"""

from .params import (GadgetParams, Q, Q_BITS, Q_MASK, RingParams, SchemeParams,  # noqa: F401
                     preset_bits, preset_for_bits)

_LAZY = {
    "ServerEngine": "engine", "ProtocolError": "engine", "RoundStats": "engine",
    "required_ksk_indices": "engine", "ModelMetadata": "engine", "RoundMeta": "engine",
    "KeySwitchEngine": "keyswitch", "KeySwitchKeySet": "keyswitch", "RlweCiphertext": "keyswitch",
    "PowerBundle": "tracepack", "KsCounter": "tracepack", "partial_extract": "tracepack",
    "fast_pack": "tracepack", "pack_rows": "tracepack",
    "encrypted_linear": "linear", "int_matmul_mod_q": "linear",
    "derive_permutation": "_native", "invert_permutation": "_native",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)
