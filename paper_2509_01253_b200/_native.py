"""ctypes binding of libsfhr_b200.so (C-ABI declared in include/sfhr_b200.h).

The shared library is built in-tree (``python -m paper_2509_01253_b200.build``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the compute modules raises.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

LIB_PATH = Path(os.environ.get("SFHR_LIB_PATH") or Path(__file__).resolve().parent / "libsfhr_b200.so")

SFHR_OK, SFHR_EINVAL, SFHR_EKEY, SFHR_ECUDA, SFHR_EMODEL, SFHR_ENOMEM = range(6)


class SfhrCudaError(RuntimeError):
    pass


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2509_01253_b200.build` "
            "(the CUDA path has no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    vp, i32, i64, u32, sz = C.c_void_p, C.c_int, C.c_int64, C.c_uint32, C.c_size_t
    sig = {
        "sfhr_ctx_create": (i32, [i32, i32, i32, i32, i32, i32, i32, i32, C.POINTER(vp)]),
        "sfhr_ctx_destroy": (i32, [vp]),
        "sfhr_ctx_info": (i32, [vp, C.POINTER(C.c_int64), i32]),
        "sfhr_ringconst_bytes": (sz, []),
        "sfhr_linear_desc_bytes": (sz, []),
        "sfhr_ctx_debug_tables": (i32, [vp, vp, sz, vp, sz]),
        "sfhr_ctx_dual": (i32, [vp, vp, vp, vp]),
        "sfhr_register_ksk": (i32, [vp, vp, i32, vp, vp, C.POINTER(vp)]),
        "sfhr_key_destroy": (i32, [vp]),
        "sfhr_automorphism_batch": (i32, [vp, u32, vp, vp, i64, vp]),
        "sfhr_keyswitch_batch": (i32, [vp, vp, u32, vp, vp, i64, i32, vp, vp]),
        "sfhr_stage_batch": (i32, [vp, vp, vp, i32, vp, vp, i64, i32, vp, vp]),
        "sfhr_extract": (i32, [vp, vp, vp, i32, i32, i64, vp, vp]),
        "sfhr_linear_pass": (i32, [vp, vp, vp]),
        "sfhr_pack_workspace_bytes": (sz, [vp, i64]),
        "sfhr_pack": (i32, [vp, vp, vp, i64, vp, vp, sz, i32, vp, vp]),
        "sfhr_derive_permutation": (i32, [vp, i32, vp, i32, u32, i64, vp]),
        "sfhr_last_error": (C.c_char_p, []),
        "sfhr_mma_b_resident_bytes": (sz, []),
        "sfhr_tc_table_bytes": (sz, [vp]),
        "sfhr_ctx_tc_tables": (i32, [vp, vp, sz, vp]),
        "sfhr_ctx_tc_enabled": (i32, [vp]),
        "sfhr_ctx_set_tc": (i32, [vp, i32]),
        "sfhr_launch_count": (C.c_ulonglong, []),
        "sfhr_profile_enable": (i32, [vp, i32]),
        "sfhr_profile_collect": (i32, [vp, C.POINTER(C.c_double), C.POINTER(C.c_longlong),
                                       C.POINTER(C.c_longlong)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def launch_count() -> int:
    return int(lib.sfhr_launch_count())


def profile_collect(ctx_handle) -> tuple[float, int, int]:
    ms, by, n = C.c_double(), C.c_longlong(), C.c_longlong()
    check(lib.sfhr_profile_collect(ctx_handle, C.byref(ms), C.byref(by), C.byref(n)))
    return ms.value, by.value, n.value


def last_error() -> str:
    msg = lib.sfhr_last_error()
    return msg.decode() if msg else ""


def check(code: int, what: str = "") -> None:
    if code == SFHR_OK:
        return
    msg = last_error() or what
    if code == SFHR_EINVAL:
        raise ValueError(msg)
    if code == SFHR_EKEY:
        raise KeyError(msg)
    if code == SFHR_EMODEL:
        from .model import ModelError
        raise ModelError(msg)
    raise SfhrCudaError(msg)


class LinearDesc(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("in_", "in_map", "round_in", "round_map", "out", "out_map",
                                         "groups")] + \
               [("n_groups", C.c_int64)] + \
               [(n, C.c_void_p) for n in ("cols", "weights", "rows", "ex_ptr", "ex_col", "ex_w",
                                         "bias", "unit")] + \
               [("lanes", C.c_int64), ("body_off", C.c_int64)] + \
               [("mma_tiles", C.c_void_p), ("n_mma_tiles", C.c_int64)] + \
               [(n, C.c_void_p) for n in ("mma_cols", "mma_rows", "mma_w")] + \
               [("mma_max_np", C.c_int32), ("mma_max_kp", C.c_int32)] + \
               [("in_rows", C.c_int64), ("round_in_rows", C.c_int64)]


# -- mirrors of the device constant block (debug / CPU verification only) --

class WinoConst(C.Structure):
    _fields_ = [("kT", C.c_uint64), ("kG", C.c_uint64), ("mu", C.c_uint32), ("rho", C.c_int32)] + \
               [(n, C.c_int32) for n in ("a00", "a01", "a10", "b00", "b01", "b10")] + \
               [(n, C.c_uint32) for n in ("k1p", "k2p", "k3p", "k4p", "k5p", "mu_w", "mu_q", "rho_w",
                                          "rho_q", "toff", "pad0", "pad1")] + \
               [(n, C.c_int32) for n in ("ka01", "ka10", "kb01", "kb10")]


class PrimeConst(C.Structure):
    _fields_ = [("p", C.c_uint32), ("pinv", C.c_uint32), ("mu", C.c_uint32), ("r2", C.c_uint32),
                ("rmod", C.c_uint32), ("z", (C.c_uint32 * 7) * 7), ("zi", (C.c_uint32 * 7) * 7),
                ("g", (C.c_uint32 * 7) * 7), ("hc", (C.c_uint32 * 3) * 3), ("hs", (C.c_uint32 * 3) * 3),
                ("q_mod64", C.c_uint64), ("inv_p", C.c_double), ("wino", WinoConst * 3),
                ("bc", C.c_uint32), ("pad_bc", C.c_uint32)]


class RingConst(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("t", "alpha", "M", "N", "n1", "nitems", "np", "l", "D",
                                       "dlog2", "shift")] + \
               [("magicM", C.c_uint32), ("magicN1", C.c_uint32), ("P_mod64", C.c_uint64),
                ("decM", C.c_uint64 * 5), ("decDp", C.c_uint64 * 5), ("pc", PrimeConst * 4)]


assert C.sizeof(RingConst) == lib.sfhr_ringconst_bytes(), "RingConst layout mismatch"
assert C.sizeof(LinearDesc) == lib.sfhr_linear_desc_bytes(), "sfhr_linear_desc layout mismatch"


def ptr(a) -> int | None:
    """Device/host address of a torch tensor or numpy array (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def derive_permutation(master_seed: bytes, session_id: bytes, round_no: int, size: int) -> np.ndarray:
    """sigma_r, bit-exact with reference confidentiality.derive_permutation (:57-76), in C++."""
    out = np.empty(max(size, 0), np.int64)
    check(lib.sfhr_derive_permutation(master_seed, len(master_seed), session_id, len(session_id),
                                      round_no, size, out.ctypes.data))
    return out


def invert_permutation(perm: np.ndarray) -> np.ndarray:
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm), dtype=perm.dtype)
    return inv
