"""ctypes loader of the C NTT oracle (oracle/ntt_ref.c) — TEST INFRASTRUCTURE ONLY.

Builds ``oracle/libntt_ref.so`` with gcc on first use (``__graft_entry__.build()``
also builds it, so the prebuilt file travels to the GPU box).
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "ntt_ref.c"
LIB = HERE / "libntt_ref.so"


def build() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", str(SRC), "-o", str(LIB)], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(str(build()))
        u64, i32, i64, vp = C.c_uint64, C.c_int, C.c_int64, C.c_void_p
        L.ntt_ref_psi.restype = u64
        L.ntt_ref_psi.argtypes = [u64, i32]
        for n in ("ntt_ref_forward", "ntt_ref_inverse"):
            getattr(L, n).restype = None
            getattr(L, n).argtypes = [vp, i32, u64]
        L.ntt_ref_negacyclic.argtypes = [vp, vp, vp, i32, u64]
        L.ntt_ref_pointwise.argtypes = [vp, vp, vp, i64, u64]
        _lib = L
    return _lib


def forward(x: np.ndarray, p: int) -> np.ndarray:
    y = np.ascontiguousarray(x, dtype=np.uint64).copy()
    lib().ntt_ref_forward(y.ctypes.data, int(y.size).bit_length() - 1, p)
    return y


def inverse(x: np.ndarray, p: int) -> np.ndarray:
    y = np.ascontiguousarray(x, dtype=np.uint64).copy()
    lib().ntt_ref_inverse(y.ctypes.data, int(y.size).bit_length() - 1, p)
    return y


def negacyclic(a: np.ndarray, b: np.ndarray, p: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    c = np.empty_like(a)
    lib().ntt_ref_negacyclic(a.ctypes.data, b.ctypes.data, c.ctypes.data, a.size, p)
    return c


def pointwise(a: np.ndarray, b: np.ndarray, p: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    c = np.empty_like(a)
    lib().ntt_ref_pointwise(a.ctypes.data, b.ctypes.data, c.ctypes.data, a.size, p)
    return c


def psi(p: int, logn: int) -> int:
    return int(lib().ntt_ref_psi(p, logn))
