"""Standalone RNS negacyclic NTT on the GPU (BASELINE.json configs[1]).

The north star's "RNS NTT/iNTT" primitive for power-of-two rings
Z_p[X]/(X^N + 1), N = 2^10..2^16, L limbs of ~50-bit primes p = 1 (mod 2N).
The reference has no such ring; this module exists for
the primitive microbenchmark and is not on the Safhire server path, whose
transforms are the Phi_M-NTTs fused inside the key-switch kernel.

Data: torch int64 tensors (batch, L, N) holding u64 residues, on the plan's
device; transforms are in place (forward: bit-reversed output order).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as nat

_lib = nat.lib
_lib.sfhr_ntt_plan_create.restype = C.c_int
_lib.sfhr_ntt_plan_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
_lib.sfhr_ntt_plan_destroy.argtypes = [C.c_void_p]
_lib.sfhr_ntt_plan_primes.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
_lib.sfhr_ntt_plan_tables.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
_lib.sfhr_ntt_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
_lib.sfhr_ntt_inverse.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
_lib.sfhr_ntt_last_error.restype = C.c_char_p


def _check(code: int) -> None:
    if code == nat.SFHR_OK:
        return
    msg = (_lib.sfhr_ntt_last_error() or b"").decode()
    if code == nat.SFHR_EINVAL:
        raise ValueError(msg)
    raise nat.SfhrCudaError(msg)


class RnsNtt:
    """Plan for (L, 2^log2n) residue polynomials; ``device=-1`` plans without a GPU."""

    def __init__(self, log2n: int, L: int, prime_bits: int = 50, device: int = 0):
        self.log2n, self.N, self.L, self.device = log2n, 1 << log2n, L, device
        h = C.c_void_p()
        _check(_lib.sfhr_ntt_plan_create(log2n, L, prime_bits, device, C.byref(h)))
        self.h = h
        pr = np.zeros(L, np.uint64)
        _check(_lib.sfhr_ntt_plan_primes(h, pr.ctypes.data, L))
        self.primes = pr

    def tables(self):
        w = np.zeros((self.L, self.N), np.uint64)
        wi = np.zeros((self.L, self.N), np.uint64)
        _check(_lib.sfhr_ntt_plan_tables(self.h, w.ctypes.data, wi.ctypes.data))
        return w, wi

    def _run(self, fn, x: torch.Tensor, stream=None):
        if not isinstance(x, torch.Tensor) or x.dtype != torch.int64 or not x.is_cuda:
            raise ValueError("expected a CUDA int64 tensor of u64 residues")
        if x.shape[-2:] != (self.L, self.N) or not x.is_contiguous():
            raise ValueError(f"expected contiguous (batch, {self.L}, {self.N}) residues")
        batch = x.numel() // (self.L * self.N)
        st = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
        _check(fn(self.h, x.data_ptr(), batch, st))
        return x

    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        return self._run(_lib.sfhr_ntt_forward, x, stream)

    def inverse(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        return self._run(_lib.sfhr_ntt_inverse, x, stream)

    def close(self):
        if self.h:
            _lib.sfhr_ntt_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
