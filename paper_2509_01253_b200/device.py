"""Device-side plumbing: one native context per (ring row, gadget, levels, GPU).

torch provides device memory, streams and the caching allocator; uint64
ciphertext arrays travel as int64 tensors (same bits; torch has no uint64
arithmetic, and none is done in torch — all arithmetic is in the kernels).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _native as nat


def require_cuda(device) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_01253_b200 runs on CUDA (sm_100a) only; no CUDA device visible")
    dev = torch.device("cuda", device if isinstance(device, int) else torch.device(device).index or 0)
    return dev


def to_dev(a: np.ndarray, dev: torch.device) -> torch.Tensor:
    """Host uint64/int64/int32 numpy array -> device tensor (bit-preserving)."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a).to(dev, non_blocking=False)


def to_host_u64(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)


def stream_ptr(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


class RingContext:
    """sfhr_ctx for one scheme row on one device (reference params.py:117-164 shapes)."""

    _cache: dict = {}
    _lock = threading.Lock()

    @classmethod
    def get(cls, t, alpha, p_bits, D, l, gamma=0, beta=0, device=0) -> "RingContext":
        key = (t, alpha, p_bits, D, l, gamma, beta, device)
        with cls._lock:
            ctx = cls._cache.get(key)
            if ctx is None:
                ctx = cls(t, alpha, p_bits, D, l, gamma, beta, device)
                cls._cache[key] = ctx
            return ctx

    @classmethod
    def for_scheme(cls, scheme, device=0) -> "RingContext":
        R = scheme.ring
        return cls.get(R.t, R.alpha, R.p_bits, scheme.gadget.D, scheme.gadget.l, scheme.gamma,
                       scheme.beta, device)

    def __init__(self, t, alpha, p_bits, D, l, gamma, beta, device):
        self.dev = require_cuda(device)
        h = C.c_void_p()
        with torch.cuda.device(self.dev):
            nat.check(nat.lib.sfhr_ctx_create(t, alpha, p_bits, D, l, gamma, beta, self.dev.index,
                                              C.byref(h)))
        self.h = h
        info = (C.c_int64 * 32)()
        k = nat.lib.sfhr_ctx_info(h, info, 32)
        self.info = list(info[:k])
        self.M, self.N, self.n1, self.np = self.info[:4]
        self.pack_factor, self.beta_eff = self.info[4], self.info[5]
        self.t, self.alpha, self.p_bits, self.D, self.l, self.gamma = t, alpha, p_bits, D, l, gamma
        e1 = np.zeros(self.N, np.int32)
        e2 = np.zeros(self.N, np.int32)
        c = np.zeros(self.N, np.int32)
        nat.check(nat.lib.sfhr_ctx_dual(h, e1.ctypes.data, e2.ctypes.data, c.ctypes.data))
        self.e1, self.e2, self.ratio_len = e1, e2, c
        self.inv_m_mod_p = self.info[7]
        self.cu = self.info[8]

    def stream(self) -> int:
        return stream_ptr(self.dev)

    @property
    def tensor_core_min_reps(self) -> int:
        """Stage launches with at least this many switched representatives use the
        tensor-core forward key switch (keyswitch_tc.cu); 0 = never."""
        return int(nat.lib.sfhr_ctx_tc_enabled(self.h))

    @tensor_core_min_reps.setter
    def tensor_core_min_reps(self, k: int) -> None:
        nat.check(nat.lib.sfhr_ctx_set_tc(self.h, int(k)))

    def counter(self) -> torch.Tensor:
        return torch.zeros(1, dtype=torch.int64, device=self.dev)

    def __del__(self):
        try:
            nat.lib.sfhr_ctx_destroy(self.h)
        except Exception:
            pass


class DeviceKey:
    """Registered key-switching key set (NTT-domain spectra live on the device)."""

    def __init__(self, ctx: RingContext, ksk):
        idx = sorted(int(d) % ctx.M for d in ksk.keys)
        l = ctx.l
        arr = np.empty((len(idx), l, 2, ctx.N), np.uint64)
        for s, d in enumerate(idx):
            row = ksk.keys[d]
            if len(row) != l:
                raise ValueError(f"key set index {d} has {len(row)} gadget levels, expected {l}")
            for i, ct in enumerate(row):
                arr[s, i, 0] = ct.a
                arr[s, i, 1] = ct.b
        self.ctx = ctx
        self.indices = idx
        dev_keys = to_dev(arr, ctx.dev)
        h = C.c_void_p()
        idx_np = np.asarray(idx, np.uint32)
        with torch.cuda.device(ctx.dev):
            nat.check(nat.lib.sfhr_register_ksk(ctx.h, idx_np.ctypes.data, len(idx), nat.ptr(dev_keys),
                                                ctx.stream(), C.byref(h)))
            torch.cuda.current_stream(ctx.dev).synchronize()
        self.h = h

    def __del__(self):
        try:
            nat.lib.sfhr_key_destroy(self.h)
        except Exception:
            pass
