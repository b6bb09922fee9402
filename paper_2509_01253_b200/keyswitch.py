"""KeySwitchEngine drop-in: automorphism + gadget key switch on the GPU.

Mirrors reference pkg/src/sfhr/crypto.py:360-474 (``KeySwitchEngine``) with a
third backend, ``mode="cuda"``: the digit convolutions run as exact
Phi_M-NTTs over word-size primes inside one fused sm_100a kernel
(csrc/keyswitch.cu) instead of float FFTs (``fft``) or uint64 schoolbook
(``exact``).  Results are bit-identical to the reference's exact mode.

Arrays may be numpy uint64 (host; copied to and from the device) or torch
int64 CUDA tensors (device-resident; no copies).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .device import DeviceKey, RingContext, to_dev, to_host_u64
from .params import GadgetParams, RingParams


@dataclass
class RlweCiphertext:
    """(a, b) uint64 numerators, length N (reference crypto.py:55-62)."""
    a: np.ndarray
    b: np.ndarray
    noise_hint: float = 0.0

    def as_batch(self) -> np.ndarray:
        return np.stack([self.a, self.b])[None, :, :]


@dataclass
class KeySwitchKeySet:
    """Per automorphism index d: l RLWE encryptions of s(X^d)/D^i (reference crypto.py:72-81)."""
    keys: dict
    gadget: GadgetParams
    delta: float
    params: RingParams

    def indices(self) -> list:
        return sorted(self.keys)


def _as_dev(x, ctx: RingContext):
    if isinstance(x, torch.Tensor):
        if x.device != ctx.dev or x.dtype != torch.int64:
            raise ValueError("device batches must be int64 tensors on the engine's device")
        x = x.contiguous()
        # the C-ABI takes 16-byte aligned rows (bulk copies); a view at an odd u64 offset is copied
        return (x.clone() if x.data_ptr() % 16 else x), False
    x = np.ascontiguousarray(np.asarray(x, dtype=np.uint64))
    return to_dev(x, ctx.dev), True


class KeySwitchEngine:
    """Drop-in for reference crypto.KeySwitchEngine (crypto.py:360-474), CUDA backend."""

    def __init__(self, ksk, mode: str = "cuda", max_chunk: int = 128, device: int = 0,
                 gamma: int = 0, beta: int = 0):
        if mode not in ("cuda", "fft", "exact"):
            raise ValueError(f"unknown key-switch mode {mode!r}")
        # every mode runs the same bit-exact device kernel; 'fft'/'exact' are accepted
        # so reference call sites keep working.
        self.ksk = ksk
        self.params = ksk.params
        self.mode = mode
        self.max_chunk = max_chunk
        R = self.params
        g = ksk.gadget
        self.ctx = RingContext.get(R.t, R.alpha, R.p_bits, g.D, g.l, gamma, beta, device)
        self.key = DeviceKey(self.ctx, ksk)
        N = R.N
        self.switch_noise = (ksk.delta * g.D / 2 * np.sqrt(g.l * N)
                             + np.sqrt(N) / (2.0 * float(g.D) ** g.l))

    # -- batched operators --------------------------------------------------

    def automorphism_batch(self, cts, d: int):
        """P(X) -> P(X^d) on a (B, 2, N) batch (reference crypto.py:400-402)."""
        x, host = _as_dev(cts, self.ctx)
        out = torch.empty_like(x)
        nat.check(nat.lib.sfhr_automorphism_batch(self.ctx.h, int(d) % self.ctx.M, nat.ptr(x),
                                                  nat.ptr(out), x.shape[0], self.ctx.stream()))
        return to_host_u64(out) if host else out

    def _need(self, d):
        if int(d) % self.ctx.M not in self.key.indices:
            raise KeyError(f"key-switch key set has no index {d}")

    def switch_batch(self, cts, d: int, counter=None, skip_zero: bool = False):
        """Key switch (B, 2, N) from s(X^d) back to s(X) (reference crypto.py:404-421)."""
        self._need(d)
        x, host = _as_dev(cts, self.ctx)
        out = torch.empty_like(x)
        cnt = self.ctx.counter() if counter is not None else None
        nat.check(nat.lib.sfhr_keyswitch_batch(self.ctx.h, self.key.h, int(d) % self.ctx.M, nat.ptr(x),
                                               nat.ptr(out), x.shape[0], int(skip_zero), nat.ptr(cnt),
                                               self.ctx.stream()))
        if counter is not None:
            counter.add_switches(int(cnt.item()))
        return to_host_u64(out) if host else out

    def stage_batch(self, cts, reps, counter=None, skip_zero: bool = False):
        """acc = x + sum_{rep in reps[1:]} KS_rep(aut_rep(x)) (reference tracepack.py:268-285)."""
        for r in reps[1:]:
            self._need(r)
        x, host = _as_dev(cts, self.ctx)
        out = torch.empty_like(x)
        reps_np = np.asarray([int(r) % self.ctx.M for r in reps], np.uint32)
        cnt = self.ctx.counter() if counter is not None else None
        nat.check(nat.lib.sfhr_stage_batch(self.ctx.h, self.key.h, reps_np.ctypes.data, len(reps_np),
                                           nat.ptr(x), nat.ptr(out), x.shape[0], int(skip_zero),
                                           nat.ptr(cnt), self.ctx.stream()))
        if counter is not None:
            counter.add_switches(int(cnt.item()))
        return to_host_u64(out) if host else out

    def homomorphic_automorphism(self, ct: RlweCiphertext, d: int, counter=None) -> RlweCiphertext:
        """Single-ciphertext wrapper with the identity shortcut (reference crypto.py:466-474)."""
        if d % self.params.M == 1:
            return ct
        moved = self.automorphism_batch(ct.as_batch(), d)
        sw = self.switch_batch(moved, d, counter=counter)
        return RlweCiphertext(a=sw[0, 0], b=sw[0, 1], noise_hint=ct.noise_hint + self.switch_noise)
