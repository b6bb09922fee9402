"""Client-side RLWE batch operations with the key product on the GPU.

Drop-ins for the client half of reference pkg/src/sfhr/crypto.py:

* ``KeyMul(s, params)`` replaces ``_KeyMulOp`` (crypto.py:106-150): s(X) * v mod Phi_M,
  exact mod 2^53, for a batch of polynomials.  The operator is the reference's own
  Toeplitz-mod-Phi matrix of s (entries in {-2..2} for binary / ternary keys), applied
  to the batch as a ct x pt linear map on the tcgen05 tensor cores (the byte-plane
  int8 GEMM of ``linear.py`` with the polynomial coefficients as rows and the batch as
  lanes) instead of three float64 limb GEMMs.
* ``encrypt_rlwe_batch`` (crypto.py:166-199) and ``rlwe_phase_batch`` (:228-230) keep every
  random draw (a*, e*) and the dual-basis scatter in numpy, in the reference's order, so
  the ciphertexts are bit-identical for the same generator state; only the s * a product
  moves to the device.

The client is off the server hot path; this serves in-process loops (``run_inference``
style benchmarks) whose client side would otherwise dominate.
"""

from __future__ import annotations

import numpy as np
import torch

from .linear import DevicePass, _ctx_for_rows, _dense_pass, run_pass
from .params import RingParams

Q = 1 << 53
_MASK = np.uint64(Q - 1)


def key_matrix(s: np.ndarray, params: RingParams) -> np.ndarray:
    """(N, N) integer operator of v -> s * v mod Phi_M (reference crypto.py:116-129)."""
    M, N, n1 = params.M, params.N, params.n1
    big = np.zeros((M, N), np.int64)
    rows = (np.arange(N)[:, None] + np.arange(N)[None, :]) % M
    np.add.at(big, (rows, np.broadcast_to(np.arange(N), (N, N))), np.asarray(s, np.int64)[:, None])
    k = np.arange(N)
    return big[:N] - big[N + k % n1]


class KeyMul:
    """s(X) * v mod Phi_M for (B, N) batches, exact mod 2^53, on the GPU."""

    def __init__(self, s: np.ndarray, params: RingParams, device: int = 0):
        self.params = params
        self.ctx = _ctx_for_rows(device, None)
        mat = key_matrix(s, params)
        self.pass_ = DevicePass(_dense_pass(mat), self.ctx.dev, lanes=2)
        if self.pass_.n_mma_tiles == 0:
            raise ValueError("key operator does not fit the tensor-core path")

    def times(self, v: np.ndarray) -> np.ndarray:
        """v: (..., N) uint64 -> s * v mod Phi_M (..., N) uint64."""
        v = np.asarray(v, dtype=np.uint64)
        N = self.params.N
        flat = v.reshape(-1, N)
        B = flat.shape[0]
        if B == 0:
            return np.zeros_like(v)
        lanes = B + (B & 1)  # the tensor-core path needs an even lane count
        x = np.zeros((N, lanes), np.uint64)
        x[:, :B] = flat.T
        xd = torch.from_numpy(x.view(np.int64)).to(self.ctx.dev)
        out = torch.empty_like(xd)
        run_pass(self.ctx, self.pass_, xd, None, xd, None, out, None, None, lanes=lanes, body_off=lanes)
        res = out.cpu().numpy().view(np.uint64)[:, :B].T
        return np.ascontiguousarray(res).reshape(v.shape)


def encrypt_rlwe_batch(payloads: np.ndarray, key_mul: KeyMul, delta: float, rng: np.random.Generator,
                       scatter_idx: np.ndarray, scatter_coef: np.ndarray) -> np.ndarray:
    """Reference encrypt_rlwe_batch (crypto.py:166-199) with the key product on the GPU.

    scatter_idx / scatter_coef are the reference DualBasis scatter tables (dual.py)."""
    payloads = np.atleast_2d(np.asarray(payloads, dtype=np.uint64))
    B, N = payloads.shape
    a_star = rng.integers(0, Q, (B, N), dtype=np.uint64)
    e_star = rng.normal(0.0, delta, (B, N)) if delta > 0 else np.zeros((B, N))
    a_t = np.zeros((N, B), np.uint64)
    e_t = np.zeros((N, B))
    for k in range(scatter_idx.shape[1]):
        idx = scatter_idx[:, k]
        coef = scatter_coef[:, k]
        np.add.at(a_t, idx, (a_star * coef.astype(np.uint64)[None, :]).T)
        np.add.at(e_t, idx, (e_star * coef[None, :]).T)
    a = a_t.T & _MASK
    e_num = np.rint(e_t.T * float(Q)).astype(np.int64).astype(np.uint64)
    out = np.empty((B, 2, N), np.uint64)
    out[:, 0] = a
    out[:, 1] = (key_mul.times(a) + payloads + e_num) & _MASK
    return out


def rlwe_phase_batch(cts: np.ndarray, key_mul: KeyMul) -> np.ndarray:
    """Phases b - s * a of a (B, 2, N) batch (reference crypto.py:228-230)."""
    cts = np.asarray(cts, dtype=np.uint64)
    return (cts[:, 1] - key_mul.times(cts[:, 0])) & _MASK


def project_p(phase: np.ndarray, params: RingParams) -> np.ndarray:
    """Round torus phases to the message grid mod p (reference crypto.py:159-163)."""
    shift = 53 - params.p_bits
    rounded = (np.asarray(phase, np.uint64) + np.uint64(1 << (shift - 1))) >> np.uint64(shift)
    return (rounded & np.uint64(params.p - 1)).astype(np.int64)
