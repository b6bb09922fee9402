"""Ciphertext-block wire codec straight to / from device memory.

Mirrors reference pkg/src/sfhr/wire.py (block layout :99-124, round request /
response payloads :208-254) for the server side:

* ``decode_round_req_device(payload, N, device)``: the host parses only the
  small per-chunk headers; the whole payload is staged once in pinned memory,
  copied to the GPU, and unpacked there (``sfhr_wire_unpack``) into the
  ``(k, npow, 2, N)`` upload layout with the reference's < 2^53 range check on
  every lane, padding included.
* ``encode_round_resp_device(packs, M, gamma)``: the zero-padded ``(count, 2, M)``
  block body is laid out on the device (``sfhr_wire_pack``) and copied once into
  a pinned buffer that already holds the payload header.

Errors raise ``WireError`` with the reference's reasons.  Byte-identical to the
reference (tests/golden/golden_wire.json).
"""

from __future__ import annotations

import ctypes as C
import struct
import threading

import numpy as np
import torch

from . import _native as nat

_lib = nat.lib
_lib.sfhr_wire_unpack.restype = C.c_int
_lib.sfhr_wire_unpack.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                  C.c_void_p, C.c_void_p]
_lib.sfhr_wire_pack.restype = C.c_int
_lib.sfhr_wire_pack.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p]


class WireError(Exception):
    """Reference wire.WireError (wire.py:51-54)."""

    def __init__(self, reason: str):
        super().__init__(reason)
        self.reason = reason


def block_size(m: int, count: int) -> int:
    return 4 + 4 + count * 2 * m * 8 + 1


class _Pinned:
    """Grow-only pinned byte buffer."""

    def __init__(self):
        self.buf = None

    def get(self, n: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < n:
            self.buf = torch.empty(max(n, 1 << 20), dtype=torch.uint8, pin_memory=True)
        return self.buf[:n]


_in_stage = _Pinned()
_out_stage = _Pinned()
_stage_lock = threading.Lock()  # the pinned staging buffers are shared by all callers


def parse_round_req(payload, n: int):
    """Host-side header walk of a ROUND_REQ payload (wire.py:220-237).

    Returns (k, exps, m, gammas, body_offsets) without touching the lanes."""
    if len(payload) < 4:
        raise WireError("truncated round request")
    (k,) = struct.unpack_from("<I", payload, 0)
    off = 4
    exps0, m0 = None, None
    gammas, offs = [], []
    for _ in range(k):
        if len(payload) < off + 4:
            raise WireError("truncated ciphertext block header")
        (npow,) = struct.unpack_from("<I", payload, off)
        off += 4
        if len(payload) < off + 4 * npow:
            raise WireError("truncated ciphertext block header")
        exps = list(struct.unpack_from(f"<{npow}I", payload, off))
        off += 4 * npow
        if len(payload) < off + 8:
            raise WireError("truncated ciphertext block header")
        m, count = struct.unpack_from("<II", payload, off)
        need = block_size(m, count)
        if len(payload) < off + need:
            raise WireError("truncated ciphertext block body")
        if count != npow:
            raise WireError("power count mismatch in round request")
        if m < n:
            raise WireError("ciphertext block narrower than the ring degree")
        if exps0 is None:
            exps0, m0 = exps, m
        elif exps != exps0 or m != m0:
            raise WireError("chunks of one round request disagree on powers or width")
        offs.append(off + 8)
        gammas.append(payload[off + need - 1])
        off += need
    return k, exps0 or [], m0, gammas, offs


def decode_round_req_device(payload, n: int, device) -> tuple[torch.Tensor, list, list]:
    """ROUND_REQ payload -> ((k, npow, 2, N) int64 device tensor, exps, gammas)."""
    dev = torch.device(device)
    k, exps, m, gammas, offs = parse_round_req(payload, n)
    if k == 0:
        return torch.zeros((0, 0, 2, n), dtype=torch.int64, device=dev), exps, gammas
    size = ((len(payload) + 3) & ~3) + 4  # whole words plus the kernel's 4-byte read slack
    with _stage_lock:
        stage = _in_stage.get(size)
        stage[:len(payload)].numpy()[:] = np.frombuffer(payload, dtype=np.uint8)
        raw = stage.to(dev, non_blocking=True)
        # the pinned buffer is reused by the next caller: the copy must have landed
        torch.cuda.current_stream(dev).synchronize()
    offs_dev = torch.tensor(offs, dtype=torch.int64).to(dev, non_blocking=True)
    out = torch.empty((k, len(exps), 2, n), dtype=torch.int64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    nat.check(_lib.sfhr_wire_unpack(raw.data_ptr(), offs_dev.data_ptr(), k, len(exps), m, n, out.data_ptr(),
                                    err.data_ptr(), stream), "wire unpack")
    if int(err.item()):
        raise WireError("torus numerator out of range")
    return out, exps, gammas


def encode_round_resp_device(packs: torch.Tensor, m: int, gamma: int) -> bytes:
    """(count, 2, N) int64 device packs -> ROUND_RESP payload bytes (wire.py:240-242)."""
    count = int(packs.shape[0])
    size = 4 + block_size(m, count)
    with _stage_lock:
        return _encode_locked(packs, m, gamma, count, size)


def _encode_locked(packs: torch.Tensor, m: int, gamma: int, count: int, size: int) -> bytes:
    n = int(packs.shape[2]) if count else 0
    host = _out_stage.get(size)
    hv = host.numpy()
    hv[:12] = np.frombuffer(struct.pack("<III", count, m, count), dtype=np.uint8)
    hv[size - 1] = gamma
    if count:
        dev = packs.device
        body = torch.empty((count, 2, m), dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        nat.check(_lib.sfhr_wire_pack(packs.contiguous().data_ptr(), count, m, n, body.data_ptr(), stream),
                  "wire pack")
        host[12:12 + count * 2 * m * 8].copy_(body.view(torch.uint8).reshape(-1))
    return bytes(hv[:size])
