"""Ciphertext-block wire codec, numpy restatement — TEST INFRASTRUCTURE ONLY.

Restates reference pkg/src/sfhr/wire.py: encode_block / decode_block
(:99-124), encode_round_req / decode_round_req (:208-237), encode_round_resp /
decode_round_resp (:240-254).  Pinned by tests/golden/golden_wire.json
(digests of the real reference's payloads, tests/golden/make_golden_wire.py).
"""

from __future__ import annotations

import struct

import numpy as np


class WireError(Exception):
    def __init__(self, reason: str):
        super().__init__(reason)
        self.reason = reason


def block_size(m: int, count: int) -> int:
    """wire.py:99-100"""
    return 4 + 4 + count * 2 * m * 8 + 1


def encode_block(cts: np.ndarray, m: int, gamma: int) -> bytes:
    """wire.py:103-108: (count, 2, N) lanes zero-padded to M, little-endian u64."""
    count = cts.shape[0]
    lanes = np.zeros((count, 2, m), dtype="<u8")
    lanes[:, :, :cts.shape[2]] = cts
    return struct.pack("<II", m, count) + lanes.tobytes() + struct.pack("<B", gamma)


def decode_block(buf: bytes, offset: int, n: int):
    """wire.py:111-124: ((count, 2, N), gamma, next offset); range check on every lane."""
    if len(buf) < offset + 8:
        raise WireError("truncated ciphertext block header")
    m, count = struct.unpack_from("<II", buf, offset)
    need = block_size(m, count)
    if len(buf) < offset + need:
        raise WireError("truncated ciphertext block body")
    lanes = np.frombuffer(buf, dtype="<u8", count=count * 2 * m, offset=offset + 8).reshape(count, 2, m)
    if np.any(lanes >= (1 << 53)):
        raise WireError("torus numerator out of range")
    return lanes[:, :, :n].astype(np.uint64), buf[offset + need - 1], offset + need


def encode_round_req(power: np.ndarray, exps, m: int, gamma: int) -> bytes:
    """wire.py:208-217 for k bundles given as one (k, npow, 2, N) array (sorted exponents)."""
    out = bytearray(struct.pack("<I", power.shape[0]))
    for j in range(power.shape[0]):
        out += struct.pack("<I", len(exps))
        out += struct.pack(f"<{len(exps)}I", *exps)
        out += encode_block(power[j], m, gamma)
    return bytes(out)


def decode_round_req(payload: bytes, n: int):
    """wire.py:220-237 -> (k, npow, 2, N) array, exps, gammas."""
    if len(payload) < 4:
        raise WireError("truncated round request")
    (k,) = struct.unpack_from("<I", payload, 0)
    off = 4
    blocks, exps_all, gammas = [], [], []
    for _ in range(k):
        (npow,) = struct.unpack_from("<I", payload, off)
        off += 4
        exps = struct.unpack_from(f"<{npow}I", payload, off)
        off += 4 * npow
        batch, gamma, off = decode_block(payload, off, n)
        if batch.shape[0] != npow:
            raise WireError("power count mismatch in round request")
        blocks.append(batch)
        exps_all.append(list(exps))
        gammas.append(gamma)
    return (np.stack(blocks) if blocks else np.zeros((0, 0, 2, n), np.uint64)), exps_all, gammas


def encode_round_resp(packed: np.ndarray, m: int, gamma: int) -> bytes:
    """wire.py:240-242"""
    batch = packed if len(packed) else np.zeros((0, 2, 0), dtype=np.uint64)
    return struct.pack("<I", len(packed)) + encode_block(batch, m, gamma)


def decode_round_resp(payload: bytes, n: int) -> np.ndarray:
    """wire.py:245-254"""
    if len(payload) < 4:
        raise WireError("truncated round response")
    (count,) = struct.unpack_from("<I", payload, 0)
    batch, _, _ = decode_block(payload, 4, n)
    if batch.shape[0] != count:
        raise WireError("pack count mismatch in round response")
    return batch
