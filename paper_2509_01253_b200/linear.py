"""Encrypted linear map (ciphertext x plaintext MAC) on the GPU.

Operator-level mirrors of reference pkg/src/sfhr/model.py:384-429
(``int_matmul_mod_q``, ``encrypted_linear``) plus the device evaluator of a
lowered round (``model.lower_round``): a chain of grouped passes whose first
pass reads the extracted rows through the unshuffle map (sigma_{r-1},
protocol.py:243-254) and whose last pass scatters through sigma_r
(protocol.py:261-263) straight into the zero-padded pack buffer.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .device import RingContext, to_dev, to_host_u64
from .model import ROWS_PER_GROUP, LinearPass, ModelError

_LIMB = 18


class DevicePass:
    """A LinearPass uploaded to one device."""

    def __init__(self, ps: LinearPass, dev: torch.device):
        self.in_len, self.out_len = ps.in_len, ps.out_len
        self.n_groups = int(ps.groups.shape[0])
        up = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa
        self.groups = up(ps.groups)
        self.cols = up(ps.cols)
        self.weights = up(ps.weights)
        self.rows = up(ps.rows)
        self.ex_ptr, self.ex_col, self.ex_w = up(ps.ex_ptr), up(ps.ex_col), up(ps.ex_w)
        self.bias = up(ps.bias)
        self.macs_per_lane = ps.macs_per_lane()


def run_pass(ctx: RingContext, p: DevicePass, inp, in_map, round_in, round_map, out, out_map, unit,
             lanes: int = 0, body_off: int = 0):
    d = nat.LinearDesc()
    d.in_ = nat.ptr(inp)
    d.in_map = nat.ptr(in_map)
    d.round_in = nat.ptr(round_in)
    d.round_map = nat.ptr(round_map)
    d.out = nat.ptr(out)
    d.out_map = nat.ptr(out_map)
    d.groups = nat.ptr(p.groups)
    d.n_groups = p.n_groups
    d.cols = nat.ptr(p.cols)
    d.weights = nat.ptr(p.weights)
    d.rows = nat.ptr(p.rows)
    d.ex_ptr, d.ex_col, d.ex_w = nat.ptr(p.ex_ptr), nat.ptr(p.ex_col), nat.ptr(p.ex_w)
    d.bias = nat.ptr(p.bias)
    d.unit = nat.ptr(unit)
    d.lanes = lanes
    d.body_off = body_off
    import ctypes as C
    nat.check(nat.lib.sfhr_linear_pass(ctx.h, C.byref(d), ctx.stream()))


def run_round(ctx: RingContext, passes: list, rows_in: torch.Tensor, in_map, out: torch.Tensor,
              out_map, unit: torch.Tensor):
    """Evaluate a lowered round: rows_in (physical, via in_map) -> out (via out_map)."""
    cur, cur_map = rows_in, in_map
    for k, p in enumerate(passes):
        last = k == len(passes) - 1
        dst = out if last else torch.empty((p.out_len, 2, ctx.N), dtype=torch.int64, device=ctx.dev)
        run_pass(ctx, p, cur, cur_map, rows_in, in_map, dst, out_map if last else None, unit)
        cur, cur_map = dst, None
    return out


def _dense_pass(w: np.ndarray) -> LinearPass:
    """Generic (E_out, E_in) integer matrix as a pass: row chunks of 16, all columns."""
    from .model import _GroupBuilder
    gb = _GroupBuilder()
    e_out, e_in = w.shape
    cols = np.arange(e_in)
    for r0 in range(0, e_out, ROWS_PER_GROUP):
        r = np.arange(r0, min(e_out, r0 + ROWS_PER_GROUP))
        gb.add(cols, gb.block(w[r]), r, e_in, 0)
    return gb.build(e_in, e_out, None)


def _ctx_for_rows(device: int, n: int | None):
    # any context works for a generic lane count; pick the b=12 row
    return RingContext.get(7, 4, 12, 1 << 16, 2, 1, 0, device)


def int_matmul_mod_q(w: np.ndarray, rows, device: int = 0):
    """Exact W @ rows mod 2^53 (reference model.py:384-407), on the GPU.

    Keeps the reference's exactness guard (ModelError when
    max|W| * E_in * 2^18 >= 2^53) for error-behaviour parity, although the
    device kernel itself is exact for any int32 weights.
    """
    w = np.asarray(w, np.int64)
    e_out, e_in = w.shape
    if float(np.abs(w).max(initial=0)) * e_in * (1 << _LIMB) >= 2 ** 53:
        raise ModelError("weight magnitude too large for exact lane combination")
    host = not isinstance(rows, torch.Tensor)
    ctx = _ctx_for_rows(device, None)
    x = to_dev(np.asarray(rows, np.uint64), ctx.dev) if host else rows
    lanes = int(np.prod(x.shape[1:])) if x.dim() > 1 else 1
    out = torch.empty((e_out,) + tuple(x.shape[1:]), dtype=torch.int64, device=ctx.dev)
    if e_out and e_in:
        p = DevicePass(_dense_pass(w), ctx.dev)
        run_pass(ctx, p, x, None, x, None, out, None, None, lanes=lanes, body_off=lanes)
    elif e_out:
        out.zero_()
    return to_host_u64(out) if host else out


def encrypted_linear(w: np.ndarray, bias, ct_rows, bias_unit_payload, device: int = 0):
    """Apply one round's integer matrix to extracted rows (reference model.py:410-429)."""
    if hasattr(ct_rows, "data") and not isinstance(ct_rows, (np.ndarray, torch.Tensor)):
        ct_rows = ct_rows.data
    w = np.asarray(w, np.int64)
    if w.shape[1] != ct_rows.shape[0]:
        raise ModelError(f"round matrix expects {w.shape[1]} rows, got {ct_rows.shape[0]}")
    if float(np.abs(w).max(initial=0)) * w.shape[1] * (1 << _LIMB) >= 2 ** 53:
        raise ModelError("weight magnitude too large for exact lane combination")
    host = not isinstance(ct_rows, torch.Tensor)
    ctx = _ctx_for_rows(device, None)
    x = to_dev(np.asarray(ct_rows, np.uint64), ctx.dev) if host else ct_rows
    N = x.shape[2]
    ps = _dense_pass(w)
    if bias is not None and np.any(bias):
        ps.bias = np.asarray(bias, np.int64)
    p = DevicePass(ps, ctx.dev)
    unit = to_dev(np.asarray(bias_unit_payload, np.uint64), ctx.dev)
    out = torch.empty((w.shape[0], 2, N), dtype=torch.int64, device=ctx.dev)
    run_pass(ctx, p, x, None, x, None, out, None, unit, lanes=2 * N, body_off=N)
    return to_host_u64(out) if host else out
