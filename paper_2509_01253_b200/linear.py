"""Encrypted linear map (ciphertext x plaintext MAC) on the GPU.

Operator-level mirrors of reference pkg/src/sfhr/model.py:384-429
(``int_matmul_mod_q``, ``encrypted_linear``) plus the device evaluator of a
lowered round (``model.lower_round``): a chain of grouped passes whose first
pass reads the extracted rows through the unshuffle map (sigma_{r-1},
protocol.py:243-254) and whose last pass scatters through sigma_r
(protocol.py:261-263) straight into the zero-padded pack buffer.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .device import RingContext, to_dev, to_host_u64
from .model import ROWS_PER_GROUP, LinearPass, ModelError

_LIMB = 18
MMA_MAX_ROWS = 256      # N of one tcgen05 tile group
MMA_MAX_KPAD = 8192     # taps per tile group (row-pointer table in shared memory)
MMA_ENABLED = os.environ.get("SFHR_LINEAR_MMA", "1") != "0"
# tile::gather4 TMA producer instead of per-thread cp.async gathers (A/B on B200: 153.5 vs 151.1 ms
# per ResNet-20 inference, so cp.async stays the default)
MMA_TMA = os.environ.get("SFHR_LINEAR_TMA", "0") == "1"


@dataclass
class MmaTiles:
    """Tensor-core tile groups of a pass (csrc/linear_mma.cu).

    tiles: (T, 8) int32 [cols_off, K_pad, w_off, rows_off, nrows, N_pad, 0, 0];
    cols: K_pad input columns per tile (-1 = zero tap); rows: canonical output
    rows; w: s8 weights packed as UMMA K-major core matrices (8 rows x 16 B).
    """
    tiles: np.ndarray
    cols: np.ndarray
    rows: np.ndarray
    w: np.ndarray
    max_np: int
    max_kp: int


def _pack_umma_k_major(wt: np.ndarray, n_pad: int, k_pad: int) -> np.ndarray:
    """(n, k) int8 -> canonical no-swizzle K-major layout [k/16][n/8][8][16]."""
    b = np.zeros((n_pad, k_pad), np.int8)
    b[:wt.shape[0], :wt.shape[1]] = wt
    return np.ascontiguousarray(b.reshape(n_pad // 8, 8, k_pad // 16, 16).transpose(2, 0, 1, 3)).reshape(-1)


# Cost model for merging tile groups (per 16-lane M-tile, in SM clocks): the cp.async gather of one
# 128-byte tap ~ MMA_GATHER_CLK (measured: ~20 B/clk/SM on the producer path), the tensor work of one
# tap ~ N_pad / 64 (8192 int8 MAC/clk/SM).  Merging pixels whose column windows overlap (3x3 convs)
# trades extra (zero-weight) MACs for fewer gathered taps per output row.
MMA_GATHER_CLK = float(os.environ.get("SFHR_MMA_GATHER_CLK", "6.5"))
# rows of a tile group that merges different column lists (A/B on B200, ResNet-20 linear ms per
# inference: 9.44 unmerged, 7.64 at 64 rows / 2x2 pixel blocks, 8.5-10.9 at 96-256 rows)
MMA_RUN_ROWS = int(os.environ.get("SFHR_MMA_RUN_ROWS", "64"))
MMA_SAME_ROWS = int(os.environ.get("SFHR_MMA_SAME_ROWS", str(MMA_MAX_ROWS)))  # runs sharing one list
# merged s8 weight operands stay at or below this size (A/B-tuned: larger merged tiles lose
# more to zero-weight MACs than they save in gathers); it must not exceed what the kernel keeps
# resident in shared memory (sfhr_mma_b_resident_bytes(), B_RESIDENT_MAX in csrc/linear_mma.cu)
MMA_MERGE_B_MAX = min(96 * 1024, int(nat.lib.sfhr_mma_b_resident_bytes()))


def _run_cost(k_pad: int, n_pad: int, rows: int) -> float:
    return max(MMA_GATHER_CLK * k_pad, k_pad * n_pad / 64.0) / rows


def split_mma_tiles(ps: LinearPass):
    """Merge runs of groups into tcgen05 tile groups.

    Returns (rest_group_indices, MmaTiles | None).  A run of consecutive groups
    becomes one tile group over the union of their column lists (conv: the
    output-channel chunks of a pixel, then neighbouring pixels of the lowering's
    pixel blocks, whose 3x3 windows overlap; fc / dense: all row chunks) while
    the cost model above improves, N <= 256 and the merged s8 weights stay within
    MMA_MERGE_B_MAX (<= the kernel's resident-weight limit, so merged runs never stream
    their weights; unmerged wide layers above it do).  Runs with |w| > 127 stay on the CUDA-core kernel; per-row column
    lists (pooling, identity) join as block-sparse tile groups over the union of their
    rows' columns.
    """
    g = ps.groups
    G = len(g)
    if not MMA_ENABLED or G == 0:
        return np.arange(G), None
    wv = ps.weights
    rest, tiles, tcols, trows, tw = [], [], [], [], []
    cache = {}
    ncols = nrows = nw = 0
    max_np = max_kp = 0

    def gcols(q):  # every valid input column the group reads (per-row lists concatenated)
        c0, nc, nr, per = int(g[q][0]), int(g[q][1]), int(g[q][4]), int(g[q][5])
        c = ps.cols[c0:c0 + (nr * nc if per else nc)].astype(np.int64)
        return c[c >= 0]

    i = 0
    while i < G:
        c0, nc, w0, r0, nr, per = (int(x) for x in g[i])
        if nc == 0:
            rest.append(i)
            i += 1
            continue
        # per-row column lists (pooling, identity) become a tile group over their union with
        # block-sparse weights: each input row is still gathered once per output group
        run, tot, j = [i], nr, i + 1
        union = np.unique(gcols(i))
        best = _run_cost((len(union) + 31) // 32 * 32, (tot + 15) // 16 * 16, tot)
        all_same = not per
        while j < G:
            cj, ncj, _, _, nrj, perj = (int(x) for x in g[j])
            if ncj == 0 or tot + nrj > min(MMA_MAX_ROWS, MMA_SAME_ROWS):
                break
            same = not per and not perj and ncj == nc and (
                cj == c0 or np.array_equal(ps.cols[cj:cj + ncj], ps.cols[c0:c0 + nc]))
            all_same = all_same and same
            if not all_same and tot + nrj > MMA_RUN_ROWS:
                break
            u2 = union if same else np.union1d(union, gcols(j))
            k2, n2 = (len(u2) + 31) // 32 * 32, (tot + nrj + 15) // 16 * 16
            if k2 > MMA_MAX_KPAD or (n2 * k2 > MMA_MERGE_B_MAX and not same):
                break
            c2 = _run_cost(k2, n2, tot + nrj)
            if not same and c2 > 0.98 * best:
                break
            run.append(j)
            tot += nrj
            union, best = u2, min(best, c2)
            j += 1
        rows_run = np.concatenate([ps.rows[int(g[q][3]):int(g[q][3]) + int(g[q][4])] for q in run])
        # residual extras (CSR into the round input) become extra taps
        ex_cols, ex_vals = np.zeros(0, np.int64), None
        if ps.ex_ptr is not None:
            lo, hi = ps.ex_ptr[rows_run], ps.ex_ptr[rows_run + 1]
            if np.any(hi > lo):
                idx = np.concatenate([np.arange(a, b) for a, b in zip(lo, hi)])
                ex_cols = np.unique(ps.ex_col[idx])
                ex_vals = np.zeros((tot, len(ex_cols)), np.int64)
                for ri, (a, b) in enumerate(zip(lo, hi)):
                    np.add.at(ex_vals[ri], np.searchsorted(ex_cols, ps.ex_col[a:b]), ps.ex_w[a:b])
        nu = len(union)
        nu4 = (nu + 3) // 4 * 4 if len(ex_cols) else nu  # TMA gathers 4 taps of one input at a time
        kk = nu4 + len(ex_cols)
        k_pad = (kk + 31) // 32 * 32
        n_pad = (tot + 15) // 16 * 16
        wt = np.zeros((tot, kk), np.int64)
        ro = 0
        for q in run:
            cq, ncq, wq, _, nrq, perq = (int(x) for x in g[q])
            blk = wv[wq:wq + ncq * ROWS_PER_GROUP].reshape(ncq, ROWS_PER_GROUP)[:, :nrq].astype(np.int64)
            sub = np.zeros((nrq, nu), np.int64)
            if perq:  # row i reads cols[cq + i*ncq : ...] with weights blk[:, i]
                cl = ps.cols[cq:cq + nrq * ncq].astype(np.int64).reshape(nrq, ncq)
                ok = cl >= 0
                np.add.at(sub, (np.nonzero(ok)[0], np.searchsorted(union, cl[ok])), blk.T[ok])
            else:
                cl = ps.cols[cq:cq + ncq].astype(np.int64)
                ok = cl >= 0
                np.add.at(sub.T, np.searchsorted(union, cl[ok]), blk[ok])
            wt[ro:ro + nrq, :nu] = sub
            ro += nrq
        if ex_vals is not None:
            wt[:, nu4:] = ex_vals
        if np.abs(wt).max(initial=0) > 127 or k_pad > MMA_MAX_KPAD or len(ex_cols) > 256:
            rest.extend(run)
            i = j
            continue
        w8 = wt.astype(np.int8)
        key = (n_pad, k_pad, w8.tobytes())  # interior pixel blocks share one weight operand
        woff = cache.get(key)
        if woff is None:
            woff = nw
            packed = _pack_umma_k_major(w8, n_pad, k_pad)
            tw.append(packed)
            nw += packed.size
            cache[key] = woff
        tiles.append((ncols, k_pad, woff, nrows, tot, n_pad, 0, 0))
        tc = np.full(k_pad, -1, np.int64)
        tc[:nu] = union
        tc[nu4:kk] = -(ex_cols + 2)
        tcols.append(tc)
        ncols += k_pad
        trows.append(rows_run)
        nrows += tot
        max_np, max_kp = max(max_np, n_pad), max(max_kp, k_pad)
        i = j
    if not tiles:
        return np.arange(G), None
    if nw >= 2 ** 31 or ncols >= 2 ** 31:
        return np.arange(G), None
    return np.asarray(rest, np.int64), MmaTiles(
        np.asarray(tiles, np.int32).reshape(-1, 8), np.concatenate(tcols).astype(np.int32),
        np.concatenate(trows).astype(np.int32), np.concatenate(tw), max_np, max_kp)


class DevicePass:
    """A LinearPass uploaded to one device (CUDA-core groups + tcgen05 tile groups)."""

    def __init__(self, ps: LinearPass, dev: torch.device, lanes: int | None = None):
        self.in_len, self.out_len = ps.in_len, ps.out_len
        up = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa
        rest, mt = split_mma_tiles(ps) if lanes is None or lanes % 2 == 0 else (np.arange(len(ps.groups)), None)
        self.n_groups = int(len(rest))
        self.groups = up(ps.groups[rest].reshape(-1, 6)) if len(rest) else None
        self.cols = up(ps.cols)
        self.weights = up(ps.weights)
        self.rows = up(ps.rows)
        self.ex_ptr, self.ex_col, self.ex_w = up(ps.ex_ptr), up(ps.ex_col), up(ps.ex_w)
        self.bias = up(ps.bias)
        self.macs_per_lane = ps.macs_per_lane()
        self.n_mma_tiles = 0 if mt is None else int(len(mt.tiles))
        self.mma_tiles = self.mma_cols = self.mma_rows = self.mma_w = None
        self.mma_max_np = self.mma_max_kp = 0
        if mt is not None:
            self.mma_tiles, self.mma_cols, self.mma_rows = up(mt.tiles), up(mt.cols), up(mt.rows)
            self.mma_w = up(mt.w.view(np.uint8))
            self.mma_max_np, self.mma_max_kp = mt.max_np, mt.max_kp


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
    d.mma_tiles, d.n_mma_tiles = nat.ptr(p.mma_tiles), p.n_mma_tiles
    d.mma_cols, d.mma_rows, d.mma_w = nat.ptr(p.mma_cols), nat.ptr(p.mma_rows), nat.ptr(p.mma_w)
    d.mma_max_np, d.mma_max_kp = p.mma_max_np, p.mma_max_kp
    if MMA_TMA and p.n_mma_tiles:
        d.in_rows = int(inp.shape[0])
        d.round_in_rows = int(round_in.shape[0]) if round_in is not None else 0
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
        p = DevicePass(_dense_pass(w), ctx.dev, lanes=lanes)
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
