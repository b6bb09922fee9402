"""Quantized model description + lowering of each round to device linear passes.

The model API (LayerSpec, RoundSpec, QuantModel, ModelError, load/save,
with_acc_bits) keeps the reference's names and semantics
(reference pkg/src/sfhr/model.py:24-121, 246-287, 436-523) so a reference
model object or manifest is accepted unchanged by ``ServerEngine``.

What differs is the lowering.  The reference builds one dense int64 round
matrix by composing per-layer dense matrices (``round_matrix``,
model.py:332-353; 66 s for a 2352-row conv round, infeasible at ResNet
sizes).  Here each layer of a round becomes one *pass* over ciphertext rows,
described by compact arrays the linear kernel consumes directly:

* group: a set of output rows sharing one input-column list (a conv output
  pixel and up to ``ROWS_PER_GROUP`` of its channels; a chunk of fc rows),
  with a dense int32 weight block;
* per-row column lists for channel-wise layers (sum pooling);
* extras: CSR entries reading the *round input* (the residual skip rows);
* bias: int64 per output row, folded in on the body lanes via the
  extracted encryption of 1 (reference model.py:425-428).

Because W2 (W1 X + b1 u) + b2 u == (W2 W1) X + (W2 b1 + b2) u exactly mod
2^53, evaluating the passes in sequence yields bit-identical rows to the
reference's single composed matrix.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np

LAYER_KINDS = ("conv2d", "fully_connected", "avg_pool", "residual_add", "flatten")
ROWS_PER_GROUP = 16
CONV_BLOCK = int(os.environ.get("SFHR_CONV_BLOCK", "2"))  # conv output pixels lowered in 2x2 blocks


class ModelError(Exception):
    pass


@dataclass
class LayerSpec:
    kind: str
    weight: Optional[np.ndarray] = None   # conv: (kh, kw, cin, cout); fc: (out, in)
    bias: Optional[np.ndarray] = None
    stride: int = 1
    padding: int = 0
    pool: int = 2
    in_shape: Optional[tuple] = None
    weight_bits: int = 4
    act_bits: int = 2
    activation: Optional[str] = None
    eta: int = 1
    clip: tuple = (0, 3)
    skip_source: int = -1

    def out_shape(self):
        if self.kind == "conv2d":
            h, w, _ = self.in_shape
            kh, kw, _, cout = self.weight.shape
            return ((h + 2 * self.padding - kh) // self.stride + 1,
                    (w + 2 * self.padding - kw) // self.stride + 1, cout)
        if self.kind == "avg_pool":
            h, w, c = self.in_shape
            return (h // self.pool, w // self.pool, c)
        if self.kind == "fully_connected":
            return (self.weight.shape[0],)
        return self.in_shape


@dataclass
class RoundSpec:
    layers: list
    input_len: int
    output_len: int
    activation: Optional[str]
    eta: int
    clip: tuple
    skip_source: int = -1
    skip_len: int = 0
    final: bool = False


def _flat(shape) -> int:
    n = 1
    for s in shape:
        n *= int(s)
    return n


@dataclass
class QuantModel:
    layers: list
    input_shape: tuple
    num_classes: int
    acc_bits: int
    input_clip: tuple = (0, 3)
    version: int = 1
    rounds: list = field(default_factory=list)

    def __post_init__(self):
        if not self.rounds:
            self.rounds = build_rounds(self)
        validate_accumulator(self)


def build_rounds(model) -> list:
    """Group layers into rounds closed by an activation (reference model.py:96-121)."""
    rounds, cur = [], []
    layers = model.layers
    for idx, L in enumerate(layers):
        cur.append(idx)
        last = idx == len(layers) - 1
        if L.activation is not None or last:
            first = layers[cur[0]]
            in_len = _flat(first.in_shape) if first.in_shape else first.weight.shape[1]
            src, slen = -1, 0
            for li in cur:
                if layers[li].kind == "residual_add":
                    src, slen = layers[li].skip_source, _flat(layers[li].in_shape)
            rounds.append(RoundSpec(cur, in_len + slen, _flat(L.out_shape()), L.activation,
                                    L.eta, tuple(L.clip), src, slen, last))
            cur = []
    return rounds


def _acc_limit(bits):
    return (1 << (bits - 1)) - 1


def _round_in_max(model, r, skip=None):
    if skip is not None:
        src = model.rounds[skip].clip if skip >= 0 else model.input_clip
        return max(abs(src[0]), abs(src[1]))
    if r == 0:
        return max(abs(model.input_clip[0]), abs(model.input_clip[1]))
    prev = model.rounds[r - 1]
    return max(abs(prev.clip[0]), abs(prev.clip[1]))


def validate_accumulator(model) -> None:
    """Worst-case L1 accumulator bound (reference model.py:246-287)."""
    lim = _acc_limit(model.acc_bits)
    for L in model.layers:
        if L.weight is not None:
            wmax = (1 << (L.weight_bits - 1)) - 1
            if np.abs(L.weight).max(initial=0) > wmax:
                raise ModelError(f"{L.kind} weight exceeds declared {L.weight_bits}-bit width")
    for r, rnd in enumerate(model.rounds):
        cur = _round_in_max(model, r)
        for li in rnd.layers:
            L = model.layers[li]
            bmax = int(np.abs(L.bias).max()) if L.bias is not None else 0
            if L.kind == "conv2d":
                co = L.weight.shape[3]
                cur = int(np.abs(L.weight).reshape(-1, co).sum(axis=0).max()) * cur + bmax
            elif L.kind == "fully_connected":
                cur = int(np.abs(L.weight).sum(axis=1).max(initial=0)) * cur + bmax
            elif L.kind == "avg_pool":
                cur = cur * L.pool * L.pool
            elif L.kind == "residual_add":
                cur = cur + _round_in_max(model, r, skip=L.skip_source)
            if cur > lim:
                raise ModelError(
                    f"worst-case accumulator {cur} exceeds 2^{model.acc_bits - 1} - 1 in round {r}")


def with_acc_bits(model: QuantModel, bits: int) -> QuantModel:
    return QuantModel(layers=model.layers, input_shape=model.input_shape,
                      num_classes=model.num_classes, acc_bits=bits,
                      input_clip=model.input_clip, version=model.version)


def save_model(model: QuantModel, json_path, blob_path=None) -> None:
    """JSON manifest + little-endian int32 blob (reference model.py:436-478)."""
    json_path = Path(json_path)
    blob_path = Path(blob_path) if blob_path else json_path.with_suffix(".bin")
    blob = bytearray()
    metas = []
    for L in model.layers:
        m = {"kind": L.kind, "stride": L.stride, "padding": L.padding, "pool": L.pool,
             "in_shape": list(L.in_shape) if L.in_shape else None,
             "weight_bits": L.weight_bits, "act_bits": L.act_bits,
             "activation": L.activation, "eta": L.eta, "clip": list(L.clip),
             "skip_source": L.skip_source}
        for name in ("weight", "bias"):
            arr = getattr(L, name)
            if arr is None:
                m[name] = None
                continue
            raw = np.ascontiguousarray(arr, dtype="<i4").tobytes()
            m[name] = {"offset": len(blob), "length": len(raw), "shape": list(arr.shape)}
            blob.extend(raw)
        metas.append(m)
    man = {"version": model.version, "accumulator_bits": model.acc_bits,
           "input_shape": list(model.input_shape), "input_clip": list(model.input_clip),
           "num_classes": model.num_classes, "weights_blob": blob_path.name, "layers": metas}
    json_path.write_text(json.dumps(man, indent=1, sort_keys=True) + "\n")
    blob_path.write_bytes(bytes(blob))


def load_model(json_path) -> QuantModel:
    """Inverse of save_model (reference model.py:481-508)."""
    json_path = Path(json_path)
    man = json.loads(json_path.read_text())
    if "version" not in man:
        raise ModelError("model manifest missing mandatory version field")
    blob = (json_path.parent / man["weights_blob"]).read_bytes()
    layers = []
    for m in man["layers"]:
        if m["kind"] not in LAYER_KINDS:
            raise ModelError(f"unknown layer kind {m['kind']!r}")
        arrs = {}
        for name in ("weight", "bias"):
            ref = m[name]
            arrs[name] = None if ref is None else np.frombuffer(
                blob[ref["offset"]:ref["offset"] + ref["length"]], dtype="<i4"
            ).astype(np.int64).reshape(ref["shape"])
        layers.append(LayerSpec(kind=m["kind"], weight=arrs["weight"], bias=arrs["bias"],
                                stride=m["stride"], padding=m["padding"], pool=m["pool"],
                                in_shape=tuple(m["in_shape"]) if m["in_shape"] else None,
                                weight_bits=m["weight_bits"], act_bits=m["act_bits"],
                                activation=m["activation"], eta=m["eta"],
                                clip=tuple(m["clip"]), skip_source=m["skip_source"]))
    return QuantModel(layers=layers, input_shape=tuple(man["input_shape"]),
                      num_classes=man["num_classes"], acc_bits=man["accumulator_bits"],
                      input_clip=tuple(man.get("input_clip", (0, 3))), version=man["version"])


# ---------------------------------------------------------------------------
# lowering to device passes


@dataclass
class LinearPass:
    """One linear map over ciphertext rows: out = W @ in (+ extras) (+ bias*unit).

    groups: (G, 6) int32 rows [cols_off, ncols, w_off, rows_off, nrows, per_row_cols]
      - per_row_cols == 0: the nrows (<= 16) rows share cols[cols_off : cols_off+ncols]
      - per_row_cols == 1: row i uses cols[cols_off + i*ncols : ... + ncols]
      weight of (row i, col c) = weights[w_off + c*16 + i]   ([ncols][16] block)
    cols: int32 input-row index into this pass's input (-1 = absent / zero padding)
    rows: int32 canonical output row of each group row
    ex_ptr/ex_col/ex_w: CSR extras (length out_len+1) into the ROUND input
    bias: int64 (out_len,) or None
    """
    in_len: int
    out_len: int
    groups: np.ndarray
    cols: np.ndarray
    weights: np.ndarray
    rows: np.ndarray
    ex_ptr: Optional[np.ndarray] = None
    ex_col: Optional[np.ndarray] = None
    ex_w: Optional[np.ndarray] = None
    bias: Optional[np.ndarray] = None

    def macs_per_lane(self) -> int:
        g = self.groups
        return int((g[:, 1].astype(np.int64) * g[:, 4]).sum()) + \
            (0 if self.ex_col is None else len(self.ex_col))

    def restrict_rows(self, keep: np.ndarray) -> "LinearPass":
        """Same pass computing only canonical rows with keep[row] (multi-GPU sharding)."""
        gb = _GroupBuilder()
        gb.w = [self.weights.astype(np.int64)]
        gb.nw = self.weights.size
        for c0, nc, w0, r0, nr, per in self.groups.tolist():
            rows = self.rows[r0:r0 + nr]
            sel = np.flatnonzero(keep[rows])
            if sel.size == 0:
                continue
            if sel.size == nr:
                cols = self.cols[c0:c0 + (nr * nc if per else nc)]
                gb.add(cols, w0, rows, nc, per)
                continue
            blk = self.weights[w0:w0 + nc * ROWS_PER_GROUP].reshape(nc, ROWS_PER_GROUP)[:, sel]
            woff = gb.block(blk.T)
            cols = self.cols[c0:c0 + nr * nc].reshape(nr, nc)[sel] if per else self.cols[c0:c0 + nc]
            gb.add(cols, woff, rows[sel], nc, per)
        out = gb.build(self.in_len, self.out_len, None)
        out.ex_ptr, out.ex_col, out.ex_w, out.bias = self.ex_ptr, self.ex_col, self.ex_w, self.bias
        return out


class _GroupBuilder:
    def __init__(self):
        self.groups, self.cols, self.w, self.rows = [], [], [], []
        self.ncols_total = 0
        self.nw = 0
        self.nrows = 0
        self._cache = {}

    def block(self, mat: np.ndarray, key=None) -> int:
        """Store an (nr <= 16, ncols) weight matrix as a [ncols][16] block; returns offset."""
        if key is not None and key in self._cache:
            return self._cache[key]
        mat = np.asarray(mat, np.int64)
        nr, nc = mat.shape
        if nr > ROWS_PER_GROUP:
            raise ModelError("weight block taller than a group")
        blk = np.zeros((nc, ROWS_PER_GROUP), np.int64)
        blk[:, :nr] = mat.T
        off = self.nw
        self.w.append(blk.reshape(-1))
        self.nw += blk.size
        if key is not None:
            self._cache[key] = off
        return off

    def add(self, cols, w_off, rows, ncols, per_row):
        self.groups.append((self.ncols_total, ncols, w_off, self.nrows, len(rows), per_row))
        self.cols.append(np.asarray(cols, np.int64).reshape(-1))
        self.ncols_total += self.cols[-1].size
        self.rows.append(np.asarray(rows, np.int64))
        self.nrows += len(rows)

    def build(self, in_len, out_len, bias) -> LinearPass:
        w = np.concatenate(self.w) if self.w else np.zeros(0, np.int64)
        if w.size and np.abs(w).max() >= 2 ** 31:
            raise ModelError("weight magnitude exceeds int32 range")
        if self.ncols_total >= 2 ** 31 or self.nw >= 2 ** 31:
            raise ModelError("lowered round too large for int32 offsets")

        def cat(xs):
            return np.concatenate(xs).astype(np.int32) if xs else np.zeros(0, np.int32)

        return LinearPass(in_len, out_len, np.asarray(self.groups, np.int32).reshape(-1, 6),
                          cat(self.cols), w.astype(np.int32), cat(self.rows),
                          bias=None if bias is None or not np.any(bias) else
                          np.asarray(bias, np.int64))


def _conv_pass(L: LayerSpec, in_len: int) -> LinearPass:
    h, w, ci = L.in_shape
    kh, kw, _, co = L.weight.shape
    oh, ow, _ = L.out_shape()
    s, p = L.stride, L.padding
    gb = _GroupBuilder()
    wmat = np.asarray(L.weight, np.int64).transpose(3, 0, 1, 2).reshape(co, kh * kw * ci)
    chunks = [(c0, min(co, c0 + ROWS_PER_GROUP)) for c0 in range(0, co, ROWS_PER_GROUP)]
    offs = [gb.block(wmat[c0:c1]) for c0, c1 in chunks]
    ky, kx, cc = np.meshgrid(np.arange(kh), np.arange(kw), np.arange(ci), indexing="ij")
    ky, kx, cc = ky.reshape(-1), kx.reshape(-1), cc.reshape(-1)
    # output pixels in CONV_BLOCK x CONV_BLOCK blocks (raster inside a block): consecutive groups
    # then have overlapping input windows, which the tensor-core tiler merges (linear.split_mma_tiles)
    blk = CONV_BLOCK
    order = [(oy, ox) for by in range(0, oh, blk) for bx in range(0, ow, blk)
             for oy in range(by, min(oh, by + blk)) for ox in range(bx, min(ow, bx + blk))]
    for oy, ox in order:
        iy, ix = oy * s + ky - p, ox * s + kx - p
        ok = (iy >= 0) & (iy < h) & (ix >= 0) & (ix < w)
        cols = np.where(ok, (iy * w + ix) * ci + cc, -1)
        base = (oy * ow + ox) * co
        for (c0, c1), off in zip(chunks, offs):
            gb.add(cols, off, np.arange(base + c0, base + c1), cols.size, 0)
    bias = None
    if L.bias is not None:
        bias = np.tile(np.asarray(L.bias, np.int64), oh * ow)
    return gb.build(in_len, oh * ow * co, bias)


def _pool_pass(L: LayerSpec, in_len: int) -> LinearPass:
    h, w, c = L.in_shape
    k = L.pool
    oh, ow = h // k, w // k
    gb = _GroupBuilder()
    w_off = gb.block(np.ones((ROWS_PER_GROUP, k * k), np.int64))
    dy, dx = np.meshgrid(np.arange(k), np.arange(k), indexing="ij")
    dy, dx = dy.reshape(-1), dx.reshape(-1)
    ch = np.arange(c)
    for oy in range(oh):
        for ox in range(ow):
            pix = ((oy * k + dy) * w + ox * k + dx)
            base = (oy * ow + ox) * c
            for c0 in range(0, c, ROWS_PER_GROUP):
                cs = ch[c0:c0 + ROWS_PER_GROUP]
                gb.add(pix[None, :] * c + cs[:, None], w_off, base + cs, k * k, 1)
    return gb.build(in_len, oh * ow * c, None)


def _fc_pass(L: LayerSpec, in_len: int) -> LinearPass:
    W = np.asarray(L.weight, np.int64)
    n_out, n_in = W.shape
    if n_in != in_len:
        raise ModelError(f"fc expects {n_in} inputs, got {in_len}")
    gb = _GroupBuilder()
    cols = np.arange(n_in)
    for r0 in range(0, n_out, ROWS_PER_GROUP):
        r = np.arange(r0, min(n_out, r0 + ROWS_PER_GROUP))
        gb.add(cols, gb.block(W[r]), r, n_in, 0)
    return gb.build(in_len, n_out, L.bias)


def _identity_pass(n: int) -> LinearPass:
    gb = _GroupBuilder()
    w_off = gb.block(np.ones((ROWS_PER_GROUP, 1), np.int64))
    for r0 in range(0, n, ROWS_PER_GROUP):
        r = np.arange(r0, min(n, r0 + ROWS_PER_GROUP))
        gb.add(r[:, None], w_off, r, 1, 1)
    return gb.build(n, n, None)


def lower_round(model, r: int) -> list:
    """Passes whose sequential evaluation equals round_matrix(model, r) exactly."""
    rnd = model.rounds[r]
    E = rnd.input_len
    main = E - rnd.skip_len
    passes: list[LinearPass] = []
    cur_len = main
    for li in rnd.layers:
        L = model.layers[li]
        if L.kind == "flatten":
            continue
        if L.kind == "residual_add":
            n = _flat(L.in_shape)
            if cur_len != n:
                raise ModelError("residual branches have mismatched shapes")
            if not passes:
                passes.append(_identity_pass(cur_len))
            ps = passes[-1]
            if ps.ex_ptr is None:
                ps.ex_ptr = np.arange(n + 1, dtype=np.int32)
                ps.ex_col = (E - rnd.skip_len + np.arange(n)).astype(np.int32)
                ps.ex_w = np.ones(n, np.int32)
            else:  # a second residual in the same round: merge CSR rows
                ptr, col, w = ps.ex_ptr, ps.ex_col, ps.ex_w
                new_col, new_w, new_ptr = [], [], [0]
                for o in range(n):
                    new_col.extend(col[ptr[o]:ptr[o + 1]].tolist() + [E - rnd.skip_len + o])
                    new_w.extend(w[ptr[o]:ptr[o + 1]].tolist() + [1])
                    new_ptr.append(len(new_col))
                ps.ex_ptr = np.asarray(new_ptr, np.int32)
                ps.ex_col = np.asarray(new_col, np.int32)
                ps.ex_w = np.asarray(new_w, np.int32)
            continue
        if L.kind == "conv2d":
            ps = _conv_pass(L, cur_len)
        elif L.kind == "avg_pool":
            ps = _pool_pass(L, cur_len)
        elif L.kind == "fully_connected":
            ps = _fc_pass(L, cur_len)
        else:
            raise ModelError(f"layer kind {L.kind!r} has no matrix form")
        if ps.in_len != cur_len:
            raise ModelError("layer input size mismatch")
        passes.append(ps)
        cur_len = ps.out_len
    if not passes:
        passes.append(_identity_pass(main))
    if passes[-1].out_len != rnd.output_len:
        raise ModelError("round output length mismatch")
    return passes


def dense_round_matrix(model, r: int):
    """Dense (W, bias) of a round from its passes (tests/small models only)."""
    rnd = model.rounds[r]
    E = rnd.input_len
    main = E - rnd.skip_len
    W = np.zeros((main, E), np.int64)
    W[:, :main] = np.eye(main, dtype=np.int64)
    bias = np.zeros(main, np.int64)
    for ps in lower_round(model, r):
        P = np.zeros((ps.out_len, ps.in_len), np.int64)
        for g in ps.groups:
            c0, nc, w0, r0, nr, per = (int(x) for x in g)
            blk = ps.weights[w0:w0 + nc * ROWS_PER_GROUP].reshape(nc, ROWS_PER_GROUP)
            for i in range(nr):
                o = int(ps.rows[r0 + i])
                cl = ps.cols[c0 + (i * nc if per else 0): c0 + (i * nc if per else 0) + nc]
                wv = blk[:, i]
                for c, wt in zip(cl, wv):
                    if c >= 0:
                        P[o, c] += wt
        newW = P @ W
        newb = P @ bias + (ps.bias if ps.bias is not None else 0)
        if ps.ex_ptr is not None:
            for o in range(ps.out_len):
                for j in range(ps.ex_ptr[o], ps.ex_ptr[o + 1]):
                    newW[o, ps.ex_col[j]] += ps.ex_w[j]
        W, bias = newW, newb
    return W, bias
