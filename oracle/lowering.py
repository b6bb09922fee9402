"""Oracle: quantized model semantics, round lowering, encrypted linear map.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Layers/models are duck-typed: any object exposing the reference LayerSpec
attributes (kind, weight, bias, stride, padding, pool, in_shape, activation,
eta, clip, skip_source, weight_bits) works; rounds are rebuilt here.

Restates:
  * _build_rounds                                reference model.py:96-121
  * conv / sum-pool / fc / residual semantics     reference model.py:127-170
  * requantize / relu / cleartext_forward         reference model.py:173-243
  * validate_accumulator                          reference model.py:246-287
  * layer_matrix / round_matrix (dense, small)    reference model.py:290-353
  * int_matmul_mod_q / encrypted_linear           reference model.py:384-429
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .scheme import MASK, U64, UMASK


class OracleModelError(Exception):
    pass


@dataclass
class Round:
    layers: list
    input_len: int
    output_len: int
    activation: object
    eta: int
    clip: tuple
    skip_source: int = -1
    skip_len: int = 0
    final: bool = False


def _flat(shape):
    n = 1
    for s in shape:
        n *= s
    return n


def out_shape(L):
    if L.kind == "conv2d":
        h, w, _ = L.in_shape
        kh, kw, _, co = L.weight.shape
        return ((h + 2 * L.padding - kh) // L.stride + 1,
                (w + 2 * L.padding - kw) // L.stride + 1, co)
    if L.kind == "avg_pool":
        h, w, c = L.in_shape
        return (h // L.pool, w // L.pool, c)
    if L.kind == "fully_connected":
        return (L.weight.shape[0],)
    return L.in_shape


def build_rounds(layers) -> list[Round]:
    rounds, cur = [], []
    for idx, L in enumerate(layers):
        cur.append(idx)
        last_layer = idx == len(layers) - 1
        if L.activation is not None or last_layer:
            first = layers[cur[0]]
            in_len = _flat(first.in_shape) if first.in_shape else first.weight.shape[1]
            src, slen = -1, 0
            for li in cur:
                if layers[li].kind == "residual_add":
                    src, slen = layers[li].skip_source, _flat(layers[li].in_shape)
            rounds.append(Round(cur, in_len + slen, _flat(out_shape(L)), L.activation,
                                L.eta, tuple(L.clip), src, slen, last_layer))
            cur = []
    return rounds


# ---------------------------------------------------------------------------
# cleartext integer semantics


def _conv(x, L):
    h, w, ci = L.in_shape
    kh, kw, _, co = L.weight.shape
    p, s = L.padding, L.stride
    xp = np.zeros((h + 2 * p, w + 2 * p, ci), np.int64)
    xp[p:p + h, p:p + w] = x.reshape(h, w, ci)
    oh, ow, _ = out_shape(L)
    out = np.zeros((oh, ow, co), np.int64)
    wt = L.weight.astype(np.int64)
    for ky in range(kh):
        for kx in range(kw):
            patch = xp[ky:ky + s * oh:s, kx:kx + s * ow:s]  # (oh, ow, ci)
            out += patch @ wt[ky, kx]
    if L.bias is not None:
        out += np.asarray(L.bias, np.int64)
    return out.reshape(-1)


def run_layer(x, L, round_in):
    if L.kind == "conv2d":
        return _conv(x, L)
    if L.kind == "avg_pool":
        h, w, c = L.in_shape
        k = L.pool
        return x.reshape(h // k, k, w // k, k, c).sum(axis=(1, 3)).reshape(-1)
    if L.kind == "flatten":
        return x
    if L.kind == "fully_connected":
        out = L.weight.astype(np.int64) @ x
        return out + (np.asarray(L.bias, np.int64) if L.bias is not None else 0)
    if L.kind == "residual_add":
        return x + round_in[-_flat(L.in_shape):]
    raise OracleModelError(f"unknown layer kind {L.kind!r}")


def requantize(y, eta, clip):
    y = np.asarray(y)
    if float(eta) == int(eta):
        e = int(eta)
        q = np.sign(y) * ((2 * np.abs(y.astype(np.int64)) + e) // (2 * e))
    else:
        q = np.sign(y) * np.floor(np.abs(y) / float(eta) + 0.5)
    return np.clip(q.astype(np.int64), clip[0], clip[1])


def activation(v, spec):
    if spec is None:
        return v
    if spec == "relu":
        return np.maximum(v, 0)
    raise OracleModelError(f"unknown activation {spec!r}")


def round_linear(layers, rnd: Round, v_in, acc_bits):
    lim = (1 << (acc_bits - 1)) - 1
    cur = (v_in[:rnd.input_len - rnd.skip_len] if rnd.skip_len else v_in).astype(np.int64)
    for li in rnd.layers:
        cur = run_layer(cur, layers[li], v_in.astype(np.int64))
        if np.abs(cur).max(initial=0) > lim:
            raise OracleModelError("accumulator overflow")
    return cur


def cleartext_forward(model, x):
    """Golden integer forward pass -> logits (model.py:223-243)."""
    layers = model.layers
    rounds = build_rounds(layers)
    v = np.asarray(x, np.int64).reshape(-1)
    trace = []
    for rnd in rounds:
        if rnd.skip_len:
            skip = trace[rnd.skip_source][1] if rnd.skip_source >= 0 else np.asarray(x).reshape(-1)
            v = np.concatenate([v, skip.astype(np.int64)])
        y = round_linear(layers, rnd, v, model.acc_bits)
        if rnd.final:
            return y
        v = requantize(activation(y, rnd.activation), rnd.eta, rnd.clip)
        trace.append((y, v))
    raise OracleModelError("model has no rounds")


# ---------------------------------------------------------------------------
# lowering to integer matrices (dense; for small models only)


def layer_matrix(L):
    if L.kind == "conv2d":
        h, w, ci = L.in_shape
        kh, kw, _, co = L.weight.shape
        oh, ow, _ = out_shape(L)
        W = np.zeros((oh * ow * co, h * w * ci), np.int64)
        bvec = np.zeros(oh * ow * co, np.int64)
        for oy in range(oh):
            for ox in range(ow):
                o0 = (oy * ow + ox) * co
                for ky in range(kh):
                    for kx in range(kw):
                        iy, ix = oy * L.stride + ky - L.padding, ox * L.stride + kx - L.padding
                        if 0 <= iy < h and 0 <= ix < w:
                            i0 = (iy * w + ix) * ci
                            W[o0:o0 + co, i0:i0 + ci] = np.asarray(L.weight[ky, kx]).T
                if L.bias is not None:
                    bvec[o0:o0 + co] = L.bias
        return W, bvec
    if L.kind == "avg_pool":
        h, w, c = L.in_shape
        k = L.pool
        W = np.zeros(((h // k) * (w // k) * c, h * w * c), np.int64)
        for oy in range(h // k):
            for ox in range(w // k):
                for ch in range(c):
                    o = (oy * (w // k) + ox) * c + ch
                    for dy in range(k):
                        for dx in range(k):
                            W[o, ((oy * k + dy) * w + ox * k + dx) * c + ch] = 1
        return W, np.zeros(W.shape[0], np.int64)
    if L.kind == "fully_connected":
        bvec = (np.asarray(L.bias, np.int64) if L.bias is not None
                else np.zeros(L.weight.shape[0], np.int64))
        return np.asarray(L.weight, np.int64), bvec
    raise OracleModelError(f"layer kind {L.kind!r} has no matrix form")


def round_matrix(layers, rnd: Round):
    """(W, bias) with round_out = W @ round_in + bias (model.py:332-353)."""
    E = rnd.input_len
    main = E - rnd.skip_len
    W = np.zeros((main, E), np.int64)
    W[:, :main] = np.eye(main, dtype=np.int64)
    bias = np.zeros(main, np.int64)
    for li in rnd.layers:
        L = layers[li]
        if L.kind == "flatten":
            continue
        if L.kind == "residual_add":
            n = _flat(L.in_shape)
            if W.shape[0] != n:
                raise OracleModelError("residual branches have mismatched shapes")
            W[:, E - rnd.skip_len:] += np.eye(n, dtype=np.int64)
            continue
        lw, lb = layer_matrix(L)
        bias = lw @ bias + lb
        W = lw @ W
    return W, bias


# ---------------------------------------------------------------------------
# ciphertext rows


def int_matmul_mod_q(W, rows):
    """Exact W @ rows mod 2^53 with three 18-bit float64 limbs (model.py:384-407)."""
    e_out, e_in = W.shape
    flat = rows.reshape(rows.shape[0], -1)
    if float(np.abs(W).max(initial=0)) * e_in * (1 << 18) >= 2 ** 53:
        raise OracleModelError("weight magnitude too large for exact lane combination")
    density = np.count_nonzero(W) / max(1, W.size)
    if density < 0.125 and W.size > 65536:   # reference model.py:395-399
        from scipy.sparse import csr_matrix
        Wf = csr_matrix(W.astype(np.float64))
    else:
        Wf = W.astype(np.float64)
    acc = np.zeros((e_out, flat.shape[1]), U64)
    for k in range(3):
        limb = ((flat >> U64(18 * k)) & U64((1 << 18) - 1)).astype(np.float64)
        acc += np.rint(Wf @ limb).astype(np.int64).astype(U64) << U64(18 * k)
    acc &= UMASK
    return acc.reshape((e_out,) + rows.shape[1:])


def encrypted_linear(W, bias, rows, unit):
    """model.py:410-429."""
    if W.shape[1] != rows.shape[0]:
        raise OracleModelError(f"round matrix expects {W.shape[1]} rows, got {rows.shape[0]}")
    out = int_matmul_mod_q(W, rows)
    if bias is not None and np.any(bias):
        body = (np.asarray(bias, np.int64).astype(U64)[:, None] * unit[None, :]) & UMASK
        out[:, 1] = (out[:, 1] + body) & UMASK
    return out


def int_matmul_exact_objects(W, rows):
    """Python-int oracle of W @ rows mod 2^53 (reference tests/test_model.py:170-181)."""
    out = np.zeros((W.shape[0],) + rows.shape[1:], U64)
    R = rows.astype(object)
    for o in range(W.shape[0]):
        acc = np.zeros(rows.shape[1:], dtype=object)
        for i in range(W.shape[1]):
            if W[o, i]:
                acc = acc + int(W[o, i]) * R[i]
        out[o] = (acc % (1 << 53)).astype(U64)
    return out


assert MASK == (1 << 53) - 1
