"""Synthetic quantized models for the BASELINE.json configs.

Datasets/checkpoints are not available (and image content does not change
server work, reference PAPER.md:470), so every model here is random-init
with the published architecture shape, quantized symmetrically per tensor,
BatchNorm folded with identity statistics (bias 0).  Forced deviations from
the named architectures (the reference supports only identity residuals of
equal shape and non-overlapping sum pooling, reference model.py:149-171):
stride-2 blocks carry no shortcut, max-pool becomes avg_pool 2, and the final
fc keeps at most ``fc_keep`` nonzeros per class so that the worst-case
accumulator bound (model.py:246-287) holds at the chosen width b.
"""

from __future__ import annotations

import numpy as np

from .model import LayerSpec, QuantModel


def _quantize(w: np.ndarray, bits: int) -> np.ndarray:
    """Symmetric per-tensor quantization; 2-bit uses the ternary threshold 0.7 * mean|w|."""
    if bits == 2:
        thr = 0.7 * np.abs(w).mean()
        return (np.sign(w) * (np.abs(w) > thr)).astype(np.int64)
    qmax = (1 << (bits - 1)) - 1
    s = np.abs(w).max() / qmax if np.abs(w).max() > 0 else 1.0
    return np.clip(np.rint(w / s), -qmax, qmax).astype(np.int64)


def _kaiming(rng, shape, fan_in):
    return rng.normal(0.0, np.sqrt(2.0 / fan_in), shape)


def toy_model(b: int, seed: int, num_classes: int = 10) -> QuantModel:
    """Random two-conv + pool + fc toy, 8x8x1 input (reference testing.py:63-86 shape).

    Draws the same seeded integers in the same order as the reference helper,
    so the same seed yields the same model.
    """
    rng = np.random.default_rng(seed)
    k1 = rng.integers(-1, 2, (3, 3, 1, 2))
    b1 = rng.integers(-2, 3, 2)
    k2 = rng.integers(-1, 2, (3, 3, 2, 2))
    b2 = rng.integers(-2, 3, 2)
    fc = rng.integers(-1, 2, (num_classes, 8))
    bf = rng.integers(-2, 3, num_classes)
    layers = [
        LayerSpec("conv2d", weight=k1, bias=b1, stride=1, padding=1, in_shape=(8, 8, 1),
                  weight_bits=2, act_bits=2, activation="relu", eta=4, clip=(0, 3)),
        LayerSpec("conv2d", weight=k2, bias=b2, stride=2, padding=1, in_shape=(8, 8, 2),
                  weight_bits=2, act_bits=2, activation="relu", eta=4, clip=(0, 3)),
        LayerSpec("avg_pool", pool=2, in_shape=(4, 4, 2)),
        LayerSpec("flatten", in_shape=(2, 2, 2)),
        LayerSpec("fully_connected", weight=fc, bias=bf, weight_bits=2, act_bits=2, eta=1,
                  clip=(-128, 127)),
    ]
    return QuantModel(layers=layers, input_shape=(8, 8, 1), num_classes=num_classes, acc_bits=b,
                      input_clip=(0, 3))


def synthetic_conv_model(b: int, side: int, channels: int = 3) -> QuantModel:
    """One 3x3 conv round (reference bench.py:78-88 shape, same seed)."""
    rng = np.random.default_rng(7)
    k = rng.integers(-1, 2, (3, 3, channels, channels))
    L = LayerSpec("conv2d", weight=k, bias=np.zeros(channels, np.int64), stride=1, padding=1,
                  in_shape=(side, side, channels), weight_bits=2, act_bits=2, eta=1,
                  clip=(-(1 << (b - 1)), (1 << (b - 1)) - 1))
    return QuantModel(layers=[L], input_shape=(side, side, channels), num_classes=1, acc_bits=b,
                      input_clip=(0, 3))


def mlp_model(seed: int = 0) -> QuantModel:
    """BASELINE config 1: MLP 784->128->10, b=16."""
    rng = np.random.default_rng(seed)
    w1 = _quantize(rng.uniform(-0.1, 0.1, (128, 784)), 4)
    w2 = _quantize(rng.uniform(-0.1, 0.1, (10, 128)), 4)
    layers = [
        LayerSpec("fully_connected", weight=w1, bias=np.zeros(128, np.int64), weight_bits=4,
                  activation="relu", eta=64, clip=(0, 3)),
        LayerSpec("fully_connected", weight=w2, bias=np.zeros(10, np.int64), weight_bits=4,
                  clip=(-32768, 32767)),
    ]
    return QuantModel(layers=layers, input_shape=(784,), num_classes=10, acc_bits=16,
                      input_clip=(0, 3))


def mlp_input(seed: int = 0) -> np.ndarray:
    x = np.random.default_rng(seed + 1).uniform(0, 1, 784)
    return np.clip(np.floor(4 * x), 0, 3).astype(np.int64)


def _conv(rng, h, w, cin, cout, k, stride, pad, act="relu", eta=64, clip=(0, 3), bits=2):
    wt = _quantize(_kaiming(rng, (k, k, cin, cout), k * k * cin), bits)
    return LayerSpec("conv2d", weight=wt, bias=np.zeros(cout, np.int64), stride=stride,
                     padding=pad, in_shape=(h, w, cin), weight_bits=bits, activation=act,
                     eta=eta, clip=clip)


def _fc_pruned(rng, n_in, n_out, keep, bits=2):
    w = _quantize(_kaiming(rng, (n_out, n_in), n_in), bits)
    if keep < n_in:
        order = np.argsort(-np.abs(w), axis=1, kind="stable")
        mask = np.zeros_like(w, dtype=bool)
        np.put_along_axis(mask, order[:, :keep], True, axis=1)
        w = np.where(mask, w, 0)
    return w


def resnet_model(depth_blocks, widths, in_hw, stem_k, stem_stride, stem_pool, num_classes, b,
                 seed, final_pool, fc_keep) -> QuantModel:
    """Generic ResNet-shaped model: rounds = stem, (conv1, conv2[+residual]) per block, final."""
    rng = np.random.default_rng(seed)
    layers = []
    h = in_hw
    cin = 3
    layers.append(_conv(rng, h, h, cin, widths[0], stem_k, stem_stride, stem_k // 2))
    h = (h + 2 * (stem_k // 2) - stem_k) // stem_stride + 1
    cin = widths[0]
    round_idx = 0
    pending_pool = stem_pool
    for si, (nb, wd) in enumerate(zip(depth_blocks, widths)):
        for bi in range(nb):
            stride = 2 if (bi == 0 and si > 0) else 1
            block_in_round = round_idx
            pooled = bool(pending_pool)
            if pending_pool:
                layers.append(LayerSpec("avg_pool", pool=pending_pool, in_shape=(h, h, cin)))
                h //= pending_pool
                pending_pool = 0
            layers.append(_conv(rng, h, h, cin, wd, 3, stride, 1))
            round_idx += 1
            h2 = (h + 2 - 3) // stride + 1
            shortcut = stride == 1 and cin == wd and not pooled
            c2 = _conv(rng, h2, h2, wd, wd, 3, 1, 1)
            if shortcut:
                c2.activation = None
                layers.append(c2)
                layers.append(LayerSpec("residual_add", in_shape=(h2, h2, wd),
                                        skip_source=block_in_round, activation="relu", eta=64,
                                        clip=(0, 3)))
            else:
                layers.append(c2)
            round_idx += 1
            h, cin = h2, wd
    layers.append(LayerSpec("avg_pool", pool=final_pool, in_shape=(h, h, cin)))
    hp = h // final_pool
    layers.append(LayerSpec("flatten", in_shape=(hp, hp, cin)))
    fc = _fc_pruned(rng, hp * hp * cin, num_classes, fc_keep)
    layers.append(LayerSpec("fully_connected", weight=fc, bias=np.zeros(num_classes, np.int64),
                            weight_bits=2, eta=1, clip=(-(1 << (b - 1)), (1 << (b - 1)) - 1)))
    return QuantModel(layers=layers, input_shape=(in_hw, in_hw, 3), num_classes=num_classes,
                      acc_bits=b, input_clip=(-3, 3))


def resnet20_model(b: int = 12, seed: int = 0) -> QuantModel:
    """BASELINE config 3: ResNet-20 shape, 3x32x32, 10 classes."""
    return resnet_model([3, 3, 3], [16, 32, 64], 32, 3, 1, 0, 10, b, seed, final_pool=8,
                        fc_keep=10)


def resnet18_model(b: int = 16, seed: int = 0) -> QuantModel:
    """BASELINE config 4: ResNet-18 shape, 3x64x64, 200 classes."""
    return resnet_model([2, 2, 2, 2], [64, 128, 256, 512], 64, 7, 2, 2, 200, b, seed,
                        final_pool=2, fc_keep=512)


def resnet34_model(b: int = 16, seed: int = 0) -> QuantModel:
    """BASELINE config 5: ResNet-34 shape, 3x224x224, 1000 classes."""
    return resnet_model([3, 4, 6, 3], [64, 128, 256, 512], 224, 7, 2, 2, 1000, b, seed,
                        final_pool=7, fc_keep=200)


def image_input(model: QuantModel, seed: int = 0) -> np.ndarray:
    """x ~ N(0,1) quantized to the input clip."""
    x = np.random.default_rng(seed).normal(0, 1, model.input_shape)
    lo, hi = model.input_clip
    return np.clip(np.rint(x), lo, hi).astype(np.int64)
