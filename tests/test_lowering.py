"""The per-layer pass lowering equals the reference's dense round matrix
(oracle/lowering.round_matrix, restating reference model.py:290-353)."""

import numpy as np
import pytest

from oracle import lowering as olo
from paper_2509_01253_b200 import model as mm
from paper_2509_01253_b200 import workloads as W


def small_resnet(seed):
    return W.resnet_model([2, 1], [3, 4], 8, 3, 1, 2, 5, 12, seed, final_pool=2, fc_keep=6)


MODELS = {
    "toy8": lambda: W.toy_model(8, 3),
    "toy16": lambda: W.toy_model(16, 11),
    "small_resnet": lambda: small_resnet(1),
    "mlp_small": lambda: mm.QuantModel(
        layers=[mm.LayerSpec("fully_connected", weight=np.random.default_rng(2).integers(-7, 8, (20, 33)),
                             bias=np.random.default_rng(3).integers(-5, 6, 20), weight_bits=4,
                             activation="relu", eta=64, clip=(0, 3)),
                mm.LayerSpec("fully_connected", weight=np.random.default_rng(4).integers(-7, 8, (7, 20)),
                             weight_bits=4, clip=(-32768, 32767))],
        input_shape=(33,), num_classes=7, acc_bits=16),
}


@pytest.mark.parametrize("name", sorted(MODELS))
def test_passes_equal_dense_round_matrix(name):
    m = MODELS[name]()
    orounds = olo.build_rounds(m.layers)
    assert [(r.input_len, r.output_len, r.skip_len, r.skip_source, r.final) for r in orounds] == \
           [(r.input_len, r.output_len, r.skip_len, r.skip_source, r.final) for r in m.rounds]
    for r, orr in enumerate(orounds):
        W1, b1 = mm.dense_round_matrix(m, r)
        W0, b0 = olo.round_matrix(m.layers, orr)
        assert np.array_equal(W1, W0), (name, r)
        assert np.array_equal(b1, b0), (name, r)


def test_small_resnet_has_residual_and_pool_rounds():
    m = small_resnet(1)
    kinds = [[m.layers[i].kind for i in r.layers] for r in m.rounds]
    assert any("residual_add" in k for k in kinds)
    assert any(k[0] == "avg_pool" and "conv2d" in k for k in kinds)


def test_restrict_rows_is_a_row_subset():
    m = small_resnet(2)
    rng = np.random.default_rng(0)
    for r in range(len(m.rounds)):
        ps = mm.lower_round(m, r)[-1]
        keep = rng.random(ps.out_len) < 0.4
        sub = ps.restrict_rows(keep)
        assert set(sub.rows.tolist()) == set(np.flatnonzero(keep).tolist())


def test_resnet_workloads_validate():
    for fn in (W.resnet20_model, W.resnet18_model, W.mlp_model):
        m = fn()
        assert m.rounds[-1].final
