"""Tensor-core (tcgen05 kind::i8) linear map: host tiling on CPU, device parity on GPU.

The device kernel (csrc/linear_mma.cu) computes out[o][u] = sum_j D[8u+j][o] << 8j
with D = (bytes of the gathered input rows) x (s8 weights).  The CPU tests
replay exactly that decomposition in numpy from the packed operands the host
uploads, so the packing and the byte algebra are pinned before any GPU run;
the GPU tests compare the kernel against the CUDA-core kernel and the oracle's
exact object-integer matmul (reference model.py:384-407)."""

import numpy as np
import pytest

from conftest import has_cuda, u53
from oracle import lowering as olo
from paper_2509_01253_b200 import linear as lin
from paper_2509_01253_b200 import model as mm
from paper_2509_01253_b200 import workloads as W


def _unpack(tw, n_pad, k_pad):
    return tw.reshape(k_pad // 16, n_pad // 8, 8, 16).transpose(1, 2, 0, 3).reshape(n_pad, k_pad)


def _emulate_tile(mt, t, rows_in, round_in=None):
    """numpy replay of one tile group: byte-plane int8 GEMM + recombination."""
    c0, kp, w0, r0, nr, np_, _, _ = (int(x) for x in mt.tiles[t])
    B = _unpack(mt.w[w0:w0 + np_ * kp], np_, kp).astype(np.int64)      # (N_pad, K_pad) s8
    cols = mt.cols[c0:c0 + kp]
    X = np.zeros((kp,) + rows_in.shape[1:], np.uint64)
    X[cols >= 0] = rows_in[cols[cols >= 0]]
    if np.any(cols <= -2):  # folded residual extras read the round input
        X[cols <= -2] = round_in[-(cols[cols <= -2] + 2)]
    Xb = X.reshape(kp, -1).view(np.uint8).reshape(kp, -1, 8).astype(np.int64)  # (K, lanes, 8 bytes)
    D = np.einsum("ok,klj->olj", B[:nr], Xb)                            # s32-exact accumulators
    assert np.abs(D).max(initial=0) < 2 ** 31
    out = np.zeros(D.shape[:2], np.uint64)
    for j in range(8):
        out += (D[:, :, j].astype(np.int64).astype(np.uint64) << np.uint64(8 * j))
    return mt.rows[r0:r0 + nr], out & np.uint64((1 << 53) - 1)


PASSES = {
    "resnet20_r1": lambda: mm.lower_round(W.resnet20_model(12, 0), 1),
    "resnet20_r2_residual": lambda: mm.lower_round(W.resnet20_model(12, 0), 2),
    "resnet20_r7": lambda: mm.lower_round(W.resnet20_model(12, 0), 7),
    "resnet20_fc": lambda: mm.lower_round(W.resnet20_model(12, 0), 19),
    "toy": lambda: mm.lower_round(W.toy_model(8, 3), 0),
    "toy_pool": lambda: mm.lower_round(W.toy_model(8, 3), 2),  # per-row (pooling) groups as tiles
    "mlp": lambda: mm.lower_round(W.mlp_model(0), 0),
    "dense_wide": lambda: [lin._dense_pass(np.random.default_rng(5).integers(-127, 128, (300, 45)))],
    "dense_big_w": lambda: [lin._dense_pass(np.random.default_rng(6).integers(-500, 500, (20, 8)))],
}


@pytest.mark.parametrize("name", sorted(PASSES))
def test_tiles_cover_rows_once_and_replay_exactly(name):
    rng = np.random.default_rng(9)
    for ps in PASSES[name]():
        rest, mt = lin.split_mma_tiles(ps)
        seen = []
        for gi in rest:
            c0, nc, w0, r0, nr, per = (int(x) for x in ps.groups[gi])
            seen.extend(ps.rows[r0:r0 + nr].tolist())
        if mt is not None:
            seen.extend(mt.rows.tolist())
            assert mt.tiles[:, 5].max() <= lin.MMA_MAX_ROWS
            assert np.all(mt.tiles[:, 1] % 32 == 0) and np.all(mt.tiles[:, 5] % 16 == 0)
        assert sorted(seen) == sorted(ps.rows.tolist())
        if name == "dense_big_w":
            assert mt is None  # |w| > 127 stays on the CUDA-core kernel
            continue
        if mt is None:  # per-row column lists (pooling, identity) stay on the CUDA cores
            assert np.all(ps.groups[:, 5] == 1)
            continue
        # replay a few tiles against the exact dense product of the pass
        Wd = np.zeros((ps.out_len, ps.in_len), np.int64)
        for c0, nc, w0, r0, nr, per in ps.groups.tolist():
            blk = ps.weights[w0:w0 + nc * 16].reshape(nc, 16)
            for i in range(nr):
                cl = ps.cols[c0 + (i * nc if per else 0): c0 + (i * nc if per else 0) + nc]
                for c, col in enumerate(cl):
                    if col >= 0:
                        Wd[ps.rows[r0 + i], col] += blk[c, i]
        x = rng.integers(0, 1 << 53, (ps.in_len, 2, 5), dtype=np.uint64)
        xr, We = None, None
        if ps.ex_ptr is not None:
            xr = rng.integers(0, 1 << 53, (int(ps.ex_col.max()) + 1, 2, 5), dtype=np.uint64)
            We = np.zeros((ps.out_len, len(xr)), np.int64)
            for o in range(ps.out_len):
                for e in range(ps.ex_ptr[o], ps.ex_ptr[o + 1]):
                    We[o, ps.ex_col[e]] += ps.ex_w[e]
        for t in sorted({0, len(mt.tiles) // 2, len(mt.tiles) - 1}):
            rows, got = _emulate_tile(mt, t, x, xr)
            if We is None:
                want = olo.int_matmul_exact_objects(Wd[rows], x).reshape(len(rows), -1)
            else:
                want = olo.int_matmul_exact_objects(np.concatenate([Wd[rows], We[rows]], 1),
                                                    np.concatenate([x, xr])).reshape(len(rows), -1)
            assert np.array_equal(got, want), (name, t)


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("shape", [(1, 1, 2), (16, 32, 16), (17, 33, 18), (300, 45, 30), (5, 700, 2),
                                   (64, 576, 4116), (128, 784, 100),
                                   # streamed weight operands (N_pad x K_pad > 96 KB)
                                   (256, 576, 100), (64, 4608, 18), (200, 1000, 34)])
def test_mma_matmul_matches_oracle(shape):
    e_out, e_in, lanes = shape
    rng = np.random.default_rng(sum(shape))
    w = rng.integers(-127, 128, (e_out, e_in))
    if e_in * 127 * 255 >= 2 ** 31 or float(np.abs(w).max()) * e_in * (1 << 18) >= 2 ** 53:
        w = rng.integers(-1, 2, (e_out, e_in))
    rows = u53(sum(shape) + 1, (e_in, lanes))
    ps = lin._dense_pass(w)
    _, mt = lin.split_mma_tiles(ps)
    assert mt is not None
    got = lin.int_matmul_mod_q(w, rows)
    assert np.array_equal(got, olo.int_matmul_exact_objects(w, rows))


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("net,r", [("r20", 0), ("r20", 1), ("r20", 2), ("r20", 7), ("r20", 13), ("r20", 19),
                                   ("r18", 1), ("r18", 12), ("r18", 15), ("r18", 16)])
def test_mma_round_matches_cuda_core_kernel(net, r, monkeypatch):
    """A full ResNet round map (maps, residual extras, bias) through both kernels."""
    import torch
    from paper_2509_01253_b200.device import RingContext
    from paper_2509_01253_b200.params import preset_for_bits
    b = 12 if net == "r20" else 16
    model = W.resnet20_model(12, 0) if net == "r20" else W.resnet18_model(16, 0)
    sch = preset_for_bits(b, 0)
    R = sch.ring
    ctx = RingContext.get(R.t, R.alpha, R.p_bits, sch.gadget.D, sch.gadget.l, 0, sch.beta, 0)
    rnd = model.rounds[r]
    E = rnd.input_len
    rng = np.random.default_rng(r)
    x = torch.from_numpy(rng.integers(0, 1 << 53, (E, 2, R.N), dtype=np.uint64).view(np.int64)).cuda()
    in_map = torch.from_numpy(rng.permutation(E).astype(np.int64)).cuda()
    out_map = torch.from_numpy(rng.permutation(rnd.output_len).astype(np.int64)).cuda()
    unit = torch.from_numpy(rng.integers(0, 1 << 53, R.N, dtype=np.uint64).view(np.int64)).cuda()
    passes = mm.lower_round(model, r)
    if r == 1:  # exercise the bias path as well
        passes[-1].bias = rng.integers(-5, 6, passes[-1].out_len)
    outs = []
    for enabled, tma in ((True, False), (True, True), (False, False)):
        monkeypatch.setattr(lin, "MMA_ENABLED", enabled)
        monkeypatch.setattr(lin, "MMA_TMA", tma)
        dps = [lin.DevicePass(p, ctx.dev) for p in passes]
        assert any(dp.n_mma_tiles > 0 for dp in dps) == enabled
        out = torch.zeros((rnd.output_len, 2, R.N), dtype=torch.int64, device=ctx.dev)
        lin.run_round(ctx, dps, x, in_map, out, out_map, unit)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    assert np.array_equal(outs[0], outs[2]) and np.array_equal(outs[1], outs[2])


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("run_rows,same_rows", [(16, 16), (128, 128), (256, 256)])
def test_tiler_knobs_do_not_change_results(run_rows, same_rows, monkeypatch):
    """Any tile-group merging (pixel runs, shared-list runs) gives the CUDA-core result."""
    import torch
    from paper_2509_01253_b200.device import RingContext
    from paper_2509_01253_b200.params import preset_for_bits
    model = W.resnet20_model(12, 0)
    sch = preset_for_bits(12, 0)
    R = sch.ring
    ctx = RingContext.get(R.t, R.alpha, R.p_bits, sch.gadget.D, sch.gadget.l, 0, sch.beta, 0)
    r = 2  # 16-channel 3x3 conv with a residual extra
    rnd = model.rounds[r]
    rng = np.random.default_rng(77)
    x = torch.from_numpy(rng.integers(0, 1 << 53, (rnd.input_len, 2, R.N), dtype=np.uint64).view(np.int64)).cuda()
    in_map = torch.from_numpy(rng.permutation(rnd.input_len).astype(np.int64)).cuda()
    unit = torch.from_numpy(rng.integers(0, 1 << 53, R.N, dtype=np.uint64).view(np.int64)).cuda()
    passes = mm.lower_round(model, r)
    outs = []
    for knobs in ((run_rows, same_rows, True), (64, 256, False)):
        monkeypatch.setattr(lin, "MMA_RUN_ROWS", knobs[0])
        monkeypatch.setattr(lin, "MMA_SAME_ROWS", knobs[1])
        monkeypatch.setattr(lin, "MMA_ENABLED", knobs[2])
        dps = [lin.DevicePass(p, ctx.dev) for p in passes]
        out = torch.zeros((rnd.output_len, 2, R.N), dtype=torch.int64, device=ctx.dev)
        lin.run_round(ctx, dps, x, in_map, out, None, unit)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
