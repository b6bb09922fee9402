#!/usr/bin/env python
"""Primitive microbenchmarks (BASELINE.json configs[1]) on one B200.

Sections (one JSON line per measurement, then a summary line):

* ntt   — standalone RNS negacyclic NTT (csrc/ntt64.cu): forward and inverse
          over (batch, L, N) u64 residues of ~50-bit primes, N in {2^14, 2^15,
          2^16}, L in {4, 8, 16}, batch in {1, 64, 1024}.  "NTT GB/s" =
          algorithmic bytes 16 * N * L * batch (read + write every residue
          once) / kernel time, also as a fraction of the measured HBM peak.
* ks    — key switching at the reference's rings (b = 8/12/16, gamma = 0):
          switch_batch over B in {1, 8, 64, 256, 1024} uniform ciphertexts,
          KS/s and GB/s at 32 N bytes per switch (SURVEY §8(d) roofline row).
* hoist — 32 hoisted rotations of one 64-ciphertext batch: the fused stage
          kernel (one read of x, up to 8 automorphism+switches accumulated in
          the NTT domain per launch) vs 32 separate automorphism + switch_batch
          calls.
* mac   — ct x pt multiply-accumulate over 64 plaintexts: int_matmul_mod_q
          with a 64 x 64 integer matrix over 64 ciphertext rows (tensor cores).
* extract — partial_extract of a full chunk (N rows).
* client  — the client's s * a key product for one ResNet-20 inference's packs on the GPU
          (client_ops.KeyMul) vs the reference's float64-limb algorithm on the host.

Timing: CUDA events on the launching stream, warm-up first, L2 flushed
(256 MiB write) before every timed launch; inputs are seeded uniform residues
resident in HBM.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def _peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 7700.0, "B200_PROFILING.md fallback"


class Timer:
    def __init__(self):
        import torch
        self.torch = torch
        self.flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")

    def __call__(self, fn, reps=5, warm=2):
        torch = self.torch
        for _ in range(warm):
            fn()
        times = []
        for _ in range(reps):
            self.flush.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        return float(np.median(times))  # ms


def bench_ntt(tm, quick):
    import torch
    from paper_2509_01253_b200.ntt import RnsNtt
    peak, src = _peak()
    out = []
    for logn in (14, 15, 16):
        for L in (4, 8, 16):
            pl = RnsNtt(logn, L, 50, device=0)
            P = torch.tensor(pl.primes.view(np.int64), device="cuda")
            for batch in ((1, 64) if quick else (1, 64, 1024)):
                n = 1 << logn
                if batch * L * n * 8 > (16 << 30):
                    continue
                g = torch.Generator(device="cuda").manual_seed(logn * 100 + L)
                x = torch.randint(0, 1 << 62, (batch, L, n), device="cuda", generator=g, dtype=torch.int64)
                x = torch.remainder(x, P[None, :, None])
                ref = x.clone()
                byts = 16 * n * L * batch
                for kind in ("forward", "inverse"):
                    fn = (lambda: pl.forward(x)) if kind == "forward" else (lambda: pl.inverse(x))
                    ms = tm(fn, reps=5 if batch < 1024 else 3)
                    gbs = byts / ms / 1e6
                    out.append({"section": "ntt", "op": kind, "N": n, "L": L, "batch": batch,
                                "ms": round(ms, 4), "GB/s": round(gbs, 1),
                                "transforms/s": round(batch * L / ms * 1e3, 1),
                                "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak,
                                             "unit": "GB/s", "frac": round(gbs / peak, 4),
                                             "peak_source": src}})
                    print(json.dumps(out[-1]), flush=True)
                # forward/inverse counts are odd-even balanced only when equal: restore
                pl.forward(x)
                pl.inverse(x)
                del ref, x
            pl.close()
    return out


def _ksk(sch, seed):
    from paper_2509_01253_b200.engine import required_ksk_indices
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet, RlweCiphertext
    rng = np.random.default_rng(seed)
    R = sch.ring
    keys = {d: [RlweCiphertext(rng.integers(0, 1 << 53, R.N, dtype=np.uint64),
                               rng.integers(0, 1 << 53, R.N, dtype=np.uint64)) for _ in range(sch.gadget.l)]
            for d in required_ksk_indices(sch)}
    return KeySwitchKeySet(keys=keys, gadget=sch.gadget, delta=0.0, params=R)


def bench_ks(tm, quick):
    import torch
    from paper_2509_01253_b200.keyswitch import KeySwitchEngine
    from paper_2509_01253_b200.params import preset_for_bits
    peak, src = _peak()
    out = []
    for b in (8, 12, 16):
        sch = preset_for_bits(b, 0)
        R = sch.ring
        eng = KeySwitchEngine(_ksk(sch, b), gamma=0)
        idx = sorted(eng.key.indices)
        d = idx[len(idx) // 2]
        for B in ((1, 64, 1024) if quick else (1, 8, 64, 256, 1024)):
            g = torch.Generator(device="cuda").manual_seed(B)
            x = torch.randint(0, 1 << 53, (B, 2, R.N), device="cuda", generator=g, dtype=torch.int64)
            ms = tm(lambda: eng.switch_batch(x, d))
            gbs = B * 32 * R.N / ms / 1e6
            out.append({"section": "ks", "b": b, "M": R.M, "N": R.N, "D": sch.gadget.D, "l": sch.gadget.l,
                        "batch": B, "ms": round(ms, 4), "KS/s": round(B / ms * 1e3, 1),
                        "GB/s": round(gbs, 2), "hbm_frac": round(gbs / peak, 5)})
            print(json.dumps(out[-1]), flush=True)
        # 32 hoisted rotations of one 64-ct batch
        B = 64
        x = torch.randint(0, 1 << 53, (B, 2, R.N), device="cuda", dtype=torch.int64)
        rots = [idx[i % len(idx)] for i in range(32)]
        groups = [rots[i:i + 8] for i in range(0, 32, 8)]
        ms_h = tm(lambda: [eng.stage_batch(x, [1] + grp) for grp in groups])
        ms_u = tm(lambda: [eng.switch_batch(eng.automorphism_batch(x, r), r) for r in rots])
        out.append({"section": "hoist", "b": b, "batch": B, "rotations": 32,
                    "hoisted_ms": round(ms_h, 4), "unhoisted_ms": round(ms_u, 4),
                    "hoisted_KS/s": round(32 * B / ms_h * 1e3, 1), "unhoisted_KS/s": round(32 * B / ms_u * 1e3, 1)})
        print(json.dumps(out[-1]), flush=True)
        # ct x pt MAC over 64 plaintexts
        from paper_2509_01253_b200.linear import int_matmul_mod_q
        W = np.random.default_rng(5).integers(-7, 8, (64, 64))
        rows = torch.randint(0, 1 << 53, (64, 2, R.N), device="cuda", dtype=torch.int64)
        ms = tm(lambda: int_matmul_mod_q(W, rows))
        out.append({"section": "mac", "b": b, "shape": [64, 64], "lanes": 2 * R.N, "ms": round(ms, 4),
                    "ct_pt_MAC/s": round(64 * 64 / ms * 1e3, 1)})
        print(json.dumps(out[-1]), flush=True)
        # partial extraction of a full chunk
        from paper_2509_01253_b200.tracepack import extract_device, power_exponents
        exps = power_exponents(0, R)
        power = torch.randint(0, 1 << 53, (1, len(exps), 2, R.N), device="cuda", dtype=torch.int64)
        ms = tm(lambda: extract_device(eng.ctx, power, exps, R.N))
        out.append({"section": "extract", "b": b, "rows": R.N, "ms": round(ms, 4),
                    "rows/s": round(R.N / ms * 1e3, 1), "GB/s": round(16 * R.N * R.N / ms / 1e6, 1)})
        print(json.dumps(out[-1]), flush=True)
    return out


def bench_client(tm):
    """Client-side key product s * a for the packs of one ResNet-20 inference (645 polys, b=12):
    the GPU operator (tcgen05 linear map, host copies included) vs the reference algorithm
    (three float64 limb GEMMs, numpy/BLAS on the host)."""
    import time
    from oracle import keyswitch as oks
    from oracle import scheme as osc
    from paper_2509_01253_b200.client_ops import KeyMul
    from paper_2509_01253_b200.params import RingParams
    R = osc.preset(12, 0).ring
    sk = oks.keygen(R, "binary", seed=1)
    km = KeyMul(sk.s, RingParams(R.t, R.alpha, R.p_bits))
    v = np.random.default_rng(0).integers(0, 1 << 53, (645, R.N), dtype=np.uint64)
    km.times(v)
    t0 = time.perf_counter()
    got = km.times(v)
    t_gpu = time.perf_counter() - t0
    oks.key_times(sk, v[:1])
    t0 = time.perf_counter()
    want = oks.key_times(sk, v)
    t_cpu = time.perf_counter() - t0
    assert np.array_equal(got, want)
    out = {"section": "client", "op": "s*a mod Phi_M, 645 polys, b=12", "gpu_s": round(t_gpu, 4),
           "cpu_reference_algorithm_s": round(t_cpu, 4)}
    print(json.dumps(out), flush=True)
    return [out]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sections", default="ntt,ks,client")
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    import torch
    assert torch.cuda.is_available(), "bench_primitives needs a GPU"
    tm = Timer()
    res = []
    if "ntt" in a.sections:
        res += bench_ntt(tm, a.quick)
    if "ks" in a.sections:
        res += bench_ks(tm, a.quick)
    if "client" in a.sections:
        res += bench_client(tm)
    ntt = [r for r in res if r["section"] == "ntt" and r["batch"] >= 64]
    summ = {"summary": "primitives", "ntt_best_GB/s": max((r["GB/s"] for r in ntt), default=None),
            "ntt_best_frac": max((r["roofline"]["frac"] for r in ntt), default=None),
            "ks_best_KS/s": max((r["KS/s"] for r in res if r["section"] == "ks"), default=None)}
    print(json.dumps(summ), flush=True)


if __name__ == "__main__":
    main()
