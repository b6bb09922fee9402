#!/usr/bin/env python
"""Benchmark: ResNet-20-shape hybrid inference, server side, on B200.

Workload (BASELINE.json configs[2], mapped onto the reference's scheme per
SURVEY.md §8(d)-C): one step = the full server side of one inference — all
20 rounds of extract -> unshuffle -> W_r -> shuffle -> fast pack — for a
random-init ResNet-20-shaped quantized model at b=12 (M = 7^4), gamma
selectable (default 0).  Inputs are seeded uniform ciphertext uploads of the
exact per-round shapes (the server's work does not depend on their values).

metric: key switches per second ("ct-ops/s") over the whole
server inference; the line also reports latency per inference.
  value: uploads already resident in HBM (device timing, CUDA events).
  e2e:   through ServerEngine.server_round with host bundles (H2D of the
         uploads from pinned memory and D2H of the packed ciphertexts inside
         the timed region), one session per step.

--impl reference times the reference algorithm's CPU path (oracle/ port of
pkg/src/sfhr, fft key switching, thread pool over the host cores) on a
bounded sample: the ResNet-20 stem round.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = ROOT / "MEASURED_PEAKS.json"
METRIC = "ct-ops/s (key switches per second), ResNet-20-shape server inference"


def metric_for(workload):
    return METRIC if workload == "resnet20" else \
        f"ct-ops/s (key switches per second), {WORKLOADS[workload][0].split(' (')[0]}"
UNIT = "key-switches/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--b", type=int, default=None)
    ap.add_argument("--gamma", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="resnet20",
                    help="BASELINE configs: mlp = [0], resnet20 = [2] (default, the metric's config), "
                         "resnet18 = [3], resnet34 = [4] (one request per GPU)")
    a = ap.parse_args()
    if a.b is None:
        a.b = WORKLOADS[a.workload][1]
    if a.gamma is None:
        a.gamma = WORKLOADS[a.workload][2]
    return a


# workload -> (description, default b, default gamma, rounds label)
WORKLOADS = {
    "resnet20": ("ResNet-20-shape server inference (3x32x32, 10 classes)", 12, 0),
    "mlp": ("hybrid MLP 784-128-10 server inference", 16, 0),
    "resnet18": ("ResNet-18-shape server inference (3x64x64, 200 classes)", 16, 1),
    "resnet34": ("ResNet-34-shape server inference (3x224x224, 1000 classes), one request", 16, 1),
}


def make_model(workload, b, seed):
    from paper_2509_01253_b200 import workloads as W
    if workload == "mlp":
        return W.mlp_model(seed)
    return {"resnet20": W.resnet20_model, "resnet18": W.resnet18_model,
            "resnet34": W.resnet34_model}[workload](b, seed=seed)


# ---------------------------------------------------------------------------
# shared synthetic inputs


def synthetic_inputs(model, scheme, seed):
    """Per round: (k, npow, 2, N) uniform uploads < 2^53 and the exponent list."""
    from paper_2509_01253_b200.tracepack import power_exponents
    R = scheme.ring
    exps = power_exponents(scheme.gamma, R)
    rng = np.random.default_rng(seed)
    out = []
    for rnd in model.rounds:
        k = -(-rnd.input_len // R.N)
        out.append(rng.integers(0, 1 << 53, (k, len(exps), 2, R.N), dtype=np.uint64))
    return out, exps


def synthetic_ksk(scheme, seed):
    from paper_2509_01253_b200.engine import required_ksk_indices
    R = scheme.ring
    rng = np.random.default_rng(seed + 99)

    class Ct:
        def __init__(self, a, b):
            self.a, self.b = a, b

    keys = {d: [Ct(rng.integers(0, 1 << 53, R.N, dtype=np.uint64),
                   rng.integers(0, 1 << 53, R.N, dtype=np.uint64)) for _ in range(scheme.gadget.l)]
            for d in required_ksk_indices(scheme)}
    return keys


def as_bundles(power, exps, gamma):
    from paper_2509_01253_b200.keyswitch import RlweCiphertext
    from paper_2509_01253_b200.tracepack import PowerBundle
    return [PowerBundle(gamma, {d: RlweCiphertext(power[j, q, 0], power[j, q, 1])
                                for q, d in enumerate(exps)}) for j in range(power.shape[0])]


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)


class ClockSampler:
    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# our arm


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2509_01253_b200 import _native as nat
    from paper_2509_01253_b200.engine import ServerEngine
    from paper_2509_01253_b200.keyswitch import KeySwitchKeySet
    from paper_2509_01253_b200.params import preset_for_bits
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    scheme = preset_for_bits(args.b, args.gamma)
    model = make_model(args.workload, args.b, args.seed)
    R = scheme.ring
    engine = ServerEngine(model, scheme, master_seed=bytes(32), device=local_rank)
    keys = synthetic_ksk(scheme, args.seed)
    kid = engine.register_client(KeySwitchKeySet(keys, scheme.gadget, 0.0, R))
    key = engine.clients[kid].key
    powers, exps = synthetic_inputs(model, scheme, args.seed + 1000 * rank)
    powers_dev = [torch.from_numpy(p.view(np.int64)).to(dev) for p in powers]

    # session maps for the HBM-resident leg (sigma_r precomputed, uploaded once)
    sid = bytes([rank]) * 16
    engine.open_session(sid, kid)
    st = engine.sessions[sid]
    maps = []
    for r in range(1, len(model.rounds) + 1):
        im, om = engine.round_maps(st, sid, r)
        maps.append((torch.from_numpy(im).to(dev), None if om is None else torch.from_numpy(om).to(dev)))
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.int64, device=dev)

    ks_dev = torch.zeros(1, dtype=torch.int64, device=dev)

    def one_inference():
        # no host synchronisation between rounds: the KS count accumulates on the device
        for r in range(1, len(model.rounds) + 1):
            engine.round_device(r, key, powers_dev[r - 1], exps, maps[r - 1][0], maps[r - 1][1],
                                timed=False, counter=ks_dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        flush.fill_(1)
        one_inference()
    torch.cuda.synchronize()
    ks_dev.zero_()
    clocks = ClockSampler(local_rank)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    launches0 = nat.launch_count()
    nat.lib.sfhr_profile_enable(engine.ctx.h, 1)
    step_ms = []
    ks_total = 0
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush between timed steps (outside the events)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one_inference()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    barrier()
    ks_total = int(ks_dev.item())
    nat.lib.sfhr_profile_enable(engine.ctx.h, 0)
    launches = (nat.launch_count() - launches0) // args.steps
    ks_ms, ks_bytes, ks_launches = nat.profile_collect(engine.ctx.h)
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms, float(ks_total)], dtype=torch.float64, device=dev)
        mx = t.clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        sm = t.clone()
        torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
        total_ms_max, ks_all = mx[0].item(), sm[1].item()
    else:
        total_ms_max, ks_all = total_ms, float(ks_total)
    value = ks_all / (total_ms_max / 1e3)
    ks_per_step = ks_total // args.steps

    # ---- e2e through the public API (host bundles, one session per step) ----
    e2e = None
    if not args.no_e2e:
        bundles = [as_bundles(p, exps, args.gamma) for p in powers]
        h2d = sum(p.nbytes for p in powers)
        d2h = 0
        for rnd in model.rounds:
            G = -(-rnd.output_len // scheme.pack_factor)
            d2h += G * 2 * R.N * 8 + 8
        for r, rnd in enumerate(model.rounds):
            h2d += 8 * (rnd.input_len + (0 if rnd.final else rnd.output_len))
        wall = []
        for s in range(args.warmup + args.steps):
            sid2 = bytes([rank, 1]) + s.to_bytes(14, "little")
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            engine.open_session(sid2, kid)
            for r in range(1, len(model.rounds) + 1):
                engine.server_round(sid2, r, bundles[r - 1])
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            if s >= args.warmup:
                wall.append(t1 - t0)
        tot = sum(wall)
        if world > 1:
            t = torch.tensor([tot], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            tot = t.item()
        e2e = {"value": ks_all / tot, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "latency_s_per_inference": tot / args.steps,
               "path": f"ServerEngine.open_session + server_round x{len(model.rounds)} (host numpy bundles)"}
    clk = clocks.stop()

    # ---- roofline of the dominant kernel (fused key-switch stage) ----
    traffic = stage_traffic(R.N)
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    achieved = (ks_bytes / (ks_ms / 1e3)) / 1e9 if ks_ms > 0 else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": (achieved / hbm) if achieved else None,
            "traffic": traffic.get("traffic"), "traffic_detail": traffic,
            "kernel": "ks_stage_kernel (fused automorphism+decompose+Phi_M-NTT key switch+CRT)",
            "algorithmic_bytes": "rows * 32 * N per launch (read a,b; write a',b')",
            "launches_timed": ks_launches, "kernel_ms_per_step": ks_ms / args.steps,
            "kernel_share_of_step": (ks_ms / total_ms) if total_ms else None,
            "peak_source": "MEASURED_PEAKS.json" if PEAKS.exists() else "fallback 6650 GB/s",
            "note": "bound by the integer-multiply (fmaheavy) pipe at these ring sizes, see traffic_detail.int_mul_pipe_busy_frac (SURVEY §8(d)); HBM fraction reported as required"}

    line = {
        "metric": metric_for(args.workload), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64 (mod 2^53) / u32 NTT residues",
        "data": "synthetic uniform uploads of the exact per-round shapes; random-init quantized weights",
        "config": {"workload": f"{WORKLOADS[args.workload][0]}, {len(model.rounds)} rounds, b={args.b} "
                               f"(M={R.M}), gamma={args.gamma}",
                   "key_switches_per_step": int(ks_per_step), "rounds": len(model.rounds),
                   "latency_s_per_inference": total_ms_max / args.steps / 1e3,
                   "l2": "256 MiB L2 flush between timed steps; per-step working set > L2",
                   "parallelism": f"replicas x{world} (one independent inference per GPU)"},
        "gpu_launches": int(launches), "clocks": clk, "roofline": roof, "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, model, scheme, powers, exps, keys, sample_reps=1)
    return line


def stage_traffic(N):
    """DRAM bytes per ks_stage_kernel launch from the committed `ncu --set full` capture.

    Returned per launch (mean over the captured launches), with the ratio to the
    algorithmic 32 N bytes per row (rows = grid / 3 CTAs per cluster); the capture
    is of the b = 12 (N = 2058) ResNet-20 stem pack, so the ratio is only quoted
    for that ring."""
    f = ROOT / "profiles" / "r02j" / "ncu_stage_summary.json"
    try:
        launches = [l for l in json.loads(f.read_text())["launches"] if "ks_stage_kernel" in l["kernel"]]
    except Exception:
        return {"traffic": None, "note": f"{f.name} missing"}
    tr = [1e6 * (l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"]) for l in launches]
    alg = [l["launch__grid_size"] / 3 * 32 * 2058 for l in launches]
    out = {"traffic": sum(tr) / len(tr), "unit": "bytes per launch", "launches": len(tr),
           "algorithmic_bytes_per_launch": sum(alg) / len(alg), "source": str(f.relative_to(ROOT))}
    # the compute side of the same capture: this kernel is bound by the integer-multiply pipe
    # (IMAD / IMAD.HI / IMAD.WIDE run only on fmaheavy), not by HBM
    def mean(key):
        v = [l.get(key) for l in launches if isinstance(l.get(key), float)]
        return sum(v) / len(v) / 100.0 if v else None
    out["int_mul_pipe_busy_frac"] = mean("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed")
    out["alu_pipe_busy_frac"] = mean("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active")
    out["sm_issue_active_frac"] = mean("smsp__issue_active.avg.pct_of_peak_sustained_active")
    if N == 2058:
        out["traffic_over_algorithmic"] = sum(tr) / sum(alg)
    return out


# ---------------------------------------------------------------------------
# CPU arm (oracle port of the reference's algorithm)


def cpu_stem_round(args, model, scheme, powers, exps, keys, threads):
    """One timed reference-algorithm stem round: extract + linear + pack, fft KS."""
    from oracle import keyswitch as oks
    from oracle import lowering as olo
    from oracle import pack as opk
    from oracle import protocol as opr
    from oracle import scheme as osc
    os_ = osc.preset(args.b, args.gamma)
    R = os_.ring
    ksk = oks.KskSet({d: [oks.Ct(c.a, c.b) for c in row] for d, row in keys.items()}, os_.gadget, 0.0, R)
    orounds = olo.build_rounds(model.layers)
    # single-layer stem round: its round matrix is the layer matrix (same integers, no O(E^3) setup)
    W, bias = olo.layer_matrix(model.layers[orounds[0].layers[0]])
    srv = opr.OracleServer(model, os_, ksk, master_seed=bytes(32), session_id=bytes(16), ks_mode="fft",
                           round_mats=[(W, bias)] + [None] * (len(orounds) - 1), threads=threads)
    bundles = [opk.Bundle(args.gamma, {d: oks.Ct(powers[0][j, q, 0], powers[0][j, q, 1])
                                       for q, d in enumerate(exps)}) for j in range(powers[0].shape[0])]
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:
        lim = None
    t0 = time.perf_counter()
    packs, st = srv.server_round(1, bundles)
    dt = time.perf_counter() - t0
    if lim is not None:
        lim.unregister()
    return dt, st.key_switches


def cpu_pack_sample(args, keys, n_groups, threads):
    """Bounded CPU sample for the large workloads: fast_pack of n_groups full
    pack groups of uniform rows (the reference's dominant phase)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import keyswitch as oks
    from oracle import pack as opk
    from oracle import scheme as osc
    os_ = osc.preset(args.b, args.gamma)
    R = os_.ring
    ksk = oks.KskSet({d: [oks.Ct(c.a, c.b) for c in row] for d, row in keys.items()}, os_.gadget, 0.0, R)
    eng = oks.KsEngine(ksk, "fft")
    F = os_.pack_factor
    rng = np.random.default_rng(5)
    groups = [rng.integers(0, 1 << 53, (F, 2, R.N), dtype=np.uint64) for _ in range(n_groups)]
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:
        lim = None
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(lambda g: opk.fast_pack(g, os_, eng), groups))
    dt = time.perf_counter() - t0
    if lim is not None:
        lim.unregister()
    ks = n_groups * opk.expected_pack_switches(R.t, R.alpha, os_.beta_eff, args.gamma)
    return dt, ks


def cpu_baseline(args, model, scheme, powers, exps, keys, sample_reps=1):
    cores = os.cpu_count() or 1
    if args.workload in ("resnet18", "resnet34"):
        n = 2 * cores
        dt, ks = cpu_pack_sample(args, keys, n, cores)
        return {"value": ks / dt, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": f"{n} full pack groups (fast_pack, fft key switching) of uniform rows, b={args.b} "
                          f"gamma={args.gamma}, thread pool of {cores}; {ks} key switches in {dt:.2f} s "
                          f"(extraction + linear excluded: full CPU rounds of this shape take hours)"}
    ts, ks = [], 0
    for _ in range(sample_reps):
        dt, k = cpu_stem_round(args, model, scheme, powers, exps, keys, cores)
        ts.append(dt)
        ks += k
    return {"value": ks / sum(ts), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"ResNet-20 stem round (3072->16384 rows, 56 packs), b={args.b} gamma={args.gamma}: "
                      f"extract + CSR linear + fast_pack with fft key switching, thread pool of {cores}; "
                      f"{ks // sample_reps} key switches in {statistics.mean(ts):.2f} s"}


def run_reference(args):
    from paper_2509_01253_b200.params import preset_for_bits
    scheme = preset_for_bits(args.b, args.gamma)
    model = make_model(args.workload, args.b, args.seed)
    powers, exps = synthetic_inputs(model, scheme, args.seed + 1000)
    keys = synthetic_ksk(scheme, args.seed)
    cores = os.cpu_count() or 1
    big = args.workload in ("resnet18", "resnet34")
    one = (lambda: cpu_pack_sample(args, keys, 2 * cores, cores)) if big else \
        (lambda: cpu_stem_round(args, model, scheme, powers[:1], exps, keys, cores))
    for _ in range(args.warmup):
        one()
    ts, ks = [], 0
    for _ in range(args.steps):
        dt, k = one()
        ts.append(dt)
        ks += k
    value = ks / sum(ts)
    r0 = model.rounds[0]
    sample = (f"{args.workload} first round ({r0.input_len}->{r0.output_len} rows), b={args.b} gamma={args.gamma}, "
              f"oracle port of the reference CPU path (fft KS), {cores} threads")
    if big:
        sample = (f"{2 * cores} full pack groups per step (fast_pack, fft KS) of uniform rows, b={args.b} "
                  f"gamma={args.gamma}, {cores} threads (extraction + linear excluded)")
    return {"impl": "reference", "metric": metric_for(args.workload), "value": value, "unit": UNIT,
            "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(ts) / len(ts),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64 (mod 2^53) / f64 FFT", "data": "synthetic",
            "config": {"workload": f"{WORKLOADS[args.workload][0]}, {len(model.rounds)} rounds, b={args.b} "
                                   f"(M={scheme.ring.M}), gamma={args.gamma}", "sample": "first (stem) round"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl")
    line = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
