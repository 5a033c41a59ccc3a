#!/usr/bin/env python
"""bench.py — BSA (arXiv 2509.01085) sparse-attention fwd+bwd on B200.

One "step" = the whole hot path over one batch of synthetic input:
partition, query pruning (Eq.2), KV-block admission (Eq.3 + Eq.4), sparse attention forward + fill
(Eq.5) and backward, all through the C ABI of libbsa.so.

    python bench.py                        # N=1, Wan2.1-1.3B-shaped 32k workload (BASELINE configs[1])
    python bench.py --config wan14b_75k    # 75,600 tokens, 40 heads
    torchrun --nproc-per-node N bench.py --gpus N   # weak scaling: one independent problem per rank
    python bench.py --impl reference       # the CPU fp64 oracle as the reference arm

Metric (BASELINE.json): effective (executed) TFLOPS of fwd+bwd = 14*d*P / step time, where P is the
number of admitted (query, key) pairs; also ms per step and the same library's own
dense path (r = 1, k = N, tau = 1) for the speedup. Inputs are larger than L2 (4 x 100 MB) and L2
is additionally flushed (256 MiB write) between timed steps.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json metric; value = effective (executed-FLOP) TFLOPS, ms_per_step = fwd+bwd ms
METRIC = "BSA attention fwd+bwd ms & effective TFLOPS at 32k/75k tokens vs own dense"

CONFIGS = {
    # name: grid, block, B, Hh, d, r, f (k = ceil(f N)), tau, generator
    "tiny": dict(grid=(4, 8, 8), block=(2, 4, 4), B=1, Hh=2, d=64, r=0.5, f=0.5, tau=0.9, kind="video"),
    "wan1.3b_32k": dict(grid=(21, 30, 52), block=(4, 4, 4), B=1, Hh=12, d=128, r=0.5, f=0.1, tau=0.9, kind="video"),
    "wan14b_75k": dict(grid=(21, 45, 80), block=(4, 4, 4), B=1, Hh=40, d=128, r=0.5, f=0.1, tau=0.9, kind="video"),
    "long_147k": dict(grid=(41, 45, 80), block=(4, 4, 4), B=1, Hh=40, d=128, r=0.5, f=0.1, tau=0.9, kind="video"),
}
KERNEL_NAMES = ["partition", "select_queries", "pool", "scores", "admit", "k2q", "gather", "attn_fwd", "fill",
                "bwd_prep", "attn_bwd", "bwd_finalize", "kv_image", "sp_relayout", "fwd_group", "bwd_pairs", "bwd_dq",
                "fwd_union"]
SELECTION_IDS = range(0, 7)


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d.get("bf16_tflops_sustained"),
                    source="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, source="fallback")


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    def __init__(self, dev_index: int, period=0.005):
        self.samples, self.reasons, self.period = [], set(), period
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------ reference arm
def oracle_sample(cfg, seed, heads, threads, unit=(0, 0, 0), inputs=None):
    """The fp64 oracle as it stands on `heads` heads of the workload: selection + fwd + bwd.
    Returns (seconds, executed fwd+bwd FLOPs of the sample)."""
    import ctypes

    import numpy as np

    import bsa_gen
    import oracle as orc
    orc.set_threads(threads)
    g = orc.Geom(*cfg["grid"], *cfg["block"], *unit)
    d, r, tau = cfg["d"], cfg["r"], cfg["tau"]
    N, Lq = orc.sizes(g, r)
    k = orc.resolve_k(cfg["f"], N)
    if inputs is None:
        Q, K, V = bsa_gen.make_inputs(cfg["kind"], seed, 1, heads, cfg["grid"], d)
        dO = bsa_gen.grad_output(seed, (1, heads, g.L, d))
    else:  # the exact bf16 values the GPU run used (generated on the device)
        Q, K, V, dO = (x[:1, :heads].cpu() for x in inputs)
    Qd, Kd, Vd, dOd = (x.double().numpy().reshape(heads, g.L, d) for x in (Q, K, V, dO))
    t0 = time.perf_counter()
    qs = orc.select_queries(g, r, Qd)
    kv = orc.select_kv(g, Qd, Kd, k, tau)
    scale = 1.0 / math.sqrt(d)
    O, lse = orc.attn_fwd(g, r, Qd, Kd, Vd, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], scale)
    orc.attn_bwd(g, r, Qd, Kd, Vd, dOd, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], scale)
    dt = time.perf_counter() - t0
    p = orc.partition(g, r)
    bsz = np.diff(p["block_off"]).astype(np.int64)
    kept = np.diff(p["kept_off"]).astype(np.int64)
    P = 0
    for h in range(heads):
        for i in range(N):
            P += int(kept[i]) * int(bsz[kv["q2k_idx"][h, i, :kv["q2k_num"][h, i]]].sum())
    oracle_sample.last = (qs, kv)  # selection of the sample, for the GPU-vs-oracle spot check
    return dt, 14 * d * P


def selection_spot_check(layer, qs, kv):
    """Head 0's selection from the timed GPU run against the oracle's (SURVEY §8(c) protocol): kept sets, donors
    and q2k rows must be equal; a disagreement is a near-tie when the oracle's own margin (reading C24) is below
    1e-6, else a mismatch. Returns the equality flags and both counts."""
    import numpy as np
    NEAR = 1e-6
    kept = layer.kept_tok[0, 0].cpu().numpy()
    donor = layer.donor[0, 0].cpu().numpy()
    num = layer.q2k_num[0, 0].cpu().numpy()
    idx = layer.q2k_idx[0, 0].cpu().numpy()
    L = donor.shape[0]
    kg, kr = np.zeros(L, bool), np.zeros(L, bool)
    kg[kept] = True
    kr[qs["kept_tok"][0]] = True
    near = mism = 0
    for t in np.nonzero(kg != kr)[0]:
        near, mism = (near + 1, mism) if qs["unit_margin"][0, t] < NEAR else (near, mism + 1)
    for t in np.nonzero(donor != qs["donor"][0])[0]:
        if kg[t] != kr[t]:
            continue
        near, mism = (near + 1, mism) if qs["donor_margin"][0, t] < NEAR else (near, mism + 1)
    rows_eq = 0
    for i in range(len(num)):
        if num[i] == kv["q2k_num"][0, i] and np.array_equal(idx[i, :num[i]], kv["q2k_idx"][0, i, :num[i]]):
            rows_eq += 1
            continue
        m = min(kv["thr_margin"][0, i], kv["mass_margin"][0, i], kv["order_margin"][0, i])
        near, mism = (near + 1, mism) if m < NEAR else (near, mism + 1)
    return {"head": 0, "kept_tok_equal": bool(np.array_equal(kept, qs["kept_tok"][0])),
            "donor_equal": bool(np.array_equal(donor, qs["donor"][0])), "q2k_rows_equal": rows_eq,
            "q2k_rows": int(len(num)), "near_ties": near, "mismatches": mism}


def run_reference(args, cfg, rank, world):
    if world > 1 and rank != 0:
        return
    import oracle as orc
    orc.build()
    threads = os.cpu_count() or 1
    heads = 1
    times, flops = [], 0
    for s in range(args.warmup + args.steps):
        dt, fl = oracle_sample(cfg, args.seed, heads, threads)
        if s >= args.warmup:
            times.append(dt)
            flops = fl
    t = sum(times) / len(times)
    val = flops / t / 1e12
    sample = f"1 of {cfg['Hh']} heads of the {args.config} workload (full selection + fwd + bwd of that head), " \
             f"fp64, {threads} threads"
    line = {
        "impl": "reference", "metric": METRIC, "value": val,
        "unit": "TFLOPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "sample": "1 head", **{k: v for k, v in cfg.items() if k != "kind"},
                   "generator": cfg["kind"]},
        "cpu_baseline": {"value": val, "unit": "TFLOPS", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="bsa", choices=["bsa", "reference"])
    ap.add_argument("--config", default="wan1.3b_32k", choices=sorted(CONFIGS))
    ap.add_argument("--r", type=float, default=None)
    ap.add_argument("--f", type=float, default=None, help="Eq.3 key fraction: k = ceil(f N)")
    ap.add_argument("--tau", type=float, default=None)
    ap.add_argument("--kind", default=None, choices=["video", "iid"])
    ap.add_argument("--unit", default=None, help="query-selection window ut,uh,uw (P:168; default = whole block)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dense-steps", type=int, default=3, help="steps of the own-dense path (0 = skip)")
    ap.add_argument("--e2e-steps", type=int, default=16, help="e2e steps (pipelined H2D / compute / D2H; more steps amortise the pipeline fill)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="problem", choices=["problem", "heads", "ulysses"],
                    help="N>1: problem = one independent problem per rank (weak); heads = split the heads; "
                         "ulysses = token-sharded inputs regathered per head group by all-to-all (strong)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    for key in ("r", "f", "tau", "kind"):
        if getattr(args, key) is not None:
            cfg[key] = getattr(args, key)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist

    import bsa_gen
    import paper_2509_01085_b200 as bsa
    from paper_2509_01085_b200.runner import BSAAttention

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl_log = None
    if world > 1:
        # NCCL's own communicator lines (ranks, NVLink/NVLS transport), filtered into the JSON line so the scaling
        # run can be checked against what NCCL actually set up
        if "NCCL_DEBUG" not in os.environ:
            nccl_log = f"/tmp/bsa_nccl_{os.getpid()}.log"
            os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,NVLS", NCCL_DEBUG_FILE=nccl_log)
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    L = bsa.lib()

    unit = tuple(int(x) for x in args.unit.split(",")) if args.unit else (0, 0, 0)
    g = bsa.Geometry(*cfg["grid"], *cfg["block"], *unit)
    B, Hh, d = cfg["B"], cfg["Hh"], cfg["d"]
    from paper_2509_01085_b200.shard import head_range, problem_seed, rank_time_spread, reduce_step_stats
    if args.shard == "heads":
        # strong scaling: the heads of ONE problem are split over the ranks (no collective on the path)
        seed = args.seed
        h0, h1 = head_range(Hh, world, rank)
    else:
        # weak scaling: each rank owns an independent problem (its own batch element / seed)
        seed, h0, h1 = problem_seed(args.seed, rank), 0, Hh
    if args.shard == "ulysses":
        seed, h0, h1 = args.seed, 0, Hh
    Q, K, V = bsa_gen.make_inputs(cfg["kind"], seed, B, Hh, cfg["grid"], d, device=dev)
    dO = bsa_gen.grad_output(seed, (B, Hh, g.L, d)).to(dev)
    if (h0, h1) != (0, Hh):
        Q, K, V, dO = (x[:, h0:h1].contiguous() for x in (Q, K, V, dO))
    Hh = h1 - h0
    if args.shard == "ulysses":
        # sequence-parallel layout: this rank's contiguous token chunk of all heads, [B, L/P, Hh, d]
        from paper_2509_01085_b200.ulysses import UlyssesBSA
        uly = UlyssesBSA(g, cfg["r"], cfg["f"], cfg["tau"], B, Hh, d, device=dev)
        Ls = g.L // world
        Q, K, V, dO = (x.permute(0, 2, 1, 3)[:, rank * Ls:(rank + 1) * Ls].contiguous() for x in (Q, K, V, dO))
        layer = uly.layer
        layer.cache_partition = False

        def fwd_bwd(q, k, v, do):
            O = uly.forward(q, k, v)
            return (O, *uly.backward(do))
    else:
        layer = BSAAttention(g, cfg["r"], cfg["f"], cfg["tau"], B, Hh, d, device=dev, cache_partition=False)

        def fwd_bwd(q, k, v, do):
            layer.forward(q, k, v)
            layer.backward(do)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        fwd_bwd(Q, K, V, dO)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    fl = layer.flops()

    # ---------------------------------------------------------------- timed region (headline, no instrumentation)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = L.bsa_launch_count()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            starts[s].record()
            step()
            ends[s].record()
        torch.cuda.synchronize()
    launches = L.bsa_launch_count() - n0
    if world > 1:
        dist.barrier()
    # ---------------------------------------------------------------- the same K steps again with the library's
    # per-kernel event instrumentation (kernel_ms, phases, roofline): kept out of the headline region
    L.bsa_timing_read(None, None, 0)
    L.bsa_timing_enable(1)
    for s in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    L.bsa_timing_enable(0)
    import ctypes
    nk = len(KERNEL_NAMES)
    kms = (ctypes.c_double * nk)()
    kcnt = (ctypes.c_int32 * nk)()
    L.bsa_timing_read(kms, kcnt, nk)
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    total_ms = sum(step_ms)
    t_max, f_sum = reduce_step_stats(total_ms, fl["total"] * args.steps, device=dev)
    t_hi, t_lo = rank_time_spread(total_ms, device=dev)
    value = f_sum / (t_max * 1e-3) / 1e12
    ms_per_step = t_max / args.steps
    kernel_ms = {KERNEL_NAMES[i]: kms[i] / max(1, args.steps) for i in range(nk) if kcnt[i]}
    phases = {
        "selection_ms": sum(kms[i] for i in SELECTION_IDS) / args.steps,
        "fwd_ms": (kms[7] + kms[8] + kms[12] + kms[14] + kms[17]) / args.steps,
        "bwd_ms": (kms[9] + kms[10] + kms[11] + kms[15] + kms[16]) / args.steps,
        "sp_relayout_ms": kms[13] / args.steps,
    }

    # ---------------------------------------------------------------- roofline (dominant kernel)
    # The backward's dQ path (include/bsa.h bsa_attn_bwd): the dS path when the admitted (query block, KV block)
    # pairs fit the workspace -- attn_bwd then executes S, dP, dV, dK (8 d P flops) and bwd_dq dQ (2 d P) --
    # else the reduce path, where attn_bwd executes all five contractions (10 d P).
    peaks = read_peaks()
    n_pairs = int(layer.q2k_num.to(torch.int64).sum().item())
    cap = bsa.bwd_ds_capacity(g, layer.r, B, layer.Hh, d)
    ds_path = 0 <= n_pairs <= cap
    P = fl["pairs"]
    per_kernel = {"attn_fwd": (7, fl["fwd"]), "attn_bwd": (10, (8 if ds_path else 10) * d * P)}
    if ds_path:
        per_kernel["bwd_dq"] = (16, 2 * d * P)
    kernels_roof = {}
    for kname, (kid, kfl) in per_kernel.items():
        kms_avg = kms[kid] / max(1, kcnt[kid])
        kernels_roof[kname] = {"avg_launch_ms": kms_avg, "algorithmic_flops_per_launch": kfl,
                               "achieved_tflops": kfl / (kms_avg * 1e-3) / 1e12 if kms_avg > 0 else None,
                               "frac": kfl / (kms_avg * 1e-3) / 1e12 / peaks["bf16"] if kms_avg > 0 else None}
    dom = max(("attn_fwd", "attn_bwd"), key=lambda k: kms[per_kernel[k][0]])
    dom_ms = kernels_roof[dom]["avg_launch_ms"]
    dom_flops = per_kernel[dom][1]
    achieved = dom_flops / (dom_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peaks["bf16"], "unit": "TFLOP/s",
                "frac": achieved / peaks["bf16"], "traffic": traffic, "peak_source": f"{peaks['source']} bf16 burst",
                "algorithmic_flops_per_launch": dom_flops, "avg_launch_ms": dom_ms,
                "bwd_dq_path": "ds" if ds_path else "reduce", "admitted_pairs": n_pairs, "ds_capacity": cap,
                "kernels": kernels_roof}
    if ds_path:
        # bwd_dq streams one K tile (BT d 2 B, L2) and one dS tile (SR rows x 128 B, HBM) per admitted pair
        tile_b = layer.g.BT * d * 2 + layer.SR * 128
        dq_ms = kernels_roof["bwd_dq"]["avg_launch_ms"]
        roofline["secondary"] = {"bound": "l2_copy", "kernel": "bwd_dq", "bytes_per_launch": n_pairs * tile_b,
                                 "achieved_tbs": n_pairs * tile_b / (dq_ms * 1e-3) / 1e12 if dq_ms > 0 else None,
                                 "peak_tbs": 19.0,
                                 "peak_source": "measured L2 -> smem bulk copies, tools/microbench/bulk_bench.cu "
                                                "(profiles/r01_microbench.md)"}
    else:
        # every admitted (query row, KV block) sends one fp32 dQ partial row of d values to the L2 reduce units;
        # measured ceiling of that path 6.2 TB/s (tools/microbench/red_rate.cu, 128-byte-row tensor reduce boxes)
        dq_bytes = layer.admitted_block_rows() * d * 4
        bwd_ms = kms[10] / max(1, kcnt[10])
        roofline["secondary"] = {"bound": "l2_reduce", "kernel": "attn_bwd", "bytes_per_launch": dq_bytes,
                                 "achieved_tbs": dq_bytes / (bwd_ms * 1e-3) / 1e12, "peak_tbs": 6.2,
                                 "frac": dq_bytes / (bwd_ms * 1e-3) / 1e12 / 6.2,
                                 "peak_source": "measured, tools/microbench/red_rate.cu (profiles/r01_microbench.md)"}
    # selection kernels against HBM (algorithmic bytes), per (b,h): read Q and K once (4 L d B);
    # write kept_tok + donor (4 Lq + 4 L B); q2k and its transpose k2q, counts and the admitted block ids
    # (2 x 4 N (1 + avg|S_i|) B, blocks not tokens); the pooled Q_c (8 N d B) and Q^s (2 Lq d B) outputs
    BH, Lq, N = B * layer.Hh, layer.Lq, layer.N
    sp = layer.sparsity()
    avg_S = sp["mean_admitted_blocks"]
    sel_parts = {"read_QK": 4 * g.L * d, "kept_donor": 4 * Lq + 4 * g.L, "q2k_k2q": 2 * 4 * N * (1 + avg_S),
                 "pooled_Qc": 8 * N * d, "packed_Qs": 2 * Lq * d}
    sel_bytes = BH * sum(sel_parts.values())
    sel_ms = phases["selection_ms"]

    # ---------------------------------------------------------------- the same step as one CUDA graph
    graph = None
    if args.shard != "ulysses":
        from paper_2509_01085_b200.runner import BSAStepGraph
        sg = BSAStepGraph(layer, Q, K, V, dO)
        gev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
        for s in range(args.steps):
            flush.zero_()
            gev[2 * s].record()
            sg.replay()
            gev[2 * s + 1].record()
        torch.cuda.synchronize()
        gms = sum(gev[2 * s].elapsed_time(gev[2 * s + 1]) for s in range(args.steps)) / args.steps
        graph = {"ms_per_step": gms, "tflops": fl["total"] / (gms * 1e-3) / 1e12,
                 "note": "selection + fwd + bwd captured once (runner.BSAStepGraph), replayed per step"}
        del sg

    # ---------------------------------------------------------------- own dense path (r=1, k=N, tau=1)
    dense = None
    if args.dense_steps > 0:
        dl = BSAAttention(g, 1.0, 1.0, 1.0, B, Hh, d, device=dev)
        for _ in range(2):
            dl.forward(Q, K, V)
            dl.backward(dO)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.dense_steps)]
        for s in range(args.dense_steps):
            flush.zero_()
            ev[2 * s].record()
            dl.forward(Q, K, V)
            dl.backward(dO)
            ev[2 * s + 1].record()
        torch.cuda.synchronize()
        dms = sum(ev[2 * s].elapsed_time(ev[2 * s + 1]) for s in range(args.dense_steps)) / args.dense_steps
        dfl = dl.flops()
        dense = {"ms_per_step": dms, "tflops": dfl["total"] / (dms * 1e-3) / 1e12, "speedup": dms / ms_per_step}
        del dl
        torch.cuda.empty_cache()

    # ---------------------------------------------------------------- e2e: host buffers, copies inside the region
    # Each step copies its four input tensors Q, K, V, dO host->device (pinned, on a copy stream) and its four
    # results O, dQ, dK, dV device->host (pinned, on a second copy stream). Inputs and outputs are double-buffered
    # so the copies of neighbouring steps overlap this step's kernels (PCIe is full duplex).
    hQ, hK, hV, hdO = (x.cpu().pin_memory() for x in (Q, K, V, dO))
    h_out = [[torch.empty(Q.shape, dtype=torch.bfloat16).pin_memory() for _ in range(4)] for _ in range(2)]
    bufs = [[torch.empty_like(Q) for _ in range(4)] for _ in range(2)]
    obufs = [[torch.empty_like(Q) for _ in range(4)] for _ in range(2)]
    cstream, dstream = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    main = torch.cuda.current_stream(dev)
    n_e2e = max(1, args.e2e_steps)
    copied = [torch.cuda.Event() for _ in range(n_e2e)]
    consumed = [torch.cuda.Event() for _ in range(n_e2e)]
    computed = [torch.cuda.Event() for _ in range(n_e2e)]
    drained = [torch.cuda.Event() for _ in range(n_e2e)]
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e_start.record(cstream)
    main.wait_stream(cstream)
    dstream.wait_stream(cstream)
    for s in range(n_e2e):
        with torch.cuda.stream(cstream):
            if s >= 2:
                cstream.wait_event(consumed[s - 2])  # step s-2 is done reading this input set
            for dst, src in zip(bufs[s % 2], (hQ, hK, hV, hdO)):
                dst.copy_(src, non_blocking=True)
            copied[s].record(cstream)
        main.wait_event(copied[s])
        if s >= 2:
            main.wait_event(drained[s - 2])  # this output set has reached the host
        Qg, Kg, Vg, dOg = bufs[s % 2]
        Og, dQg, dKg, dVg = obufs[s % 2]
        if args.shard == "ulysses":
            Og, dQg, dKg, dVg = fwd_bwd(Qg, Kg, Vg, dOg)
            for x in (Og, dQg, dKg, dVg):
                x.record_stream(dstream)
        else:
            layer.forward(Qg, Kg, Vg, out=Og)
            layer.backward(dOg, out=(dQg, dKg, dVg))
        consumed[s].record(main)
        computed[s].record(main)
        with torch.cuda.stream(dstream):
            dstream.wait_event(computed[s])
            for dst, src in zip(h_out[s % 2], (Og, dQg, dKg, dVg)):
                dst.copy_(src, non_blocking=True)
            drained[s].record(dstream)
    main.wait_stream(dstream)
    e_end.record(main)
    torch.cuda.synchronize()
    e2e_ms = e_start.elapsed_time(e_end) / n_e2e
    e2e_max, e2e_flops = reduce_step_stats(e2e_ms, fl["total"], device=dev)
    e2e_val = e2e_flops / (e2e_max * 1e-3) / 1e12 if args.e2e_steps else None
    tensor_bytes = Q.numel() * 2

    # ---------------------------------------------------------------- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle as orc
        orc.build()
        threads = os.cpu_count() or 1
        same = args.shard != "ulysses"
        dt, cfl = oracle_sample(cfg, args.seed, 1, threads, unit, inputs=(Q, K, V, dO) if same else None)
        cpu = {"value": cfl / dt / 1e12, "unit": "TFLOPS", "cores": threads, "kind": "oracle",
               "sample": f"head 0 of {Hh} of the {args.config} workload: full selection + fwd + bwd, fp64, "
                         f"{dt:.1f} s"}
        if same:
            cpu["selection_check"] = selection_spot_check(layer, *oracle_sample.last)

    nccl_lines = None
    if nccl_log and os.path.exists(nccl_log):
        keep = ("comm ", "nRanks", "NVLS", "NVLink", "P2P", "Init COMPLETE", "version")
        nccl_lines = [ln.strip()[-200:] for ln in open(nccl_log, errors="replace") if any(k in ln for k in keep)][:16]
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.shard in ("heads", "ulysses") else "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded G_video latents, bsa_gen)",
            "config": {"workload": args.config, "grid": list(cfg["grid"]), "block": list(cfg["block"]), "B": B,
                       "heads": Hh, "d": d, "r": cfg["r"], "k": layer.k, "k_frac": cfg["f"], "tau": cfg["tau"],
                       "generator": cfg["kind"], "tokens": g.L, "N_blocks": N,
                       "unit": list(unit) if args.unit else "block",
                       "l2": "inputs > L2 (4 x %.0f MB) and 256 MiB L2 flush between timed steps" % (tensor_bytes / 1e6),
                       "parallelism": (f"head-shard x{world} (heads of one problem split over ranks, no collective)"
                                       if args.shard == "heads" else
                                       f"ulysses x{world} (token-sharded [B, L/P, Hh, d] inputs; NCCL all-to-all "
                                       f"to head groups and back, inside the timed step)"
                                       if args.shard == "ulysses" else
                                       f"bh-shard x{world} (independent problems, no collective)")},
            "gpu_launches": int(launches),
            "nccl": nccl_lines,
            "rank_imbalance": t_hi / t_lo if t_lo > 0 else None,
            "clocks": clk.summary(),
            "roofline": roofline,
            "selection_hbm": {"bytes": sel_bytes, "bytes_per_head": sel_parts, "ms": sel_ms,
                              "achieved_gbs": sel_bytes / (sel_ms * 1e-3) / 1e9,
                              "peak_gbs": peaks["hbm"], "frac": sel_bytes / (sel_ms * 1e-3) / 1e9 / peaks["hbm"]},
            "sparsity": {**sp, "pair_density": fl["density"], "pair_sparsity": 1 - fl["density"]},
            "near_ties": (cpu or {}).get("selection_check", {}).get("near_ties"),
            "phases_ms": phases, "kernel_ms": kernel_ms,
            "executed": {"pairs": fl["pairs"], "density": fl["density"], "flops_per_step": fl["total"],
                         "dense_equiv_tflops": fl["dense_total"] * world / (t_max * 1e-3 / args.steps) / 1e12},
            "own_dense": dense,
            "cuda_graph": graph,
            "e2e": {"value": e2e_val, "unit": "TFLOPS", "ms_per_step": e2e_max,
                    "h2d_bytes_per_step": 4 * tensor_bytes, "d2h_bytes_per_step": 4 * tensor_bytes,
                    "note": "every step: pinned H2D of Q, K, V, dO and pinned D2H of O, dQ, dK, dV (two copy streams, "
                            "double-buffered so neighbouring steps' copies overlap this step's kernels), through "
                            "BSAAttention.forward/backward; PCIe-bound"},
            "cpu_baseline": cpu,
            "paper_context": "17.79x attention-training speedup and 20x FLOP reduction at 153,600 tokens on H100 "
                             "(Triton, precision unstated; PAPER.md P:234, P:22) — context, not the target",
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
