"""Sparsity sweep at 32,760 tokens (BASELINE configs[4]; SURVEY.md §8(d) "sweep @32k").

r in {1, .5, .25} x tau in {1, .95, .9}, run twice: k = N (Eq.3 threshold off; (1, 1) is the dense
path) and k = ceil(.1 N) (the paper's end-of-anneal k). Each point: fwd+bwd ms (CUDA events,
median of `steps`, 256 MiB L2 flush between steps), executed TFLOPS (14 d P), realised pair density,
speedup vs the same library's dense point, and the ideal 1 / density.

    python tools/profiling/sweep.py [--steps 5] > profiles/rNN_sweep.json
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bsa_gen  # noqa: E402
import paper_2509_01085_b200 as bsa  # noqa: E402
from paper_2509_01085_b200.runner import BSAAttention  # noqa: E402


def time_layer(layer, Q, K, V, dO, steps, flush):
    for _ in range(3):
        layer.forward(Q, K, V)
        layer.backward(dO)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        layer.forward(Q, K, V)
        layer.backward(dO)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--kind", default="video")
    args = ap.parse_args()
    grid, Hh, d = (21, 30, 52), 12, 128
    g = bsa.Geometry(*grid)
    Q, K, V = bsa_gen.make_inputs(args.kind, 0, 1, Hh, grid, d, device="cuda")
    dO = bsa_gen.grad_output(0, (1, Hh, g.L, d)).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    pts = []
    dense_ms = None
    for f in (1.0, 0.1):
        for r in (1.0, 0.5, 0.25):
            for tau in (1.0, 0.95, 0.9):
                layer = BSAAttention(g, r, f, tau, 1, Hh, d)
                ms = time_layer(layer, Q, K, V, dO, args.steps, flush)
                fl = layer.flops()
                if f == 1.0 and r == 1.0 and tau == 1.0:
                    dense_ms = ms
                pts.append({"r": r, "k_frac": f, "k": layer.k, "tau": tau, "ms": ms,
                            "tflops_executed": fl["total"] / (ms * 1e-3) / 1e12, "density": fl["density"],
                            "speedup_vs_dense": None, "ideal_speedup": 1.0 / fl["density"]})
                del layer
                torch.cuda.empty_cache()
    # selection variant (C28): SPEC's unified_prob at the paper's end point (r = .5, k = ceil(.1 N))
    layer = BSAAttention(g, 0.5, 0.1, 1.0, 1, Hh, d, kv_mode=1)
    ms = time_layer(layer, Q, K, V, dO, args.steps, flush)
    fl = layer.flops()
    pts.append({"r": 0.5, "k_frac": 0.1, "k": layer.k, "tau": None, "kv_mode": "unified_prob", "ms": ms,
                "tflops_executed": fl["total"] / (ms * 1e-3) / 1e12, "density": fl["density"],
                "speedup_vs_dense": None, "ideal_speedup": 1.0 / fl["density"],
                "kv_blocks_per_row": float(layer.q2k_num.float().mean().item())})
    for p in pts:
        p["speedup_vs_dense"] = dense_ms / p["ms"]
    print(json.dumps({"workload": "wan1.3b_32k sweep", "grid": grid, "heads": Hh, "d": d, "generator": args.kind,
                      "steps": args.steps, "dense_ms": dense_ms, "points": pts}))


if __name__ == "__main__":
    main()
