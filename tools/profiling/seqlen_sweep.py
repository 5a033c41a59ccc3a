"""Sequence-length sweep (the analogue of the paper's Fig. 6).

Wan-1.3B-shaped heads (12 x d=128, 4x4x4 blocks) on the paper's two grids 16x28x52 (23,296 tokens) and
40x48x80 (153,600) plus the BASELINE 32k / 75k grids: BSA fwd+bwd (r = .5, k = ceil(.1 N), tau = .9)
against the same library's dense path (r = 1, k = N, tau = 1); device ms (CUDA events, L2 flushed).

    python tools/profiling/seqlen_sweep.py > profiles/rNN_seqlen_sweep.json
"""
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


def timed(layer, Q, K, V, dO, steps, flush):
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
    Hh, d = 12, 128
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for grid in [(16, 28, 52), (21, 30, 52), (21, 45, 80), (31, 45, 80), (40, 48, 80)]:
        g = bsa.Geometry(*grid)
        Q, K, V = bsa_gen.make_inputs("video", 0, 1, Hh, grid, d, device="cuda")
        dO = bsa_gen.grad_output(0, (1, Hh, g.L, d)).cuda()
        sp = BSAAttention(g, 0.5, 0.1, 0.9, 1, Hh, d)
        ms = timed(sp, Q, K, V, dO, 5, flush)
        fl = sp.flops()
        del sp
        dn = BSAAttention(g, 1.0, 1.0, 1.0, 1, Hh, d)
        dms = timed(dn, Q, K, V, dO, 2 if g.L > 100000 else 3, flush)
        dfl = dn.flops()
        del dn
        torch.cuda.empty_cache()
        rows.append({"grid": grid, "tokens": g.L, "bsa_ms": ms, "dense_ms": dms, "speedup": dms / ms,
                     "density": fl["density"], "ideal_speedup": 1 / fl["density"],
                     "bsa_tflops_executed": fl["total"] / (ms * 1e-3) / 1e12,
                     "dense_tflops": dfl["total"] / (dms * 1e-3) / 1e12})
        print(json.dumps(rows[-1]), file=sys.stderr)
    print(json.dumps({"sweep": "sequence length, Wan-1.3B-shaped (12 heads, d=128), r=.5 k=ceil(.1N) tau=.9, "
                               "G_video, fwd+bwd device ms", "paper_context": "12.85x -> 17.79x attention-training "
                               "speedup from 23K to 153K tokens on H100 (PAPER.md Fig. 6, P:282-288)", "rows": rows}))


if __name__ == "__main__":
    main()
