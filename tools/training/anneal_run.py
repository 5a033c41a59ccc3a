"""Synthetic DiT-block training run through the paper's sparsity anneal (PAPER.md
P:253: "training begins with full attention, and every 30 steps, the sparsity is increased by 0.03 until
reaching a maximum of 0.9 ... the number of top-k tokens selected is gradually reduced from the total number of
blocks to 0.1x the total").

One step = DiTAttentionBlock forward (LayerNorm -> fused QKV projection -> BSA -> out-projection -> residual),
MSE loss against a fixed synthetic target, backward, AdamW update. The knobs (r, k, tau) follow
training.AnnealSchedule (reading C27). Per step it records the library's own device times of the selection,
forward and backward kernels (bsa_timing_*), the whole step's device time, the realised density and the loss.

    python tools/training/anneal_run.py --steps 1000 --out profiles/r02_anneal.json
"""
import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bsa_gen  # noqa: E402
import paper_2509_01085_b200 as bsa  # noqa: E402
from bench import KERNEL_NAMES, SELECTION_IDS  # noqa: E402
from paper_2509_01085_b200.training import AnnealSchedule, DiTAttentionBlock  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--grid", default="21,30,52")
    ap.add_argument("--heads", type=int, default=12)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "anneal.json"))
    args = ap.parse_args()
    grid = tuple(int(x) for x in args.grid.split(","))
    Hh, d = args.heads, args.d
    g = bsa.Geometry(*grid)
    torch.manual_seed(0)
    dev = torch.device("cuda", 0)
    sched = AnnealSchedule()
    blk = DiTAttentionBlock(g, 1, Hh, d, schedule=sched, device=dev)
    C = Hh * d
    with torch.no_grad():  # projections near the identity, so attention sees the latents' video structure
        for lin in (blk.qkv,):
            w = torch.eye(C, device=dev).repeat(3, 1) + 0.05 * torch.randn(3 * C, C, device=dev)
            lin.weight.copy_(w.to(lin.weight.dtype))
            lin.bias.zero_()
    Q, _, _ = bsa_gen.make_inputs("video", 0, 1, Hh, grid, d, device=dev)  # [1, Hh, L, d] structured latents
    x = Q.transpose(1, 2).reshape(1, g.L, C).contiguous()
    y = torch.randn_like(x)
    opt = torch.optim.AdamW(blk.parameters(), lr=1e-4)
    lib = bsa.lib()
    nk = len(KERNEL_NAMES)
    ms = (ctypes.c_double * nk)()
    recs = []
    t_wall = time.time()
    for step in range(args.steps):
        blk.set_step(step)
        r, f, tau = sched.knobs(step)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        lib.bsa_timing_read(None, None, 0)
        lib.bsa_timing_enable(1)
        e0.record()
        out = blk(x)
        loss = torch.nn.functional.mse_loss(out.float(), y.float())
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        e1.record()
        torch.cuda.synchronize()
        lib.bsa_timing_enable(0)
        lib.bsa_timing_read(ms, None, nk)
        lay = blk.attn._layer()
        fl = lay.flops()
        rec = {"step": step, "r": r, "k_frac": f, "k": lay.k, "tau": tau, "N": lay.N,
               "selection_ms": sum(ms[i] for i in SELECTION_IDS), "fwd_ms": ms[7] + ms[8] + ms[12] + ms[14] + ms[17],
               "bwd_ms": ms[9] + ms[10] + ms[11] + ms[15] + ms[16], "step_ms": e0.elapsed_time(e1), "pair_density": fl["density"],
               "mean_admitted_blocks": lay.sparsity()["mean_admitted_blocks"], "loss": float(loss.item())}
        rec["attn_ms"] = rec["selection_ms"] + rec["fwd_ms"] + rec["bwd_ms"]
        recs.append(rec)
        if step % 100 == 0:
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in rec.items()}), flush=True)
    summary = []
    for s0 in range(0, args.steps, 100):
        w = recs[s0:s0 + 100]
        summary.append({"steps": [s0, s0 + len(w) - 1], "r": [w[0]["r"], w[-1]["r"]], "k": [w[0]["k"], w[-1]["k"]],
                        **{k: sum(x[k] for x in w) / len(w) for k in ("selection_ms", "fwd_ms", "bwd_ms", "attn_ms",
                                                                     "step_ms", "pair_density", "loss")}})
    doc = {"what": "DiTAttentionBlock (LayerNorm -> fused QKV -> BSA -> out-proj -> residual) trained with AdamW "
                   "through the P:253 anneal (training.AnnealSchedule, reading C27); synthetic G_video latents, "
                   "MSE to a fixed random target; per-step device times from the library's event timing",
           "grid": list(grid), "heads": Hh, "d": d, "steps": args.steps, "wall_s": time.time() - t_wall,
           "gpu": torch.cuda.get_device_name(0), "summary_per_100_steps": summary, "per_step": recs}
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    json.dump(doc, open(args.out, "w"), indent=1)
    print("wrote", args.out, "wall", round(doc["wall_s"], 1), "s")


if __name__ == "__main__":
    main()
