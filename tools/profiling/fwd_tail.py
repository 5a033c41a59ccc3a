"""Tail of the persistent attn_fwd: per-CTA start / end (globaltimer stamps of a -DBSA_TRACE build) over one 32k
forward, plus the union-length spread of its tiles. BSA_LIB_PATH=variant.so python tools/profiling/fwd_tail.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bsa_gen  # noqa: E402
import paper_2509_01085_b200 as bsa  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2509_01085_b200.runner import BSAAttention  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "wan1.3b_32k"
cfg = CONFIGS[name]
g = bsa.Geometry(*cfg["grid"], *cfg["block"])
Q, K, V = bsa_gen.make_inputs(cfg["kind"], 0, cfg["B"], cfg["Hh"], cfg["grid"], cfg["d"], device="cuda")
layer = BSAAttention(g, cfg["r"], cfg["f"], cfg["tau"], cfg["B"], cfg["Hh"], cfg["d"])
for _ in range(2):
    layer.forward(Q, K, V)
torch.cuda.synchronize()
L = bsa.lib()
ncta = torch.cuda.get_device_properties(0).multi_processor_count
for rep in range(3):
    buf = torch.zeros(ncta * 2, dtype=torch.int64, device="cuda")
    L.bsa_debug_trace_fwd(ctypes.c_void_p(buf.data_ptr()), -1)
    layer.forward(Q, K, V)
    torch.cuda.synchronize()
    L.bsa_debug_trace_fwd(None, 0)
    t = buf.view(ncta, 2).cpu().numpy().astype(np.int64)
    t0 = t[:, 0].min()
    st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    print(f"{name} rep {rep}: start max {st.max():.1f} us; end min {en.min():.1f} p10 {np.percentile(en, 10):.1f} "
          f"median {np.median(en):.1f} p90 {np.percentile(en, 90):.1f} max {en.max():.1f} us; "
          f"SM-idle fraction in the tail {np.mean(en.max() - en) / en.max():.3f}")
