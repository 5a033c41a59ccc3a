"""One selection (a1-a6) of a bench workload, for ncu captures of the selection kernels.

    ncu --set full -k regex:'k_admit|k_scores|k_select_queries' python tools/profiling/sel_once.py long_147k
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bsa_gen  # noqa: E402
import paper_2509_01085_b200 as bsa  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2509_01085_b200.runner import BSAAttention  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "wan1.3b_32k"]
g = bsa.Geometry(*cfg["grid"], *cfg["block"])
Q, K, V = bsa_gen.make_inputs(cfg["kind"], 0, cfg["B"], cfg["Hh"], cfg["grid"], cfg["d"], device="cuda")
layer = BSAAttention(g, cfg["r"], cfg["f"], cfg["tau"], cfg["B"], cfg["Hh"], cfg["d"])
layer.select(Q, K)
torch.cuda.synchronize()
print("ok", layer.N, layer.k)
if len(sys.argv) > 2 and sys.argv[2] == "time":
    import ctypes
    L = bsa.lib()
    for _ in range(2):
        layer.select(Q, K)
    torch.cuda.synchronize()
    L.bsa_timing_read(None, None, 0)
    L.bsa_timing_enable(1)
    for _ in range(5):
        layer.select(Q, K)
    torch.cuda.synchronize()
    L.bsa_timing_enable(0)
    names = ["partition", "select_queries", "pool", "scores", "admit", "k2q"]
    ms = (ctypes.c_double * 6)()
    L.bsa_timing_read(ms, None, 6)
    print({n: round(ms[i] / 5, 4) for i, n in enumerate(names)})
