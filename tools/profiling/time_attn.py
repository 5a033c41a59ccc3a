"""Per-kernel device times of one workload through BSAAttention (library event timing), for A/B runs of
library variants: BSA_LIB_PATH=variant.so python tools/profiling/time_attn.py [config] [steps]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bsa_gen  # noqa: E402
import paper_2509_01085_b200 as bsa  # noqa: E402
from bench import CONFIGS, KERNEL_NAMES  # noqa: E402
from paper_2509_01085_b200.runner import BSAAttention  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "wan1.3b_32k"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = CONFIGS[name]
g = bsa.Geometry(*cfg["grid"], *cfg["block"])
Q, K, V = bsa_gen.make_inputs(cfg["kind"], 0, cfg["B"], cfg["Hh"], cfg["grid"], cfg["d"], device="cuda")
dO = bsa_gen.grad_output(0, (cfg["B"], cfg["Hh"], g.L, cfg["d"])).cuda()
if os.environ.get("BSA_BWD_PATH") == "ds":
    bsa.set_bwd_path(bsa.BWD_DS)
dense = os.environ.get("BSA_DENSE") == "1"  # the own dense path: r = 1, k = N, tau = 1
layer = BSAAttention(g, *((1.0, 1.0, 1.0) if dense else (cfg["r"], cfg["f"], cfg["tau"])), cfg["B"], cfg["Hh"], cfg["d"])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    layer.forward(Q, K, V)
    layer.backward(dO)
torch.cuda.synchronize()
L = bsa.lib()
L.bsa_timing_read(None, None, 0)
L.bsa_timing_enable(1)
for _ in range(steps):
    flush.zero_()
    layer.forward(Q, K, V)
    layer.backward(dO)
torch.cuda.synchronize()
L.bsa_timing_enable(0)
nk = len(KERNEL_NAMES)
ms = (ctypes.c_double * nk)()
L.bsa_timing_read(ms, None, nk)
print(os.path.basename(os.environ.get("BSA_LIB_PATH", "libbsa.so")), name + (" dense" if dense else ""),
      os.environ.get("BSA_BWD_PATH", "reduce"),
      {n: round(ms[i] / steps, 4) for i, n in enumerate(KERNEL_NAMES) if ms[i] > 0})
