"""Per-CTA timeline of the forward (BSA_TRACE build, trace mode -1):
BSA_LIB_PATH=dbg/libbsa_trace.so python tools/profiling/cta_times_fwd.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bsa_gen  # noqa: E402
import paper_2509_01085_b200 as bsa  # noqa: E402
from paper_2509_01085_b200.runner import BSAAttention  # noqa: E402

g = bsa.Geometry(21, 30, 52)
Q, K, V = bsa_gen.make_inputs("video", 0, 1, 12, (21, 30, 52), 128, device="cuda")
layer = BSAAttention(g, 0.5, 0.1, 0.9, 1, 12, 128)
layer.forward(Q, K, V)
torch.cuda.synchronize()
L = bsa.lib()
ncta = ((layer.N + 3) // 4) * 12
buf = torch.zeros(ncta * 16, dtype=torch.int64, device="cuda")
L.bsa_debug_trace_fwd(ctypes.c_void_p(buf.data_ptr()), -1)
layer.attend(Q, K, V)
torch.cuda.synchronize()
L.bsa_debug_trace_fwd(None, 0)
t = buf.view(ncta, 16).cpu().numpy().astype(np.int64)
dur = (t[:, 3] - t[:, 0]) / 1e3
U = t[:, 5]
pro = (t[:, 1] - t[:, 0]) / 1e3
epi = (t[:, 3] - t[:, 2]) / 1e3
span = (t[:, 3].max() - t[:, 0].min()) / 1e3
print(f"kernel span {span:.1f} us; SM-busy fraction {dur.sum() / (148 * span):.3f}")
A = np.vstack([np.ones_like(U), U]).T.astype(float)
coef = np.linalg.lstsq(A, dur, rcond=None)[0]
print(f"fit: dur = {coef[0]:.2f} us + {coef[1] * 1e3:.1f} ns * U   (mean U {U.mean():.0f}, mean dur {dur.mean():.1f} us)")
print(f"prologue (start -> first S ready) mean {pro.mean():.2f} us; epilogue (last PV issued -> end) mean {epi.mean():.2f} us")
un = (t[:, 6] - t[:, 0]) / 1e3
ql = (t[:, 7] - t[:, 0]) / 1e3
st = lambda k: ((t[:, k] - t[:, 0]) / 1e3).mean()
print(f"  start -> masks/zero issued {st(8):.2f} us; -> first barrier (kept_off, q2k loads) {st(9):.2f} us; -> bitmaps {st(10):.2f} us")
print(f"  start -> union list built {un.mean():.2f} us; -> Q^s in TMEM {ql.mean():.2f} us; -> first S ready {pro.mean():.2f} us")
ends = np.sort(t[:, 3] - t[:, 0].min()) / 1e3
print(f"tail: last 148 CTAs end within {ends[-1] - ends[-148]:.1f} us")
