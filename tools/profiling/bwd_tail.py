"""Tail of the persistent attn_bwd: per-CTA start / end (globaltimer stamps of a -DBSA_TRACE build, slots 4 and
7) over one 32k backward. BSA_LIB_PATH=variant.so python tools/profiling/bwd_tail.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bsa_gen  # noqa: E402
import paper_2509_01085_b200 as bsa  # noqa: E402
from paper_2509_01085_b200.runner import BSAAttention  # noqa: E402

g = bsa.Geometry(21, 30, 52)
Q, K, V = bsa_gen.make_inputs("video", 0, 1, 12, (21, 30, 52), 128, device="cuda")
dO = bsa_gen.grad_output(0, (1, 12, g.L, 128)).cuda()
layer = BSAAttention(g, 0.5, 0.1, 0.9, 1, 12, 128)
for _ in range(2):
    layer.forward(Q, K, V)
    layer.backward(dO)
torch.cuda.synchronize()
L = bsa.lib()
ncta = torch.cuda.get_device_properties(0).multi_processor_count
for rep in range(3):
    buf = torch.zeros(ncta * 16, dtype=torch.int64, device="cuda")
    L.bsa_debug_trace_bwd(ctypes.c_void_p(buf.data_ptr()), -1)
    layer.backward(dO)
    torch.cuda.synchronize()
    L.bsa_debug_trace_bwd(None, 0)
    t = buf.view(ncta, 16).cpu().numpy().astype(np.int64)
    t0 = t[:, 4].min()
    st, en = (t[:, 4] - t0) / 1e3, (t[:, 7] - t0) / 1e3
    print(f"rep {rep}: start max {st.max():.1f} us; end min {en.min():.1f} p10 {np.percentile(en, 10):.1f} "
          f"median {np.median(en):.1f} p90 {np.percentile(en, 90):.1f} max {en.max():.1f} us; "
          f"SM-idle fraction in the tail {np.mean(en.max() - en) / en.max():.3f}")
nq = layer.k2q_num.view(-1).cpu().numpy()
print(f"items {nq.size}: k2q length mean {nq.mean():.1f} max {nq.max()} (chunks ~ length / 4)")
