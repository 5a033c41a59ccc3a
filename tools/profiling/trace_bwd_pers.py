"""Per-chunk timeline of one persistent backward CTA (BSA_TRACE build): which role sets the chunk period.
BSA_LIB_PATH=vso/v_trace.so python tools/profiling/trace_bwd_pers.py [cta]"""
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
dO = bsa_gen.grad_output(0, (1, 12, g.L, 128)).cuda()
layer = BSAAttention(g, 0.5, 0.1, 0.9, 1, 12, 128)
layer.forward(Q, K, V)
layer.backward(dO)
torch.cuda.synchronize()
L = bsa.lib()
buf = torch.zeros(16 * 1024, dtype=torch.int64, device="cuda")
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 5
L.bsa_debug_trace_bwd(ctypes.c_void_p(buf.data_ptr()), cta)
layer.backward(dO)
torch.cuda.synchronize()
L.bsa_debug_trace_bwd(None, 0)
t = buf.view(16, 1024).cpu().numpy().astype(np.int64)
names = {0: "prod_issue", 1: "sd_commit", 2: "mma_got_ps", 3: "dq_commit", 4: "sm_got_sd", 5: "sm_arr_ps",
         6: "dr_got_dq", 7: "dr_done", 8: "sm_ldS", 9: "sm_cmp", 10: "sm_psfree", 11: "sd_got_c"}
C = int((t[7] > 0).sum())
t0 = t[0, 0]
per = np.diff(t[7, :C])
print(f"CTA {cta}: {C} chunks, {t[7, C - 1] - t0} cycles, median chunk period {np.median(per):.0f}")
# median over steady-state chunks of each event relative to the chunk's S/dP commit
rel = {n: int(np.median(t[i, 10:C - 5] - t[1, 10:C - 5])) for i, n in names.items()}
print("median offsets from sd_commit(c):", rel)
# median gaps between consecutive chunks per event
gaps = {n: int(np.median(np.diff(t[i, 10:C - 5]))) for i, n in names.items()}
print("median period per event:", gaps)
