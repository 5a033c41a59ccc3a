"""Per-step timeline of one forward CTA (two softmax groups; BSA_TRACE build of libbsa):
BSA_LIB_PATH=dbg/libbsa_trace.so python tools/profiling/trace_fwd2.py [cta]
Slots (attn_fwd.cu FWD_TRACE): 0 producer issue, 1 QK issued, 2 PV issuer got P, 3 PV issued,
4+8g S ready seen by group g, 6+8g S in registers, 7+8g P buffer free seen, 5+8g P written."""
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
buf = torch.zeros(32 * 1024, dtype=torch.int64, device="cuda")
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 700
L.bsa_debug_trace_fwd(ctypes.c_void_p(buf.data_ptr()), cta)
layer.attend(Q, K, V)
torch.cuda.synchronize()
L.bsa_debug_trace_fwd(None, 0)
t = buf.view(32, 1024).cpu().numpy().astype(np.int64)
U = int((t[1] > 0).sum())
base = t[0, 0]
print(f"CTA {cta}: U = {U} steps, total {t[3, U - 1] - base} cycles, {(t[3, U - 1] - t[3, U // 4]) / (U - 1 - U // 4):.0f} cycles/step (steady)")
print("   u   prod  qk_iss  [g: s_seen s_regs pfree p_wr]  pv_got pv_iss")
for u in range(U // 2, min(U, U // 2 + 14)):
    gr = u & 1
    o = 8 * gr
    print(f"{u:4d} {t[0, u] - base:6d} {t[1, u] - base:7d}  [{gr}: {t[4 + o, u] - base:6d} {t[6 + o, u] - base:6d} "
          f"{t[7 + o, u] - base:6d} {t[5 + o, u] - base:6d}]  {t[2, u] - base:6d} {t[3, u] - base:6d}")
d = lambda a, b: np.median((t[a, U // 4:U - 1] - t[b, U // 4:U - 1]))
done = t[16, U // 4:U - 1]
seen = np.array([t[7 + 8 * (u & 1), u + 2] for u in range(U // 4, U - 3)])
print("PV(u) issued -> done (observer):", np.median(done[:len(seen)] - t[3, U // 4:U // 4 + len(seen)]),
      " PV(u) done -> P buffer free seen by group (step u+2):", np.median(seen - done[:len(seen)]))
print("median over steady steps (cycles): S ready->regs", [d(6 + 8 * k, 4 + 8 * k) for k in (0, 1)][0],
      " regs->P written", d(5, 6), d(13, 14), " pfree wait->P written", d(5, 7), " P written->PV issued", d(3, 2))
