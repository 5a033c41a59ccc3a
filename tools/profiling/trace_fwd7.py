import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import bsa_gen, paper_2509_01085_b200 as bsa
from paper_2509_01085_b200.runner import BSAAttention
g = bsa.Geometry(21, 30, 52)
Q, K, V = bsa_gen.make_inputs("video", 0, 1, 12, (21, 30, 52), 128, device="cuda")
layer = BSAAttention(g, 0.5, 0.1, 0.9, 1, 12, 128)
layer.forward(Q, K, V); torch.cuda.synchronize()
L = bsa.lib()
buf = torch.zeros(32 * 1024, dtype=torch.int64, device="cuda")
cta = 700
L.bsa_debug_trace_fwd(ctypes.c_void_p(buf.data_ptr()), cta)
layer.attend(Q, K, V); torch.cuda.synchronize()
t = buf.view(32, 1024).cpu().numpy().astype(np.int64)
U = int((t[1] > 0).sum())
u0 = U // 2
base = t[8, u0 - 1]
print("per warp: ldS, compute done, p_free done, rescale done, P written")
for u in range(u0, u0 + 8):
    print(u, f"qk_iss {t[1,u]-base} got_p {t[2,u]-base} pv_iss {t[3,u]-base}")
    for w in range(4):
        r = [t[12 + w, u], t[16 + w, u], t[20 + w, u], t[24 + w, u], t[8 + w, u]]
        print("    w", w, " ".join(f"{x - base:6d}" for x in r))
L.bsa_debug_trace_fwd(None, 0)
