import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import bsa_gen, paper_2509_01085_b200 as bsa
from paper_2509_01085_b200.runner import BSAAttention
g = bsa.Geometry(21, 30, 52)
Q, K, V = bsa_gen.make_inputs("video", 0, 1, 12, (21, 30, 52), 128, device="cuda")
dO = bsa_gen.grad_output(0, (1, 12, g.L, 128)).cuda()
layer = BSAAttention(g, 0.5, 0.1, 0.9, 1, 12, 128)
layer.forward(Q, K, V); layer.backward(dO); torch.cuda.synchronize()
L = bsa.lib()
buf = torch.zeros(16 * 1024, dtype=torch.int64, device="cuda")
kn = layer.k2q_num.view(-1).cpu().numpy()
for cta in (100, 3000):
    buf.zero_()
    L.bsa_debug_trace_bwd(ctypes.c_void_p(buf.data_ptr()), cta)
    layer.backward(dO); torch.cuda.synchronize()
    t = buf.view(16, 1024).cpu().numpy().astype(np.int64)
    C = int((t[1] > 0).sum())
    t0 = t[0, 0]
    print(f"CTA {cta}: k2q_num={kn[cta]} chunks={C}; total cycles {t[7, C-1]-t0}; per chunk {(t[7, C-1]-t0)/max(C,1):.0f}")
    names = ["prod", "sd_commit", "mma_got_ps", "dq_commit", "c_got_sd", "c_arr_ps", "c_got_dq", "c_dq_done", "ldS", "cmp", "psfree", "mma_got_c", "landed"]
    lat = t[12, :C] - t[0, :C]
    print('load latency (landed - prod) per chunk:', lat.tolist())
    for c in range(min(C, 8)):
        print(c, " ".join(f"{n}={t[i, c]-t0:7d}" for i, n in enumerate(names)))
L.bsa_debug_trace_bwd(None, 0)
