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
ncta = ((layer.N + 1) // 2) * 12  # BWD_NB = 2 KV blocks per CTA
buf = torch.zeros(ncta * 16, dtype=torch.int64, device="cuda")
L.bsa_debug_trace_bwd(ctypes.c_void_p(buf.data_ptr()), -1)
layer.backward(dO); torch.cuda.synchronize()
L.bsa_debug_trace_bwd(None, 0)
t = buf.view(ncta, 16).cpu().numpy().astype(np.int64)
t0 = t[:, 0].min(); span = t[:, 1].max() - t0
dur = t[:, 1] - t[:, 0]
nch = t[:, 3]
print(f"kernel span {span/1e3:.1f} us; sum CTA dur {dur.sum()/1e3:.0f} us; SM-busy fraction {dur.sum()/(148*span):.3f}")
for k in (0, 1, 4, 8, 12, 16, 24):
    m = nch == k
    if m.any(): print(f"  nchunks={k:3d}: {m.sum():5d} CTAs, mean dur {dur[m].mean()/1e3:.2f} us")
A = np.vstack([np.ones_like(nch), nch]).T.astype(float)
coef = np.linalg.lstsq(A, dur.astype(float), rcond=None)[0]
print(f"fit: dur = {coef[0]/1e3:.2f} us + {coef[1]/1e3:.3f} us * nchunks  (at 1.92 GHz: {coef[0]*1.92:.0f} + {coef[1]*1.92:.0f} cyc)")
# per SM: gaps between consecutive CTAs
gaps = []
for s in range(148):
    m = t[:, 2] == s
    tt = t[m]; tt = tt[np.argsort(tt[:, 0])]
    gaps += list(tt[1:, 0] - tt[:-1, 1])
gaps = np.array(gaps)
print(f"inter-CTA gap per SM: median {np.median(gaps)/1e3:.2f} us, mean {gaps.mean()/1e3:.2f} us")
ends = np.sort(t[:, 1] - t0)
print(f"tail: last 148 CTAs end within {(ends[-1]-ends[-148])/1e3:.1f} us")

names = {11: "first stage issued", 8: "first chunk landed", 9: "first S/dP ready", 4: "prologue done", 5: "softmax loop done", 6: "dK/dV stored", 7: "drain done", 1: "end"}
for k in (4, 11, 8, 9, 5, 6, 7, 1):
    d = (t[:, k] - t[:, 0]) / 1e3
    m = nch == 12
    print(f"  t[{names[k]:18s}] - start: mean {d.mean():7.2f} us   (nchunks=12: {d[m].mean():7.2f})")
