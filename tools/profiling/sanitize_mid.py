"""One selection + forward + backward on a ragged mid-size geometry (several tiles, truncated edge
blocks, two KV blocks per backward CTA) for compute-sanitizer; no oracle (the parity tests cover values)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bsa_gen  # noqa: E402
import paper_2509_01085_b200 as bsa  # noqa: E402

grid, block, Hh, d, r, tau = (6, 10, 14), (4, 4, 4), 2, 128, 0.5, 0.9
g = bsa.Geometry(*grid, *block)
Qh, Kh, Vh = bsa_gen.make_inputs("video", 0, 1, Hh, grid, d)
Q, K, V = Qh.cuda(), Kh.cuda(), Vh.cuda()
N = bsa.bsa_sizes(g, r)[0]
k = bsa.resolve_k(0.3, N)
sel = bsa.select(g, r, k, tau, Q, K)
O, lse = bsa.bsa_attn_fwd(g, r, Q, K, V, sel.part["kept_off"], sel.kept_tok, sel.donor, sel.q2k_num, sel.q2k_idx,
                          q_packed=sel.q_packed)
dO = bsa_gen.grad_output(0, (1, Hh, g.L, d)).cuda()
dQ, dK, dV = bsa.bsa_attn_bwd(g, r, Q, K, V, O, dO, sel.part["kept_off"], sel.kept_tok, sel.donor, sel.q2k_num,
                              sel.q2k_idx, sel.k2q_num, sel.k2q_idx, lse, q_packed=sel.q_packed)
torch.cuda.synchronize()
print("mid ok", float(O.float().abs().sum()), float(dQ.float().abs().sum()))
