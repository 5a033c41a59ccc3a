"""Full-size GPU parity at BASELINE.json's workloads, in the launch configuration bench.py times.

The 32k Wan-1.3B workload (configs[1]) runs through BSAAttention exactly as bench.py runs it (selection
+ forward + backward of all 12 heads, partition not cached). The oracle then checks:
  * selection for ALL heads (kept sets, donors, q2k lists bit-exact; near-ties < 1e-6 counted);
  * O, LSE, dQ, dK, dV for every row of two whole heads (the oracle is exact fp64, a few seconds a head).
The 75k Wan-14B workload (configs[2], the one bench.py shards over heads) is checked the same way on a
sample of heads.
"""

import math

import numpy as np
import pytest
import torch

import bsa_gen
import oracle as orc
import paper_2509_01085_b200 as bsa
from paper_2509_01085_b200.runner import BSAAttention
from parity_util import assert_close, assert_no_near_ties, compare_selection, record

pytestmark = pytest.mark.gpu

WAN13B = dict(grid=(21, 30, 52), block=(4, 4, 4), Hh=12, d=128, r=0.5, f=0.1, tau=0.9)
WAN14B = dict(grid=(21, 45, 80), block=(4, 4, 4), Hh=40, d=128, r=0.5, f=0.1, tau=0.9)


def _run_layer(cfg, seed, kind="video"):
    g = bsa.Geometry(*cfg["grid"], *cfg["block"])
    Q, K, V = bsa_gen.make_inputs(kind, seed, 1, cfg["Hh"], cfg["grid"], cfg["d"], device="cuda")
    dO = bsa_gen.grad_output(seed, (1, cfg["Hh"], g.L, cfg["d"])).cuda()
    layer = BSAAttention(g, cfg["r"], cfg["f"], cfg["tau"], 1, cfg["Hh"], cfg["d"], cache_partition=False)
    O = layer.forward(Q, K, V).clone()
    dQ, dK, dV = (x.clone() for x in layer.backward(dO))
    torch.cuda.synchronize()
    return g, layer, (Q, K, V, dO), (O, dQ, dK, dV)


def _check_heads(cfg, layer, inputs, outputs, heads, check_selection_heads, case):
    og = orc.Geom(*cfg["grid"], *cfg["block"])
    Q, K, V, dO = inputs
    O, dQ, dK, dV = outputs
    Hh, d, r = cfg["Hh"], cfg["d"], cfg["r"]
    # selection vs the oracle on the requested heads (bit-exact up to counted near-ties)
    Qh = Q[0, check_selection_heads].cpu().unsqueeze(0)
    Kh = K[0, check_selection_heads].cpu().unsqueeze(0)
    oq = orc.select_queries(og, r, Qh)
    okv = orc.select_kv(og, Qh, Kh, layer.k, cfg["tau"])
    hs = torch.tensor(check_selection_heads)
    near = compare_selection(og, r, layer.kept_tok[0, hs], layer.donor[0, hs], layer.q2k_num[0, hs],
                             layer.q2k_idx[0, hs], oq, okv, case=case)
    assert_no_near_ties(near, case)
    scale = float(np.float32(1.0 / math.sqrt(d)))
    N = layer.N
    for h in heads:
        kt = layer.kept_tok[0, h:h + 1].cpu().numpy()
        dn = layer.donor[0, h:h + 1].cpu().numpy()
        qn = layer.q2k_num[0, h:h + 1].cpu().numpy()
        qi = layer.q2k_idx[0, h:h + 1].cpu().numpy()
        qi = np.where(np.arange(N)[None, None, :] < qn[:, :, None], qi, -1)
        hq, hk, hv, hdo = (x[0, h:h + 1].cpu() for x in (Q, K, V, dO))
        Oref, lseref = orc.attn_fwd(og, r, hq, hk, hv, kt, dn, qn, qi, scale)
        assert_close(f"O[h{h}]", O[0, h:h + 1], Oref, case=case)
        lse_err = float(np.max(np.abs(layer.lse[0, h:h + 1].cpu().double().numpy() - lseref)))
        record(case, kind="lse", head=h, max_abs=lse_err)
        assert lse_err < 2e-2
        dQr, dKr, dVr = orc.attn_bwd(og, r, hq, hk, hv, hdo, kt, dn, qn, qi, scale)
        assert_close(f"dV[h{h}]", dV[0, h:h + 1], dVr, case=case)
        assert_close(f"dK[h{h}]", dK[0, h:h + 1], dKr, case=case)
        assert_close(f"dQ[h{h}]", dQ[0, h:h + 1], dQr, case=case)


FULL32K = [
    # case, seed, generator, (r, f, tau), heads checked element-wise
    ("wan13b_32k_seed0_video", 0, "video", (0.5, 0.1, 0.9), [0, 7]),
    ("wan13b_32k_seed1_video", 1, "video", (0.5, 0.1, 0.9), [3, 11]),
    ("wan13b_32k_seed0_iid", 0, "iid", (0.5, 0.1, 0.9), [1, 6]),
    ("wan13b_32k_r025", 2, "video", (0.25, 0.1, 0.9), [2, 9]),
    # the own-dense path (r = 1, k = N, tau = 1): the denominator of bench.py's speedup
    ("wan13b_32k_own_dense", 0, "video", (1.0, 1.0, 1.0), [0, 5]),
]


@pytest.mark.parametrize("case", FULL32K, ids=[c[0] for c in FULL32K])
def test_wan13b_32k_fullsize(case):
    name, seed, kind, (r, f, tau), heads = case
    cfg = dict(WAN13B, r=r, f=f, tau=tau)
    g, layer, inputs, outputs = _run_layer(cfg, seed=seed, kind=kind)
    assert layer.N == 624 and layer.k == bsa.resolve_k(f, 624)
    if r == 1.0 and f == 1.0 and tau == 1.0:
        assert int(layer.q2k_num.min()) == 624 and layer.Lq == g.L
    _check_heads(cfg, layer, inputs, outputs, heads=heads, check_selection_heads=list(range(cfg["Hh"])), case=name)


def test_wan14b_75k_sampled_heads():
    cfg = WAN14B
    g, layer, inputs, outputs = _run_layer(cfg, seed=3)
    assert layer.N == 6 * 12 * 20
    _check_heads(cfg, layer, inputs, outputs, heads=[5], check_selection_heads=[0, 5, 21, 39],
                 case="wan14b_75k_seed3")
