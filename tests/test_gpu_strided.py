"""Strided operands at the C ABI (include/bsa.h bsa_tensor): the problem is stated per head,
Q, K, V in R^{L x d}, so a model's own layouts go in without a copy:

  * contiguous [B, Hh, L, d];
  * a DiT's [B, L, Hh, d] activations, passed as x.transpose(1, 2) (B = 2 also exercises the backward's
    per-batch launches, since there the batch stride does not continue the head stride);
  * the Q / K / V slices of a fused [B, L, 3, Hh, d] projection, with outputs written into [B, L, Hh, d].

Selection, O, dK and dV must be bit-identical across layouts (same kernels, same order); dQ is reduced through
L2 in a non-deterministic order, so it is compared with the parity tolerance; one layout is also checked
against the fp64 oracle.
"""

import math

import numpy as np
import pytest
import torch

import bsa_gen
import oracle as orc
import paper_2509_01085_b200 as bsa
from paper_2509_01085_b200.runner import BSAAttention
from parity_util import assert_close, rel_err_all

pytestmark = pytest.mark.gpu

GRID, BLOCK, B, HH, D, R, F, TAU = (6, 10, 14), (4, 4, 4), 2, 3, 128, 0.5, 0.3, 0.9


def _inputs():
    Q, K, V = bsa_gen.make_inputs("video", 11, B, HH, GRID, D, device="cuda")
    dO = bsa_gen.grad_output(11, (B, HH, Q.shape[2], D)).cuda()
    return Q, K, V, dO


def _run(Q, K, V, dO, outs):
    g = bsa.Geometry(*GRID, *BLOCK)
    lay = BSAAttention(g, R, F, TAU, B, HH, D, cache_partition=False)
    O = lay.forward(Q, K, V, out=outs[0])
    dQ, dK, dV = lay.backward(dO, out=outs[1:])
    torch.cuda.synchronize()
    sel = tuple(x.clone() for x in (lay.kept_tok, lay.donor, lay.q2k_num, lay.q2k_idx, lay.k2q_num))
    return sel, tuple(x.contiguous().clone() for x in (O, dQ, dK, dV))


def _bhld(shape_bshd):
    return torch.empty(shape_bshd, dtype=torch.bfloat16, device="cuda")


def test_layouts_agree_and_match_oracle():
    Q, K, V, dO = _inputs()
    L = Q.shape[2]
    ref_sel, ref = _run(Q, K, V, dO, [torch.empty_like(Q) for _ in range(4)])
    # [B, L, Hh, d] model layout, viewed as [B, Hh, L, d]
    to_bshd = lambda x: x.transpose(1, 2).contiguous()  # noqa: E731
    Qs, Ks, Vs, dOs = (to_bshd(x).transpose(1, 2) for x in (Q, K, V, dO))
    assert Qs.stride() == (L * HH * D, D, HH * D, 1)
    outs = [_bhld((B, L, HH, D)).transpose(1, 2) for _ in range(4)]
    sel_s, got_s = _run(Qs, Ks, Vs, dOs, outs)
    # fused QKV projection [B, L, 3, Hh, d]
    qkv = torch.stack([to_bshd(x) for x in (Q, K, V)], dim=2)
    Qf, Kf, Vf = (qkv[:, :, i].transpose(1, 2) for i in range(3))
    assert Qf.stride()[2] == 3 * HH * D
    sel_f, got_f = _run(Qf, Kf, Vf, dOs, [_bhld((B, L, HH, D)).transpose(1, 2) for _ in range(4)])
    for sel, got, name in ((sel_s, got_s, "bshd"), (sel_f, got_f, "fused_qkv")):
        for a, b in zip(sel, ref_sel):
            assert torch.equal(a, b), name
        for t, (a, b) in zip(("O", "dK", "dV"), ((got[0], ref[0]), (got[2], ref[2]), (got[3], ref[3]))):
            assert torch.equal(a.view(torch.int16), b.view(torch.int16)), (name, t)
        e = rel_err_all(got[1], ref[1].double().cpu().numpy())
        assert e["max_over_max"] < 1e-2 and e["mean_over_rms"] < 1e-3, (name, e)
    # the strided run against the fp64 oracle (batch element 1)
    og = orc.Geom(*GRID, *BLOCK)
    k = bsa.resolve_k(F, orc.sizes(og, R)[0])
    Qn, Kn, Vn, dOn = (x[1].float().cpu().double().numpy() for x in (Q, K, V, dO))
    qs = orc.select_queries(og, R, Qn)
    kv = orc.select_kv(og, Qn, Kn, k, TAU)
    assert np.array_equal(sel_s[0][1].cpu().numpy(), qs["kept_tok"])
    assert np.array_equal(sel_s[2][1].cpu().numpy(), kv["q2k_num"])
    sc = 1.0 / math.sqrt(D)
    Or, _ = orc.attn_fwd(og, R, Qn, Kn, Vn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], sc)
    dQr, dKr, dVr = orc.attn_bwd(og, R, Qn, Kn, Vn, dOn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], sc)
    for name, a, ref_ in (("O", got_s[0], Or), ("dQ", got_s[1], dQr), ("dK", got_s[2], dKr), ("dV", got_s[3], dVr)):
        assert_close(name, a[1], ref_, case="strided_bshd_B2")


def test_ulysses_single_rank_reads_model_layout_in_place():
    """UlyssesBSA at P = 1: [B, L, Hh, d] in and out with no relayout kernel and no exchange; same numbers as the
    plain layer on the contiguous layout."""
    from paper_2509_01085_b200.ulysses import UlyssesBSA
    Q, K, V, dO = _inputs()
    g = bsa.Geometry(*GRID, *BLOCK)
    u = UlyssesBSA(g, R, F, TAU, B, HH, D)
    lib = bsa.lib()
    bshd = lambda x: x.transpose(1, 2).contiguous()  # noqa: E731
    n0 = lib.bsa_launch_count()
    lib.bsa_timing_read(None, None, 0)
    lib.bsa_timing_enable(1)
    O = u.forward(bshd(Q), bshd(K), bshd(V))
    dQ, dK, dV = u.backward(bshd(dO))
    torch.cuda.synchronize()
    import ctypes
    n = 14
    ms, cnt = (ctypes.c_double * n)(), (ctypes.c_int32 * n)()
    lib.bsa_timing_read(ms, cnt, n)
    lib.bsa_timing_enable(0)
    assert cnt[13] == 0  # BSA_K_SP_RELAYOUT: nothing reordered
    assert lib.bsa_launch_count() > n0
    ref_sel, ref = _run(Q, K, V, dO, [torch.empty_like(Q) for _ in range(4)])
    for a, b in ((O, ref[0]), (dK, ref[2]), (dV, ref[3])):
        assert torch.equal(a.transpose(1, 2).contiguous().view(torch.int16), b.view(torch.int16))
    e = rel_err_all(dQ.transpose(1, 2), ref[1].double().cpu().numpy())
    assert e["max_over_max"] < 1e-2
