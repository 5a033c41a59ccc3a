"""Training integration: the anneal schedule of P:253 (host logic, CPU) and the
autograd function over the C-ABI forward/backward (GPU, against the fp64 oracle)."""

import math

import numpy as np
import pytest
import torch

import bsa_gen
import oracle as orc
from paper_2509_01085_b200 import Geometry, resolve_k
from paper_2509_01085_b200.training import AnnealSchedule


def test_anneal_schedule_matches_p253():
    s = AnnealSchedule()
    # "training begins with full attention, and every 30 steps, the sparsity is increased by 0.03"
    assert s.sparsity_at_step(0) == 0.0 and s.sparsity_at_step(29) == 0.0
    assert math.isclose(s.sparsity_at_step(30), 0.03) and math.isclose(s.sparsity_at_step(60), 0.06)
    # "until reaching a maximum of 0.9"
    assert math.isclose(s.sparsity_at_step(900), 0.9) and math.isclose(s.sparsity_at_step(10_000), 0.9)
    # "the number of top-k tokens ... gradually reduced from the total number of blocks to 0.1x the total"
    assert s.kv_fraction_at_step(0) == 1.0 and math.isclose(s.kv_fraction_at_step(s.horizon), 0.1)
    assert math.isclose(s.kv_fraction_at_step(s.horizon // 2), 0.55)
    assert s.knobs(0) == (1.0, 1.0, 1.0)  # full attention
    r, f, tau = s.knobs(30)
    assert math.isclose(r, 0.97) and math.isclose(f, 0.97) and tau == 0.9
    r, f, _ = s.knobs(900)
    assert r == 0.5 and math.isclose(f, 0.1)  # the paper's end point: r = 0.5, k = 0.1 N
    prev = (2.0, 2.0)
    for step in range(0, 2000, 7):  # monotone: never less sparse later
        r, f, _ = s.knobs(step)
        assert r <= prev[0] + 1e-12 and f <= prev[1] + 1e-12
        prev = (r, f)
    with pytest.raises(ValueError):
        s.sparsity_at_step(-1)


@pytest.mark.gpu
@pytest.mark.parametrize("step", [0, 450, 2000])
def test_autograd_matches_oracle(step):
    from parity_util import assert_close
    from paper_2509_01085_b200.training import AnnealSchedule, BSASelfAttention
    grid, Hh, d = (8, 12, 16), 2, 128
    sched = AnnealSchedule()
    r, f, tau = sched.knobs(step)
    attn = BSASelfAttention(Geometry(*grid), 1, Hh, d, schedule=sched)
    attn.set_step(step)
    Q, K, V = (x.cuda().requires_grad_(True) for x in bsa_gen.make_inputs("video", 2, 1, Hh, grid, d))
    dO = bsa_gen.grad_output(2, (1, Hh, Q.shape[2], d)).cuda()
    O = attn(Q, K, V)
    O.backward(dO)
    torch.cuda.synchronize()
    og = orc.Geom(*grid, 4, 4, 4)
    k = resolve_k(f, orc.sizes(og, r)[0])
    Qn, Kn, Vn, dOn = (x.detach()[0].float().cpu().double().numpy() for x in (Q, K, V, dO))
    qs = orc.select_queries(og, r, Qn)
    kv = orc.select_kv(og, Qn, Kn, k, tau)
    sc = 1.0 / math.sqrt(d)
    Or, _ = orc.attn_fwd(og, r, Qn, Kn, Vn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], sc)
    dQr, dKr, dVr = orc.attn_bwd(og, r, Qn, Kn, Vn, dOn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"],
                                 sc)
    assert_close("O", O.detach()[0], Or)
    assert_close("dQ", Q.grad[0], dQr)
    assert_close("dK", K.grad[0], dKr)
    assert_close("dV", V.grad[0], dVr)


@pytest.mark.gpu
def test_autograd_rejects_stale_backward():
    from paper_2509_01085_b200 import BSAError
    from paper_2509_01085_b200.training import BSASelfAttention
    grid, Hh, d = (4, 8, 8), 1, 64
    attn = BSASelfAttention(Geometry(*grid, 2, 4, 4), 1, Hh, d, r=0.5, f=0.5, tau=0.9)
    Q, K, V = (x.cuda().requires_grad_(True) for x in bsa_gen.make_inputs("iid", 0, 1, Hh, grid, d))
    O1 = attn(Q, K, V)
    attn(Q, K, V)  # second forward through the same layer
    with pytest.raises(BSAError):
        O1.sum().backward()


@pytest.mark.gpu
def test_fused_qkv_mid_anneal_matches_oracle():
    """The DiT block's attention path at a mid-anneal step (step 450: r = 0.55, k = 0.55 N): a fused
    [B, L, 3, Hh, d] projection goes into the library as strided Q/K/V views, O comes back in [B, L, Hh, d], and
    autograd's d(qkv) is written slice by slice -- all against the fp64 oracle on the same values."""
    from parity_util import assert_close
    from paper_2509_01085_b200.training import AnnealSchedule, BSASelfAttention
    grid, Hh, d, step = (8, 12, 16), 2, 128, 450
    sched = AnnealSchedule()
    r, f, tau = sched.knobs(step)
    attn = BSASelfAttention(Geometry(*grid), 1, Hh, d, schedule=sched)
    attn.set_step(step)
    Q, K, V = bsa_gen.make_inputs("video", 6, 1, Hh, grid, d)
    qkv = torch.stack([x.transpose(1, 2) for x in (Q, K, V)], dim=2).cuda().requires_grad_(True)  # [1, L, 3, Hh, d]
    L = qkv.shape[1]
    dO = bsa_gen.grad_output(6, (1, L, Hh, d)).cuda()
    O = attn.forward_qkv(qkv)
    assert O.shape == (1, L, Hh, d)
    O.backward(dO)
    torch.cuda.synchronize()
    og = orc.Geom(*grid, 4, 4, 4)
    k = resolve_k(f, orc.sizes(og, r)[0])
    Qn, Kn, Vn = (x[0].double().numpy() for x in (Q, K, V))
    dOn = dO[0].transpose(0, 1).double().cpu().numpy()  # [Hh, L, d]
    qs = orc.select_queries(og, r, Qn)
    kv = orc.select_kv(og, Qn, Kn, k, tau)
    sc = 1.0 / math.sqrt(d)
    Or, _ = orc.attn_fwd(og, r, Qn, Kn, Vn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], sc)
    grads = orc.attn_bwd(og, r, Qn, Kn, Vn, dOn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], sc)
    assert_close("O", O.detach()[0].transpose(0, 1), Or, case="dit_qkv_step450")
    for i, (name, ref) in enumerate(zip(("dQ", "dK", "dV"), grads)):
        assert_close(name, qkv.grad[0, :, i].transpose(0, 1), ref, case="dit_qkv_step450")


@pytest.mark.gpu
def test_dit_block_trains_through_the_anneal_start():
    """A few steps of DiTAttentionBlock with AdamW across the first anneal boundary (step 29 dense -> 30 sparse):
    finite loss, gradients reach the projections, and the layer's knobs follow the schedule."""
    from paper_2509_01085_b200.training import AnnealSchedule, DiTAttentionBlock
    grid, Hh, d = (8, 12, 16), 2, 64
    g = Geometry(*grid)
    blk = DiTAttentionBlock(g, 1, Hh, d, schedule=AnnealSchedule())
    x = torch.randn(1, g.L, Hh * d, device="cuda", dtype=torch.bfloat16)
    opt = torch.optim.AdamW(blk.parameters(), lr=1e-3)
    for step in (28, 29, 30, 31):
        blk.set_step(step)
        loss = blk(x).float().pow(2).mean()
        loss.backward()
        assert torch.isfinite(loss)
        assert blk.qkv.weight.grad is not None and torch.isfinite(blk.qkv.weight.grad.float()).all()
        opt.step()
        opt.zero_grad()
        lay = blk.attn._layer()
        r, f, tau = AnnealSchedule().knobs(step)
        assert lay.r == r and lay.tau == tau and lay.k == resolve_k(f, lay.N)
