"""Ulysses sequence parallelism (SURVEY.md §8(e) mode 2; paper_2509_01085_b200/ulysses.py).

CPU (`not gpu`): the four row reorders, written here as plain torch permutes, compose with an emulated
all-to-all into "rank p holds heads [p Hp, (p+1) Hp) of the whole sequence" and back; and two gloo
ranks running UlyssesBSA around the fp64 oracle give exactly the single-process oracle result.
GPU: libbsa's bsa_sp_relayout equals the torch permutes bit for bit, and P emulated ranks of
(relayout kernels + exchange + BSAAttention on Hp heads) reproduce one BSAAttention over all heads.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bsa_gen
import oracle as orc
from paper_2509_01085_b200 import (SP_GROUP_RECV, SP_GROUP_SEND, SP_HEADS_TO_SEND, SP_RECV_T_TO_SEQ,
                                   SP_RECV_TO_HEADS, SP_RECV_TO_SEQ, SP_SEQ_TO_SEND, SP_SEQ_TO_SEND_T, Geometry,
                                   resolve_k)


def ref_relayout(mode, src, dst, B, Ls, Hh, d, P):
    """Independent statement of include/bsa.h's bsa_sp_relayout index maps."""
    Hp = Hh // P
    if mode == SP_SEQ_TO_SEND:      # [B][Ls][Hh][d] -> [P][B][Hp][Ls][d]
        out = src.reshape(B, Ls, P, Hp, d).permute(2, 0, 3, 1, 4)
    elif mode == SP_RECV_TO_HEADS:  # [P(seq chunk)][B][Hp][Ls][d] -> [B][Hp][P Ls][d]
        out = src.reshape(P, B, Hp, Ls, d).permute(1, 2, 0, 3, 4)
    elif mode == SP_HEADS_TO_SEND:  # [B][Hp][P Ls][d] -> [P][B][Hp][Ls][d]
        out = src.reshape(B, Hp, P, Ls, d).permute(2, 0, 1, 3, 4)
    elif mode == SP_RECV_TO_SEQ:    # [P(head group)][B][Hp][Ls][d] -> [B][Ls][Hh][d]
        out = src.reshape(P, B, Hp, Ls, d).permute(1, 3, 0, 2, 4)
    elif mode == SP_SEQ_TO_SEND_T:  # [B][Ls][Hh][d] -> [P][B][Ls][Hp][d]
        out = src.reshape(B, Ls, P, Hp, d).permute(2, 0, 1, 3, 4)
    else:                           # SP_RECV_T_TO_SEQ: [P(head group)][B][Ls][Hp][d] -> [B][Ls][Hh][d]
        out = src.reshape(P, B, Ls, Hp, d).permute(1, 2, 0, 3, 4)
    dst.view(-1).copy_(out.reshape(-1))
    return dst


def emulate(relayout, x_seq_shards, B, Ls, Hh, d, P, forward=True):
    """Run the reorders of P ranks with the all-to-all done by hand (chunk q of rank s -> rank q)."""
    m_send, m_recv = (SP_SEQ_TO_SEND, SP_RECV_TO_HEADS) if forward else (SP_HEADS_TO_SEND, SP_RECV_TO_SEQ)
    sends = []
    for x in x_seq_shards:
        s = torch.empty(x.numel(), dtype=x.dtype, device=x.device)
        relayout(m_send, x.contiguous(), s, B, Ls, Hh, d, P)
        sends.append(s.view(P, -1))
    outs = []
    for p in range(P):
        recv = torch.cat([sends[s][p] for s in range(P)])
        shape = (B, Hh // P, P * Ls, d) if forward else (B, Ls, Hh, d)
        o = torch.empty(shape, dtype=recv.dtype, device=recv.device)
        relayout(m_recv, recv, o, B, Ls, Hh, d, P)
        outs.append(o)
    return outs


@pytest.mark.parametrize("P,B,Hh", [(1, 1, 3), (2, 1, 4), (4, 2, 8), (2, 2, 6)])
def test_relayout_roundtrip_cpu(P, B, Hh):
    """Head-major chunks (SEQ_TO_SEND / RECV_TO_HEADS / HEADS_TO_SEND / RECV_TO_SEQ) round-trip."""
    L, d = 24, 16
    Ls = L // P
    x = torch.randn(B, L, Hh, d, dtype=torch.float64)
    shards = [x[:, s * Ls:(s + 1) * Ls] for s in range(P)]
    heads = emulate(ref_relayout, shards, B, Ls, Hh, d, P, forward=True)
    Hp = Hh // P
    for p in range(P):
        assert torch.equal(heads[p], x.permute(0, 2, 1, 3)[:, p * Hp:(p + 1) * Hp])
    back = emulate(ref_relayout, heads, B, Ls, Hh, d, P, forward=False)
    for s in range(P):
        assert torch.equal(back[s], shards[s])


@pytest.mark.parametrize("P,Hh", [(1, 3), (2, 4), (4, 8), (3, 6)])
def test_token_major_exchange_cpu(P, Hh):
    """B = 1 token-major path: after SEQ_TO_SEND_T and the all-to-all, rank p's receive buffer read as the strided
    [1, Hp, L, d] view IS heads [p Hp, (p+1) Hp) of the whole sequence (no reorder); written back in that layout and
    exchanged again, RECV_T_TO_SEQ restores each rank's [1, Ls, Hh, d] shard."""
    B, L, d = 1, 24, 16
    Ls, Hp = L // P, Hh // P
    x = torch.randn(B, L, Hh, d, dtype=torch.float64)
    shards = [x[:, s * Ls:(s + 1) * Ls] for s in range(P)]
    sends = []
    for sh in shards:
        buf = torch.empty(sh.numel(), dtype=sh.dtype)
        ref_relayout(SP_SEQ_TO_SEND_T, sh.contiguous(), buf, B, Ls, Hh, d, P)
        sends.append(buf.view(P, -1))
    recvs = [torch.cat([sends[s][p] for s in range(P)]) for p in range(P)]
    for p in range(P):
        view = recvs[p].view(1, L, Hp, d).transpose(1, 2)  # what BSA reads, strides (L Hp d, d, Hp d)
        assert view.stride()[1:] == (d, Hp * d, 1)
        assert torch.equal(view, x.permute(0, 2, 1, 3)[:, p * Hp:(p + 1) * Hp])
    # return path: the outputs, written in the received layout, are the send buffers
    back_recv = [torch.cat([recvs[s].view(P, -1)[p] for s in range(P)]) for p in range(P)]
    for s in range(P):
        out = torch.empty(B, Ls, Hh, d, dtype=x.dtype)
        ref_relayout(SP_RECV_T_TO_SEQ, back_recv[s], out, B, Ls, Hh, d, P)
        assert torch.equal(out, shards[s])


class OracleLayer:
    """The per-rank attention slot of UlyssesBSA filled with the fp64 oracle (test infrastructure)."""

    def __init__(self, og, r, k, tau, d):
        self.og, self.r, self.k, self.tau, self.scale = og, r, k, tau, 1.0 / math.sqrt(d)

    def select(self, Qh, Kh):
        Q, K = Qh[0].numpy(), Kh[0].numpy()
        self.qs = orc.select_queries(self.og, self.r, Q)
        self.kv = orc.select_kv(self.og, Q, K, self.k, self.tau)

    def attend(self, Qh, Kh, Vh, out=None):
        O, _ = orc.attn_fwd(self.og, self.r, Qh[0].numpy(), Kh[0].numpy(), Vh[0].numpy(), self.qs["kept_tok"],
                            self.qs["donor"], self.kv["q2k_num"], self.kv["q2k_idx"], self.scale)
        O = torch.from_numpy(np.ascontiguousarray(O))[None]
        return O if out is None else out.copy_(O)

    def backward(self, dOh, out=None):
        Q, K, V = (t[0].numpy() for t in self._saved)
        g = orc.attn_bwd(self.og, self.r, Q, K, V, dOh[0].numpy(), self.qs["kept_tok"], self.qs["donor"],
                         self.kv["q2k_num"], self.kv["q2k_idx"], self.scale)
        g = tuple(torch.from_numpy(np.ascontiguousarray(x))[None] for x in g)
        return g if out is None else tuple(o.copy_(x) for o, x in zip(out, g))


GRID, BLOCK, HH, D, R, F, TAU = (4, 8, 8), (2, 4, 4), 4, 64, 0.5, 0.5, 0.9


def _inputs():
    Q, K, V = bsa_gen.make_inputs("video", 3, 1, HH, GRID, D)
    dO = bsa_gen.grad_output(3, (1, HH, Q.shape[2], D))
    return [x.double() for x in (Q, K, V, dO)]  # [B, Hh, L, d], exact bf16 values


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def ref_relayout_group(mode, src, dst, Ls, Hh, d, P, hoff, Hs):
    """Independent statement of include/bsa.h's bsa_sp_relayout_group (token-major head sub-group)."""
    Hp = Hh // P
    if mode == SP_GROUP_SEND:  # [Ls][Hh][d] heads p Hp + hoff + h -> [P][Ls][Hs][d]
        dst.view(-1).copy_(src.reshape(Ls, P, Hp, d)[:, :, hoff:hoff + Hs].permute(1, 0, 2, 3).reshape(-1))
    else:                      # [P][Ls][Hs][d] -> those heads of [Ls][Hh][d]
        dst.view(Ls, P, Hp, d)[:, :, hoff:hoff + Hs] = src.reshape(P, Ls, Hs, d).permute(1, 0, 2, 3)
    return dst


def _worker(rank, world, port, out, head_groups=1):
    from paper_2509_01085_b200.ulysses import UlyssesBSA
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        og = orc.Geom(*GRID, *BLOCK)
        N = orc.sizes(og, R)[0]
        layer = OracleLayer(og, R, resolve_k(F, N), TAU, D)
        make = lambda n: OracleLayer(og, R, resolve_k(F, N), TAU, D)  # noqa: E731
        u = UlyssesBSA(Geometry(*GRID, *BLOCK), R, F, TAU, 1, HH, D, device="cpu",
                       attention=None if head_groups > 1 else layer, relayout=ref_relayout, dtype=torch.float64,
                       head_groups=head_groups, make_attention=make, group_relayout=ref_relayout_group)
        assert (len(u.groups) == min(head_groups, HH // world)) if head_groups > 1 else not u.groups
        Q, K, V, dO = _inputs()
        L = Q.shape[2]
        Ls = L // world
        shard = lambda x: x.permute(0, 2, 1, 3)[:, rank * Ls:(rank + 1) * Ls].contiguous()  # [B, Ls, Hh, d]
        O = u.forward(shard(Q), shard(K), shard(V))
        dQ, dK, dV = u.backward(shard(dO))
        out[rank] = (O.numpy(), dQ.numpy(), dK.numpy(), dV.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("head_groups", [1, 2])
def test_ulysses_gloo_two_ranks_equals_single_process_oracle(head_groups):
    """Two gloo ranks, plain (one exchange per tensor) and head-group pipelined (two sub-groups of one head per
    rank, exchanged, attended and returned one after another), against the single-process oracle."""
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out, head_groups), nprocs=world, join=True)
        res = dict(out)
    Q, K, V, dO = _inputs()
    og = orc.Geom(*GRID, *BLOCK)
    N = orc.sizes(og, R)[0]
    k = resolve_k(F, N)
    Qn, Kn, Vn, dOn = (x[0].numpy() for x in (Q, K, V, dO))
    qs = orc.select_queries(og, R, Qn)
    kv = orc.select_kv(og, Qn, Kn, k, TAU)
    sc = 1.0 / math.sqrt(D)
    O, _ = orc.attn_fwd(og, R, Qn, Kn, Vn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], sc)
    grads = orc.attn_bwd(og, R, Qn, Kn, Vn, dOn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], sc)
    full = [O, *grads]  # each [Hh, L, d]
    for i, ref in enumerate(full):
        got = np.concatenate([res[r][i][0] for r in range(world)], axis=0)  # [L, Hh, d]
        assert np.array_equal(got, np.transpose(ref, (1, 0, 2))), i


@pytest.mark.gpu
@pytest.mark.parametrize("B,Ls,Hh,d,P", [(1, 96, 4, 128, 2), (2, 50, 8, 64, 4), (1, 33, 6, 128, 3), (1, 64, 5, 128, 1)])
def test_sp_relayout_kernels_match_permutes(B, Ls, Hh, d, P):
    import paper_2509_01085_b200 as bsa
    shapes = {SP_SEQ_TO_SEND: (B, Ls, Hh, d), SP_RECV_TO_HEADS: (P, B, Hh // P, Ls, d),
              SP_HEADS_TO_SEND: (B, Hh // P, P * Ls, d), SP_RECV_TO_SEQ: (P, B, Hh // P, Ls, d),
              SP_SEQ_TO_SEND_T: (B, Ls, Hh, d), SP_RECV_T_TO_SEQ: (P, B, Ls, Hh // P, d)}
    g = torch.Generator().manual_seed(5)
    for mode, shp in shapes.items():
        src = torch.randn(*shp, generator=g).to(torch.bfloat16).cuda()
        got = torch.full((src.numel(),), float("nan"), dtype=torch.bfloat16, device="cuda")
        bsa.bsa_sp_relayout(mode, src, got, B, Ls, Hh, d, P)
        want = torch.empty_like(got)
        ref_relayout(mode, src, want, B, Ls, Hh, d, P)
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int16), want.view(torch.int16)), mode


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4])
def test_ulysses_emulated_ranks_match_single_layer(P):
    """P ranks emulated on one GPU: libbsa reorders + hand exchange + BSAAttention on Hp heads."""
    import paper_2509_01085_b200 as bsa
    from paper_2509_01085_b200.runner import BSAAttention
    grid, Hh, d = (8, 12, 16), 8, 128
    g = Geometry(*grid)
    B, L = 1, g.L
    Ls, Hp = L // P, Hh // P
    Q, K, V = bsa_gen.make_inputs("video", 1, B, Hh, grid, d, device="cuda")
    dO = bsa_gen.grad_output(1, (B, Hh, L, d)).cuda()
    full = BSAAttention(g, 0.5, 0.2, 0.9, B, Hh, d)
    full.forward(Q, K, V)
    relay = lambda *a: bsa.bsa_sp_relayout(*a)
    to_shards = lambda x: [x.permute(0, 2, 1, 3)[:, s * Ls:(s + 1) * Ls].contiguous() for s in range(P)]
    Qh, Kh, Vh, dOh = (emulate(relay, to_shards(x), B, Ls, Hh, d, P, True) for x in (Q, K, V, dO))
    outs = []
    for p in range(P):
        lay = BSAAttention(g, 0.5, 0.2, 0.9, B, Hp, d)
        o = lay.forward(Qh[p], Kh[p], Vh[p]).clone()
        assert torch.equal(lay.q2k_num, full.q2k_num[:, p * Hp:(p + 1) * Hp])
        outs.append((o, *(x.clone() for x in lay.backward(dOh[p]))))
    # The assembled Ulysses result must meet the same oracle tolerance as the single layer (the two GPU runs
    # differ only in summation order -- rotations depend on the head's index in the batch -- so they are
    # compared through the oracle rather than bit for bit).
    import math
    from parity_util import assert_close
    og = orc.Geom(*grid, 4, 4, 4)
    k = resolve_k(0.2, orc.sizes(og, 0.5)[0])
    Qn, Kn, Vn, dOn = (x[0].float().cpu().double().numpy() for x in (Q, K, V, dO))
    qs = orc.select_queries(og, 0.5, Qn)
    kv = orc.select_kv(og, Qn, Kn, k, 0.9)
    sc = 1.0 / math.sqrt(d)
    Or, _ = orc.attn_fwd(og, 0.5, Qn, Kn, Vn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], sc)
    grads = orc.attn_bwd(og, 0.5, Qn, Kn, Vn, dOn, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], sc)
    assert np.array_equal(full.q2k_num[0].cpu().numpy(), kv["q2k_num"])
    for i, (name, ref) in enumerate(zip(("O", "dQ", "dK", "dV"), (Or, *grads))):
        seq = emulate(relay, [outs[p][i] for p in range(P)], B, Ls, Hh, d, P, False)
        got = torch.cat(seq, dim=1).permute(0, 2, 1, 3)  # [B, Hh, L, d]
        torch.cuda.synchronize()
        assert_close(name, got[0], ref)


@pytest.mark.gpu
@pytest.mark.parametrize("Ls,Hh,d,P,hoff,Hs", [(96, 8, 128, 2, 0, 2), (96, 8, 128, 2, 2, 2), (33, 15, 64, 3, 1, 3),
                                               (40, 40, 128, 8, 3, 2)])
def test_sp_relayout_group_kernels_match_reference(Ls, Hh, d, P, hoff, Hs):
    import paper_2509_01085_b200 as bsa
    g = torch.Generator().manual_seed(7)
    x = torch.randn(Ls, Hh, d, generator=g).to(torch.bfloat16).cuda()
    got = torch.full((P * Ls * Hs * d,), float("nan"), dtype=torch.bfloat16, device="cuda")
    bsa.bsa_sp_relayout_group(SP_GROUP_SEND, x, got, Ls, Hh, d, P, hoff, Hs)
    want = torch.empty_like(got)
    ref_relayout_group(SP_GROUP_SEND, x, want, Ls, Hh, d, P, hoff, Hs)
    assert torch.equal(got.view(torch.int16), want.view(torch.int16))
    back = torch.zeros(Ls * Hh * d, dtype=torch.bfloat16, device="cuda")
    bsa.bsa_sp_relayout_group(SP_GROUP_RECV, got, back, Ls, Hh, d, P, hoff, Hs)
    ref = torch.zeros_like(back)
    ref_relayout_group(SP_GROUP_RECV, want, ref, Ls, Hh, d, P, hoff, Hs)
    torch.cuda.synchronize()
    assert torch.equal(back.view(torch.int16), ref.view(torch.int16))
