"""Ulysses sequence parallelism around the BSA layer (SURVEY.md §8(e) mode 2).

For sequences a sequence-parallel DiT keeps sharded by token (the 147,600-token long-video config),
each of P ranks holds a contiguous raster chunk of Ls = L/P tokens of all Hh heads, [B, Ls, Hh, d].
BSA cannot run on a token chunk: Eq.3/Eq.4 rank every pooled KV block of the head.
So, as in Ulysses, one all-to-all per tensor regathers the sequence per head group (rank p owns heads
[p Hp, (p+1) Hp), Hp = Hh/P), BSA runs locally and unchanged on [B, Hp, L, d], and one all-to-all per
output returns to the token-sharded layout:

    B = 1 (the long-video config): token-major chunks, one reorder per direction
    forward : Q, K, V  --SEQ_TO_SEND_T, a2a-->  [L][Hp][d] read in place as a strided [1, Hp, L, d] bsa_tensor
              BSAAttention writes O in that same layout = the send buffer  --a2a, RECV_T_TO_SEQ-->  O [1, Ls, Hh, d]
    backward: dO like Q; dQ, dK, dV like O
    B > 1: head-major chunks, two reorders per direction
    forward : Q, K, V  --SEQ_TO_SEND, a2a, RECV_TO_HEADS-->  BSAAttention.forward  --HEADS_TO_SEND, a2a, RECV_TO_SEQ-->  O
    P = 1: no exchange and no reorder at all: [B, L, Hh, d] is passed as the strided view x.transpose(1, 2).

The reorders are libbsa kernels (bsa_sp_relayout, csrc/sp.cu); the exchange is
torch.distributed.all_to_all_single (NCCL over NVLink/NVSwitch on GPUs; gloo in the CPU tests).
The K and V exchanges are issued asynchronously so V's transfer overlaps the selection on Q and K.
With head_groups = G > 1 (B = 1), each rank's Hp heads are split into G sub-groups that are exchanged, attended
and returned one after another, every exchange issued asynchronously up front: the all-to-all of group g+1 and the
return of group g-1 overlap the attention of group g (bsa_sp_relayout_group builds the per-group chunks).

The ring / context-parallel alternative is rejected: KV selection needs all N pooled
K_c of a head on one rank.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from . import (SP_GROUP_RECV, SP_GROUP_SEND, SP_HEADS_TO_SEND, SP_RECV_T_TO_SEQ, SP_RECV_TO_HEADS, SP_RECV_TO_SEQ,
               SP_SEQ_TO_SEND, SP_SEQ_TO_SEND_T, BSAError, Geometry, bsa_sp_relayout, bsa_sp_relayout_group)


def _cuda_relayout(mode, src, dst, B, Ls, Hh, d, P):
    return bsa_sp_relayout(mode, src, dst, B, Ls, Hh, d, P)


def _cuda_group_relayout(mode, src, dst, Ls, Hh, d, P, hoff, Hs):
    return bsa_sp_relayout_group(mode, src, dst, Ls, Hh, d, P, hoff, Hs)


class UlyssesBSA:
    """BSA over a token-sharded sequence. `attention` is the per-rank layer on Hp heads (default:
    runner.BSAAttention; it must accept strided [B, Hp, L, d] views and an `out` tensor); `relayout` is the
    row-reorder primitive (default: the libbsa kernel)."""

    def __init__(self, geom: Geometry, r: float, f, tau: float, B: int, Hh: int, d: int, group=None, device="cuda",
                 attention=None, relayout: Callable | None = None, dtype=torch.bfloat16, head_groups: int = 1,
                 make_attention: Callable | None = None, group_relayout: Callable | None = None):
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if Hh % self.P:
            raise BSAError(f"Ulysses: {Hh} heads do not split over {self.P} ranks")
        if geom.L % self.P:
            raise BSAError(f"Ulysses: L = {geom.L} tokens do not split over {self.P} ranks")
        self.g, self.B, self.Hh, self.d = geom, B, Hh, d
        self.Hp, self.Ls = Hh // self.P, geom.L // self.P
        self.device = torch.device(device)
        self.dtype = dtype
        grouped = head_groups > 1 and self.P > 1 and B == 1
        if attention is None and not grouped:
            from .runner import BSAAttention
            attention = BSAAttention(geom, r, f, tau, B, self.Hp, d, device=self.device)
        self.layer = attention
        self._relayout = relayout or _cuda_relayout
        # token-major exchange (B == 1) needs no reorder on the BSA side; B > 1 uses head-major chunks
        self.token_major = B == 1
        n = B * self.Ls * Hh * d if (self.P > 1 and not grouped) else 0
        mk = dict(dtype=dtype, device=self.device)
        # per exchanged input (Q, K, V, dO): send and receive buffers, flat [P][chunk]
        self._send = [torch.empty(n, **mk) for _ in range(4)]
        self._recv = [torch.empty(n, **mk) for _ in range(4)]
        # per output (O, dQ, dK, dV): the tensor BSA writes (= the send buffer when token-major) and the receive buffer
        self._out = [torch.empty(n, **mk) for _ in range(4)]
        self._out_recv = [torch.empty(n, **mk) for _ in range(4)]
        nh = B * self.Hp * geom.L * d if (self.P > 1 and not self.token_major) else 0
        self._heads = [torch.empty(nh, **mk) for _ in range(4)]  # B > 1: head-major [B][Hp][L][d] inputs
        # head-group pipelining (token-major only): sub-group s = heads [hoff_s, hoff_s + Hs_s) of every rank
        self.groups = []
        if grouped:
            G = min(head_groups, self.Hp)
            sizes = [self.Hp // G + (1 if s < self.Hp % G else 0) for s in range(G)]
            offs = [sum(sizes[:s]) for s in range(G)]
            if make_attention is None:
                from .runner import BSAAttention
                make_attention = lambda n: BSAAttention(geom, r, f, tau, B, n, d, device=self.device)  # noqa: E731
            self._grelayout = group_relayout or _cuda_group_relayout
            for ho, hs in zip(offs, sizes):
                ng = geom.L * hs * d
                self.groups.append(dict(hoff=ho, Hs=hs, layer=make_attention(hs),
                                        send=[torch.empty(ng, **mk) for _ in range(4)],
                                        recv=[torch.empty(ng, **mk) for _ in range(4)],
                                        out=[torch.empty(ng, **mk) for _ in range(4)],
                                        out_recv=[torch.empty(ng, **mk) for _ in range(4)]))

    # ---------------------------------------------------------------- exchanges
    def _a2a(self, recv, send, async_op=False):
        return dist.all_to_all_single(recv, send, group=self.group, async_op=async_op)

    def _check(self, x, what):
        if tuple(x.shape) != (self.B, self.Ls, self.Hh, self.d):
            raise BSAError(f"Ulysses: {what} must be [B, Ls, Hh, d] = {(self.B, self.Ls, self.Hh, self.d)}, "
                           f"got {tuple(x.shape)}")

    def _heads_view(self, flat):
        """[L][Hp][d] (token-major, B = 1) -> strided [1, Hp, L, d]; [B][Hp][L][d] -> [B, Hp, L, d]."""
        if self.token_major:
            return flat.view(1, self.g.L, self.Hp, self.d).transpose(1, 2)
        return flat.view(self.B, self.Hp, self.g.L, self.d)

    def _send_heads(self, i, x):
        """[B, Ls, Hh, d] (this rank's tokens) -> (async) exchange into slot i; returns the work handle."""
        self._check(x, "input")
        mode = SP_SEQ_TO_SEND_T if self.token_major else SP_SEQ_TO_SEND
        self._relayout(mode, x.contiguous(), self._send[i], self.B, self.Ls, self.Hh, self.d, self.P)
        return self._a2a(self._recv[i], self._send[i], async_op=True)

    def _recv_heads(self, i, work):
        if work is not None:
            work.wait()
        if self.token_major:
            return self._heads_view(self._recv[i])
        self._relayout(SP_RECV_TO_HEADS, self._recv[i], self._heads[i], self.B, self.Ls, self.Hh, self.d, self.P)
        return self._heads_view(self._heads[i])

    def _out_view(self, i):
        """Where BSA writes output i: token-major, it is the send buffer of the return exchange itself."""
        return self._heads_view(self._out[i]) if self.token_major else \
            self._out[i].new_empty(self.B, self.Hp, self.g.L, self.d)

    def _to_seq(self, i, x):
        """BSA output i (the _out_view tensor x) -> [B, Ls, Hh, d] (this rank's tokens, all heads)."""
        out = torch.empty(self.B, self.Ls, self.Hh, self.d, dtype=x.dtype, device=x.device)
        if self.token_major:
            send, mode = self._out[i], SP_RECV_T_TO_SEQ
        else:
            self._relayout(SP_HEADS_TO_SEND, x.contiguous(), self._out[i], self.B, self.Ls, self.Hh, self.d, self.P)
            send, mode = self._out[i], SP_RECV_TO_SEQ
        self._a2a(self._out_recv[i], send)
        self._relayout(mode, self._out_recv[i], out, self.B, self.Ls, self.Hh, self.d, self.P)
        return out

    # ---------------------------------------------------------------- head-group pipeline (B = 1)
    def _gview(self, flat, hs):
        return flat.view(1, self.g.L, hs, self.d).transpose(1, 2)  # [L][hs][d] as a strided [1, hs, L, d]

    def _gsend(self, gr, i, x):
        self._grelayout(SP_GROUP_SEND, x.contiguous(), gr["send"][i], self.Ls, self.Hh, self.d, self.P, gr["hoff"],
                        gr["Hs"])
        return self._a2a(gr["recv"][i], gr["send"][i], async_op=True)

    def _gcollect(self, gr, i, work, out):
        work.wait()
        self._grelayout(SP_GROUP_RECV, gr["out_recv"][i], out, self.Ls, self.Hh, self.d, self.P, gr["hoff"], gr["Hs"])

    def _forward_groups(self, q, k, v):
        for x, w in ((q, "q"), (k, "k"), (v, "v")):
            self._check(x, w)
        works = [[self._gsend(gr, i, x) for i, x in enumerate((q, k, v))] for gr in self.groups]  # all in flight
        O = torch.empty(self.B, self.Ls, self.Hh, self.d, dtype=q.dtype, device=q.device)
        back = []
        for gr, (wq, wk, wv) in zip(self.groups, works):
            hs, lay = gr["Hs"], gr["layer"]
            wq.wait()
            wk.wait()
            Qh, Kh = self._gview(gr["recv"][0], hs), self._gview(gr["recv"][1], hs)
            lay.select(Qh, Kh)           # while V of this group and the next groups are in flight
            wv.wait()
            Vh = self._gview(gr["recv"][2], hs)
            lay._saved = (Qh, Kh, Vh)
            lay.attend(Qh, Kh, Vh, out=self._gview(gr["out"][0], hs))
            back.append(self._a2a(gr["out_recv"][0], gr["out"][0], async_op=True))  # returns during the next group
        for gr, w in zip(self.groups, back):
            self._gcollect(gr, 0, w, O)
        return O

    def _backward_groups(self, dO):
        works = [self._gsend(gr, 3, dO) for gr in self.groups]
        outs = [torch.empty(self.B, self.Ls, self.Hh, self.d, dtype=dO.dtype, device=dO.device) for _ in range(3)]
        back = []
        for gr, w in zip(self.groups, works):
            hs = gr["Hs"]
            w.wait()
            dOh = self._gview(gr["recv"][3], hs)
            gr["layer"].backward(dOh, out=tuple(self._gview(gr["out"][i], hs) for i in (1, 2, 3)))
            back.append([self._a2a(gr["out_recv"][i], gr["out"][i], async_op=True) for i in (1, 2, 3)])
        for gr, ws in zip(self.groups, back):
            for i, w in zip((1, 2, 3), ws):
                self._gcollect(gr, i, w, outs[i - 1])
        return tuple(outs)

    # ---------------------------------------------------------------- layer
    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        """q, k, v: [B, Ls, Hh, d] token shards -> O [B, Ls, Hh, d]."""
        if self.groups:
            return self._forward_groups(q, k, v)
        if self.P == 1:  # the model layout is a strided [B, Hh, L, d] view: nothing to move
            for x, w in ((q, "q"), (k, "k"), (v, "v")):
                self._check(x, w)
            O = torch.empty(self.B, self.Ls, self.Hh, self.d, dtype=q.dtype, device=q.device)
            Qh, Kh, Vh = (x.transpose(1, 2) for x in (q, k, v))
            self.layer.select(Qh, Kh)
            self.layer._saved = (Qh, Kh, Vh)
            self.layer.attend(Qh, Kh, Vh, out=O.transpose(1, 2))
            return O
        wq = self._send_heads(0, q)
        wk = self._send_heads(1, k)
        wv = self._send_heads(2, v)
        Qh = self._recv_heads(0, wq)
        Kh = self._recv_heads(1, wk)
        self.layer.select(Qh, Kh)            # a1-a6 run while V is in flight
        Vh = self._recv_heads(2, wv)
        self.layer._saved = (Qh, Kh, Vh)
        O = self.layer.attend(Qh, Kh, Vh, out=self._out_view(0))    # a7 + fill
        return self._to_seq(0, O)

    def backward(self, dO: torch.Tensor):
        """dO: [B, Ls, Hh, d] -> (dQ, dK, dV), each [B, Ls, Hh, d]."""
        self._check(dO, "dO")
        if self.groups:
            return self._backward_groups(dO)
        if self.P == 1:
            outs = [torch.empty(self.B, self.Ls, self.Hh, self.d, dtype=dO.dtype, device=dO.device) for _ in range(3)]
            self.layer.backward(dO.transpose(1, 2), out=tuple(x.transpose(1, 2) for x in outs))
            return tuple(outs)
        dOh = self._recv_heads(3, self._send_heads(3, dO))
        grads = [self._out_view(i) for i in (1, 2, 3)]
        grads = self.layer.backward(dOh, out=tuple(grads))
        return tuple(self._to_seq(i, x) for i, x in zip((1, 2, 3), grads))
