"""Ulysses sequence parallelism around the BSA layer (SURVEY.md §8(e) mode 2).

For sequences a sequence-parallel DiT keeps sharded by token (the 147,600-token long-video config),
each of P ranks holds a contiguous raster chunk of Ls = L/P tokens of all Hh heads, [B, Ls, Hh, d].
BSA cannot run on a token chunk: Eq.3/Eq.4 rank every pooled KV block of the head.
So, as in Ulysses, one all-to-all per tensor regathers the sequence per head group (rank p owns heads
[p Hp, (p+1) Hp), Hp = Hh/P), BSA runs locally and unchanged on [B, Hp, L, d], and one all-to-all per
output returns to the token-sharded layout:

    forward : Q, K, V  --SEQ_TO_SEND, a2a, RECV_TO_HEADS-->  BSAAttention.forward  --HEADS_TO_SEND, a2a, RECV_TO_SEQ-->  O
    backward: dO       --(same as Q)-->                      BSAAttention.backward --(same as O)-->  dQ, dK, dV

The reorders are libbsa kernels (bsa_sp_relayout, csrc/sp.cu); the exchange is
torch.distributed.all_to_all_single (NCCL over NVLink/NVSwitch on GPUs; gloo in the CPU tests).
The K and V exchanges are issued asynchronously so V's transfer overlaps the selection on Q and K.

The ring / context-parallel alternative is rejected: KV selection needs all N pooled
K_c of a head on one rank.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from . import SP_HEADS_TO_SEND, SP_RECV_TO_HEADS, SP_RECV_TO_SEQ, SP_SEQ_TO_SEND, BSAError, Geometry, bsa_sp_relayout


def _cuda_relayout(mode, src, dst, B, Ls, Hh, d, P):
    return bsa_sp_relayout(mode, src, dst, B, Ls, Hh, d, P)


class UlyssesBSA:
    """BSA over a token-sharded sequence. `attention` is the per-rank layer on Hp heads (default:
    runner.BSAAttention); `relayout` is the row-reorder primitive (default: the libbsa kernel)."""

    def __init__(self, geom: Geometry, r: float, f, tau: float, B: int, Hh: int, d: int, group=None, device="cuda",
                 attention=None, relayout: Callable | None = None, dtype=torch.bfloat16):
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
        if attention is None:
            from .runner import BSAAttention
            attention = BSAAttention(geom, r, f, tau, B, self.Hp, d, device=self.device)
        self.layer = attention
        self._relayout = relayout or _cuda_relayout
        n = B * self.Ls * Hh * d
        mk = dict(dtype=dtype, device=self.device)
        # per exchanged tensor: send / receive buffers (flat [P][B][Hp][Ls][d]) and the head-layout result
        # (P = 1: the head layout is reached by one reorder, no exchange buffers)
        nx = n if self.P > 1 else 0
        self._send = [torch.empty(nx, **mk) for _ in range(3)]
        self._recv = [torch.empty(nx, **mk) for _ in range(3)]
        self._heads = [torch.empty(B, self.Hp, geom.L, d, **mk) for _ in range(3)]
        # dO gets its own buffers: Q^h, K^h, V^h stay saved for the backward
        self._dO_bufs = (torch.empty(nx, **mk), torch.empty(nx, **mk), torch.empty(B, self.Hp, geom.L, d, **mk))

    # ---------------------------------------------------------------- exchanges
    def _a2a(self, recv, send, async_op=False):
        if self.P == 1:
            recv.copy_(send)
            return None
        return dist.all_to_all_single(recv, send, group=self.group, async_op=async_op)

    def _send_heads(self, i, x):
        """[B, Ls, Hh, d] (this rank's tokens) -> async exchange into slot i; returns the work handle."""
        if x.shape != (self.B, self.Ls, self.Hh, self.d):
            raise BSAError(f"Ulysses: expected [B, Ls, Hh, d] = {(self.B, self.Ls, self.Hh, self.d)}, got {tuple(x.shape)}")
        if self.P == 1:  # [1][B][Hh][L][d] is already the head layout: no exchange, no second reorder
            self._relayout(SP_SEQ_TO_SEND, x.contiguous(), self._heads[i], self.B, self.Ls, self.Hh, self.d, 1)
            return None
        self._relayout(SP_SEQ_TO_SEND, x.contiguous(), self._send[i], self.B, self.Ls, self.Hh, self.d, self.P)
        return self._a2a(self._recv[i], self._send[i], async_op=True)

    def _recv_heads(self, i, work):
        if self.P == 1:
            return self._heads[i]
        if work is not None:
            work.wait()
        self._relayout(SP_RECV_TO_HEADS, self._recv[i], self._heads[i], self.B, self.Ls, self.Hh, self.d, self.P)
        return self._heads[i]

    def _to_seq(self, x, i=0):
        """[B, Hp, L, d] (this rank's heads) -> [B, Ls, Hh, d] (this rank's tokens, all heads)."""
        out = torch.empty(self.B, self.Ls, self.Hh, self.d, dtype=x.dtype, device=x.device)
        if self.P == 1:  # x is [1][B][Hh][L][d]: one reorder back to the model layout
            self._relayout(SP_RECV_TO_SEQ, x.contiguous(), out, self.B, self.Ls, self.Hh, self.d, 1)
            return out
        self._relayout(SP_HEADS_TO_SEND, x.contiguous(), self._send[i], self.B, self.Ls, self.Hh, self.d, self.P)
        self._a2a(self._recv[i], self._send[i])
        self._relayout(SP_RECV_TO_SEQ, self._recv[i], out, self.B, self.Ls, self.Hh, self.d, self.P)
        return out

    # ---------------------------------------------------------------- layer
    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        """q, k, v: [B, Ls, Hh, d] token shards -> O [B, Ls, Hh, d]."""
        wq = self._send_heads(0, q)
        wk = self._send_heads(1, k)
        wv = self._send_heads(2, v)
        Qh = self._recv_heads(0, wq)
        Kh = self._recv_heads(1, wk)
        self.layer.select(Qh, Kh)            # a1-a6 run while V is in flight
        Vh = self._recv_heads(2, wv)
        self.layer._saved = (Qh, Kh, Vh)
        O = self.layer.attend(Qh, Kh, Vh)    # a7 + fill
        return self._to_seq(O)

    def backward(self, dO: torch.Tensor):
        """dO: [B, Ls, Hh, d] -> (dQ, dK, dV), each [B, Ls, Hh, d]."""
        s, r, h = self._dO_bufs
        if dO.shape != (self.B, self.Ls, self.Hh, self.d):
            raise BSAError("Ulysses: dO must be [B, Ls, Hh, d]")
        if self.P == 1:
            self._relayout(SP_SEQ_TO_SEND, dO.contiguous(), h, self.B, self.Ls, self.Hh, self.d, 1)
        else:
            self._relayout(SP_SEQ_TO_SEND, dO.contiguous(), s, self.B, self.Ls, self.Hh, self.d, self.P)
            self._a2a(r, s)
            self._relayout(SP_RECV_TO_HEADS, r, h, self.B, self.Ls, self.Hh, self.d, self.P)
        dQ, dK, dV = self.layer.backward(h)
        # the send/recv slots of Q, K, V are free again (their head layouts live in self._heads)
        return self._to_seq(dQ, 0), self._to_seq(dK, 1), self._to_seq(dV, 2)
