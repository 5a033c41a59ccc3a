"""Training integration of the BSA layer: an autograd function over the C-ABI
forward/backward and the paper's annealed sparsity schedule (§4 Implementation Details).

    sched = AnnealSchedule()
    attn = BSASelfAttention(Geometry(21, 30, 52, 4, 4, 4, 2, 2, 2), B=1, Hh=12, d=128, schedule=sched)
    for step in range(steps):
        attn.set_step(step)                 # (r, k, tau) of this step
        O = attn(Q, K, V)                   # [B, Hh, L, d] bf16, differentiable w.r.t. Q, K, V
        loss(O).backward()

Selection (Eq.2-Eq.4) is piecewise constant in Q and K and is held fixed in the backward (reading C10);
the gradients are those of bsa_attn_bwd. Every step runs in libbsa's kernels; this module only keeps a
BSAAttention per query keep ratio r (the only knob that changes buffer sizes; k and tau are set per call) and
allocates the tensors autograd hands out.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import BSAError, Geometry, bsa_sizes, resolve_k


@dataclass(frozen=True)
class AnnealSchedule:
    """"training begins with full attention, and every 30 steps, the sparsity is increased by 0.03
    until reaching a maximum of 0.9. In KV-sparse, the number of top-k tokens selected is gradually reduced
    from the total number of blocks to 0.1x the total".

    Readings (C27): the combined sparsity s(step) = min(cap, increment * floor(step / interval));
    the query side takes it first, r = max(r_final, 1 - s) (the paper's r = 0.5 is reached at s = 0.5, SPEC
    knobs_for_sparsity); Eq.3's key fraction f = k / N falls linearly from kv_start to kv_end over the same
    horizon the sparsity anneal needs to reach its cap (cap / increment * interval = 900 steps), then stays.
    tau (Eq.4's cumulative target) is fixed."""
    interval: int = 30
    increment: float = 0.03
    cap: float = 0.9
    r_final: float = 0.5
    kv_start: float = 1.0
    kv_end: float = 0.1
    tau: float = 0.9

    @property
    def horizon(self) -> int:
        return int(round(self.cap / self.increment)) * self.interval

    def sparsity_at_step(self, step: int) -> float:
        if step < 0:
            raise ValueError("step must be >= 0")
        return min(self.cap, self.increment * (step // self.interval))

    def kv_fraction_at_step(self, step: int) -> float:
        if step < 0:
            raise ValueError("step must be >= 0")
        t = min(1.0, step / self.horizon)
        return max(self.kv_end, self.kv_start + (self.kv_end - self.kv_start) * t)

    def knobs(self, step: int) -> tuple[float, float, float]:
        """(r, f, tau) for this step; step 0 is full attention (r = 1, f = 1, tau = 1)."""
        s = self.sparsity_at_step(step)
        if s == 0.0:
            return 1.0, 1.0, 1.0
        r = max(self.r_final, 1.0 - s)
        return r, self.kv_fraction_at_step(step), self.tau


class _BSAFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, Q, K, V, layer):
        B, Hh, L, d = Q.shape
        O = torch.empty(B, Hh, L, d, dtype=Q.dtype, device=Q.device)
        layer.forward(Q, K, V, out=O)
        layer._fwd_count = getattr(layer, "_fwd_count", 0) + 1
        ctx.layer, ctx.count = layer, layer._fwd_count
        # saved through autograd: an in-place edit of Q, K, V or O before backward raises a version error
        ctx.save_for_backward(Q, K, V, O)
        return O

    @staticmethod
    def backward(ctx, dO):
        layer = ctx.layer
        if layer._fwd_count != ctx.count:
            raise BSAError("BSA backward after another forward through the same layer: the layer holds the "
                           "selection and statistics of its last forward only (use one layer per call site)")
        Q, K, V, O = ctx.saved_tensors
        if dO.stride(-1) != 1:
            dO = dO.contiguous()
        B, Hh, L, d = Q.shape
        grads = tuple(torch.empty(B, Hh, L, d, dtype=Q.dtype, device=Q.device) for _ in range(3))
        layer.backward(dO, out=grads, saved=(Q, K, V, O))
        return (*grads, None)


def bsa_attention(Q, K, V, layer):
    """Differentiable BSA attention through `layer` (a runner.BSAAttention sized for Q's shape)."""
    return _BSAFunction.apply(Q, K, V, layer)


class _BSAQKVFunction(torch.autograd.Function):
    """BSA attention on a fused projection: qkv [B, L, 3, Hh, d] -> O [B, L, Hh, d]. Q, K and V go into the library
    as strided views of qkv and O is written in the model layout, so the forward moves no activation; the
    backward writes dQ, dK, dV straight into the three slices of one d(qkv) tensor (include/bsa.h bsa_tensor)."""

    @staticmethod
    def forward(ctx, qkv, layer):
        B, L, _, Hh, d = qkv.shape
        Q, K, V = (qkv[:, :, i].transpose(1, 2) for i in range(3))
        O = torch.empty(B, L, Hh, d, dtype=qkv.dtype, device=qkv.device)
        layer.forward(Q, K, V, out=O.transpose(1, 2))
        layer._fwd_count = getattr(layer, "_fwd_count", 0) + 1
        ctx.layer, ctx.count = layer, layer._fwd_count
        ctx.save_for_backward(qkv, O)
        return O

    @staticmethod
    def backward(ctx, dO):
        layer = ctx.layer
        if layer._fwd_count != ctx.count:
            raise BSAError("BSA backward after another forward through the same layer (use one layer per call site)")
        qkv, O = ctx.saved_tensors
        if dO.stride(-1) != 1:
            dO = dO.contiguous()
        dqkv = torch.empty_like(qkv)
        Q, K, V = (qkv[:, :, i].transpose(1, 2) for i in range(3))
        grads = tuple(dqkv[:, :, i].transpose(1, 2) for i in range(3))
        layer.backward(dO.transpose(1, 2), out=grads, saved=(Q, K, V, O.transpose(1, 2)))
        return dqkv, None


def bsa_attention_qkv(qkv, layer):
    """Differentiable BSA attention of a fused [B, L, 3, Hh, d] projection -> [B, L, Hh, d] (no layout copies)."""
    return _BSAQKVFunction.apply(qkv, layer)


class BSASelfAttention(torch.nn.Module):
    """The attention op of a DiT block with BSA's sparsity: Q, K, V [B, Hh, L, d] bf16 -> O."""

    def __init__(self, geom: Geometry, B: int, Hh: int, d: int, schedule: AnnealSchedule | None = None,
                 r: float = 0.5, f: float = 0.1, tau: float = 0.9, device="cuda"):
        super().__init__()
        self.geom, self.B, self.Hh, self.d, self.device = geom, B, Hh, d, torch.device(device)
        self.schedule = schedule
        self.r, self.f, self.tau = r, f, tau
        self._layers: dict = {}

    def set_step(self, step: int):
        if self.schedule is None:
            raise BSAError("no schedule attached")
        self.r, self.f, self.tau = self.schedule.knobs(step)

    def _layer(self):
        from .runner import BSAAttention
        N = bsa_sizes(self.geom, self.r)[0]
        lay = self._layers.get(self.r)
        if lay is None:
            # buffers depend on r only (k and tau are per-call knobs); the schedule moves r monotonically, so at
            # most the current and the previous layer are kept
            while len(self._layers) >= 2:
                self._layers.pop(next(iter(self._layers)))
            lay = BSAAttention(self.geom, self.r, 1.0, 1.0, self.B, self.Hh, self.d, device=self.device,
                               scale=1.0 / math.sqrt(self.d))
            self._layers[self.r] = lay
        lay.set_knobs(resolve_k(self.f, N), self.tau)
        return lay

    def forward(self, Q, K, V):
        return bsa_attention(Q, K, V, self._layer())

    def forward_qkv(self, qkv):
        """qkv [B, L, 3, Hh, d] (a fused projection) -> O [B, L, Hh, d]."""
        return bsa_attention_qkv(qkv, self._layer())


class DiTAttentionBlock(torch.nn.Module):
    """The self-attention half of a DiT block (Wan-style, the paper's base model) with BSA as the
    attention: x [B, L, C] -> LayerNorm -> fused QKV projection [B, L, 3, Hh, d] -> BSA (strided, no copies)
    -> out-projection -> residual. The projections are plain library GEMMs (torch / cuBLAS); every step of the
    attention runs in libbsa. C = Hh * d (Wan2.1-1.3B: 12 x 128 = 1536)."""

    def __init__(self, geom: Geometry, B: int, Hh: int, d: int, schedule: AnnealSchedule | None = None,
                 r: float = 0.5, f: float = 0.1, tau: float = 0.9, device="cuda", dtype=torch.bfloat16):
        super().__init__()
        C = Hh * d
        self.Hh, self.d = Hh, d
        self.norm = torch.nn.LayerNorm(C, elementwise_affine=False, device=device, dtype=dtype)
        self.qkv = torch.nn.Linear(C, 3 * C, bias=True, device=device, dtype=dtype)
        self.out = torch.nn.Linear(C, C, bias=True, device=device, dtype=dtype)
        self.attn = BSASelfAttention(geom, B, Hh, d, schedule=schedule, r=r, f=f, tau=tau, device=device)

    def set_step(self, step: int):
        self.attn.set_step(step)

    def forward(self, x):
        B, L, C = x.shape
        qkv = self.qkv(self.norm(x)).view(B, L, 3, self.Hh, self.d)
        o = self.attn.forward_qkv(qkv)
        return x + self.out(o.reshape(B, L, C))
