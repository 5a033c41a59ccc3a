"""BSAAttention: one BSA attention layer's forward + backward with every buffer preallocated.

This is the call a training step makes (and what bench.py times): each method enqueues the
C-ABI calls of include/bsa.h on the current CUDA stream; Python only passes pointers.

    layer = BSAAttention(Geometry(21, 30, 52), r=0.5, f=0.1, tau=0.9, B=1, Hh=12, d=128)
    O = layer.forward(Q, K, V)            # a1..a7: partition (cached), selection, sparse attention + fill
    dQ, dK, dV = layer.backward(dO)       # a8

Q, K, V, dO and the outputs are bf16 [B, Hh, L, d] tensors with contiguous channels and any batch / head /
token strides (include/bsa.h bsa_tensor): a model's [B, L, Hh, d] activations go in as x.transpose(1, 2), and
the Q/K/V slices of a fused [B, L, 3, Hh, d] projection go in without a copy.

Buffer sizes depend only on the geometry, r, B, Hh and d; Eq.3's k and Eq.4's tau can change between calls
(set_knobs), which is what the annealed schedule of P:253 does every step.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import (OP_ATTN_BWD, OP_ATTN_FWD, OP_SELECT_KV, BSAError, Geometry, _check, _ptr, bsa_sizes, bsa_workspace_bytes, lib,
               resolve_k, tensor_desc)


class BSAAttention:
    def __init__(self, geom: Geometry, r: float, f, tau: float, B: int, Hh: int, d: int, device="cuda",
                 scale=None, cache_partition: bool = True, kv_mode: int = 0):
        self.g, self.r = geom, float(r)
        self.B, self.Hh, self.d = B, Hh, d
        self.N, self.Lq, self.max_kept = bsa_sizes(geom, r)
        self.SR = max(8, 1 << max(0, self.max_kept - 1).bit_length())  # query-block slot rows (kernels.h slot_rows)
        self.set_knobs(f, tau)
        self.scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None and torch.cuda.is_available():
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.cache_partition = cache_partition
        self.kv_mode = int(kv_mode)  # 0 = two_stage (the library's reading), 1 = unified_prob (C28)
        dev, N, Lq, L = self.device, self.N, self.Lq, geom.L
        i32 = dict(dtype=torch.int32, device=dev)
        self.block_off = torch.empty(N + 1, **i32)
        self.block_tok = torch.empty(L, **i32)
        self.block_ext = torch.empty(N, 3, **i32)
        self.kept_off = torch.empty(N + 1, **i32)
        self.kept_tok = torch.empty(B, Hh, Lq, **i32)
        self.donor = torch.empty(B, Hh, L, **i32)
        self.q_pooled = torch.empty(B, Hh, N, d, dtype=torch.float64, device=dev)
        self.q_packed = torch.empty(B, Hh, Lq, d, dtype=torch.bfloat16, device=dev)
        self.q2k_num = torch.empty(B, Hh, N, **i32)
        self.q2k_idx = torch.empty(B, Hh, N, N, **i32)
        self.k2q_num = torch.empty(B, Hh, N, **i32)
        self.k2q_idx = torch.empty(B, Hh, N, N, **i32)
        self.lse = torch.empty(B, Hh, Lq, dtype=torch.float32, device=dev)
        self._own = {}  # O, dQ, dK, dV: allocated on first use when the caller passes no output tensors
        self.ws_kv_bytes = bsa_workspace_bytes(OP_SELECT_KV, geom, r, B, Hh, d)
        self.ws_fwd_bytes = bsa_workspace_bytes(OP_ATTN_FWD, geom, r, B, Hh, d)
        self.ws_bwd_bytes = bsa_workspace_bytes(OP_ATTN_BWD, geom, r, B, Hh, d)
        self.ws = torch.empty(max(self.ws_kv_bytes, self.ws_fwd_bytes, self.ws_bwd_bytes, 256), dtype=torch.uint8,
                              device=dev)
        self._g = geom.c()
        self._partitioned = False
        self._saved = None
        self._O = None

    # ---------------------------------------------------------------- knobs and buffers
    def set_knobs(self, f=None, tau=None):
        """Eq.3's key count (a fraction f in (0, 1] -> k = ceil(f N) by bsa_resolve_k, or an int k) and Eq.4's
        tau for the next forward. Neither changes any buffer size."""
        if f is not None:
            self.k = resolve_k(f, self.N) if isinstance(f, float) else int(f)
            if not 1 <= self.k <= self.N:
                raise BSAError(f"k must be in [1, {self.N}] (got {self.k})")
        if tau is not None:
            self.tau = float(tau)

    def _buf(self, name):
        t = self._own.get(name)
        if t is None:
            t = torch.empty(self.B, self.Hh, self.g.L, self.d, dtype=torch.bfloat16, device=self.device)
            self._own[name] = t
        return t

    @property
    def O(self):
        return self._buf("O")

    @property
    def dQ(self):
        return self._buf("dQ")

    @property
    def dK(self):
        return self._buf("dK")

    @property
    def dV(self):
        return self._buf("dV")

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _check_rows(self, what, *ts):
        shape = (self.B, self.Hh, self.g.L, self.d)
        for t in ts:
            if tuple(t.shape) != shape or t.dtype != torch.bfloat16 or t.stride(-1) != 1 or t.device != self.device:
                raise BSAError(f"{what} must be bf16 [B, Hh, L, d] = {shape} tensors on {self.device} with contiguous "
                               f"channels (got {tuple(t.shape)} {t.dtype} stride {t.stride()} on {t.device})")

    # ---------------------------------------------------------------- the path
    def partition(self):
        """a1; geometry-only, so cached after the first call when cache_partition."""
        if self._partitioned and self.cache_partition:
            return
        _check(lib().bsa_block_partition(ctypes.byref(self._g), self.r, _ptr(self.block_off), _ptr(self.block_tok),
                                         _ptr(self.block_ext), _ptr(self.kept_off), self._stream()),
               "bsa_block_partition")
        self._partitioned = True

    def select(self, Q: torch.Tensor, K: torch.Tensor):
        """a2..a6: query pruning (Eq.2) and KV-block admission (Eq.3, Eq.4) with its transpose."""
        self._check_rows("Q, K", Q, K)
        L, st = lib(), self._stream()
        self.partition()
        _check(L.bsa_select_queries(ctypes.byref(self._g), self.r, self.B, self.Hh, self.d, tensor_desc(Q),
                                    _ptr(self.kept_off), _ptr(self.kept_tok), _ptr(self.donor), _ptr(self.q_pooled),
                                    _ptr(self.q_packed), st), "bsa_select_queries")
        _check(L.bsa_select_kv_blocks_ex(ctypes.byref(self._g), self.B, self.Hh, self.d, tensor_desc(None),
                                         _ptr(self.q_pooled), tensor_desc(K), self.k, self.tau, self.kv_mode,
                                         _ptr(self.q2k_num), _ptr(self.q2k_idx), _ptr(self.k2q_num),
                                         _ptr(self.k2q_idx), None, _ptr(self.ws), self.ws.numel(), st),
               "bsa_select_kv_blocks_ex")

    def attend(self, Q, K, V, out=None):
        """a7 (Eq.5) + fill into `out` (default: the layer's own O buffer) and self.lse."""
        O = self.O if out is None else out
        self._check_rows("Q, K, V, out", K, V, O)
        _check(lib().bsa_attn_fwd(ctypes.byref(self._g), self.r, self.B, self.Hh, self.d, tensor_desc(None),
                                  tensor_desc(K), tensor_desc(V), _ptr(self.q_packed), _ptr(self.kept_off),
                                  _ptr(self.kept_tok), _ptr(self.donor), _ptr(self.q2k_num), _ptr(self.q2k_idx),
                                  ctypes.c_float(self.scale), tensor_desc(O), _ptr(self.lse), _ptr(self.ws),
                                  self.ws.numel(), self._stream()), "bsa_attn_fwd")
        self._O = O
        return O

    def forward(self, Q, K, V, out=None):
        self._check_rows("Q, K, V", Q, K, V)
        self.select(Q, K)
        self._saved = (Q, K, V)
        return self.attend(Q, K, V, out)

    def backward(self, dO, out=None, saved=None):
        """a8: returns (dQ, dK, dV) for the last forward, into `out` = (dQ, dK, dV) if given (default: the
        layer's own buffers). `saved` = (Q, K, V, O) of that forward (default: the tensors the layer kept; autograd
        passes its own saved tensors so in-place edits are caught by their version counters)."""
        if self._saved is None:
            raise BSAError("backward() before forward()")
        Q, K, V, O = saved if saved is not None else (*self._saved, self._O)
        dQ, dK, dV = (self.dQ, self.dK, self.dV) if out is None else out
        self._check_rows("dO, dQ, dK, dV, K, V, O", dO, dQ, dK, dV, K, V, O)
        T = tensor_desc
        _check(lib().bsa_attn_bwd(ctypes.byref(self._g), self.r, self.B, self.Hh, self.d, T(None), T(K), T(V), T(O),
                                  T(dO), _ptr(self.q_packed), _ptr(self.kept_off), _ptr(self.kept_tok),
                                  _ptr(self.donor), _ptr(self.q2k_num), _ptr(self.q2k_idx), _ptr(self.k2q_num),
                                  _ptr(self.k2q_idx), _ptr(self.lse),
                                  ctypes.c_float(self.scale), T(dQ), T(dK), T(dV), _ptr(self.ws), self.ws.numel(),
                                  self._stream()), "bsa_attn_bwd")
        return dQ, dK, dV

    # ---------------------------------------------------------------- accounting (host side, untimed)
    def executed_pairs(self) -> int:
        """P = sum over (b,h,i) of |kept_i| * sum_{j in S_i} |block_j| (actual tokens)."""
        bsz = (self.block_off[1:] - self.block_off[:-1]).to(torch.int64)  # [N]
        kept = (self.kept_off[1:] - self.kept_off[:-1]).to(torch.int64)   # [N]
        N = self.N
        mask = torch.arange(N, device=self.device)[None, None, None, :] < self.q2k_num[..., None]
        idx = torch.where(mask, self.q2k_idx, torch.zeros_like(self.q2k_idx)).long()
        kv_tokens = torch.where(mask, bsz[idx], torch.zeros_like(idx)).sum(-1)  # [B,Hh,N]
        return int((kv_tokens * kept[None, None, :]).sum().item())

    def admitted_block_rows(self) -> int:
        """sum over (b,h,i) of |kept_i| * |S_i|: query rows times admitted KV blocks, i.e. the dQ partial rows the
        KV-stationary backward reduces into L2 (one row of d fp32 per admitted (query row, KV block))."""
        kept = (self.kept_off[1:] - self.kept_off[:-1]).to(torch.int64)
        return int((self.q2k_num.to(torch.int64) * kept[None, None, :]).sum().item())

    def flops(self) -> dict:
        P = self.executed_pairs()
        d = self.d
        dense = self.B * self.Hh * self.g.L * self.g.L
        return dict(pairs=P, fwd=4 * d * P, bwd=10 * d * P, total=14 * d * P, dense_total=14 * d * dense,
                    density=P / dense)

    def sparsity(self) -> dict:
        """Realised query keep fraction (Eq.2), mean KV keep fraction per query block (Eq.3 + Eq.4) and pair density."""
        kv = float(self.q2k_num.double().mean().item()) / self.N
        return dict(query_keep=self.Lq / self.g.L, kv_keep=kv, mean_admitted_blocks=kv * self.N)


class BSAStepGraph:
    """One training step of a layer (selection, forward, backward on fixed input buffers) captured into a
    CUDA graph: replay() re-runs every libbsa kernel of the step with one launch. Inputs are read from the
    captured tensors, so refill them in place (copy_) between replays; outputs land in the layer's
    O / dQ / dK / dV buffers. Library event timing (bsa_timing_enable) must be off while capturing."""

    def __init__(self, layer: BSAAttention, Q, K, V, dO, warmup: int = 2):
        self.layer, self.inputs = layer, (Q, K, V, dO)
        dev = layer.device
        self.stream = torch.cuda.Stream(dev)
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):  # partition cache, lazy buffers, allocator state
                layer.forward(Q, K, V)
                layer.backward(dO)
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            layer.forward(Q, K, V)
            layer.backward(dO)
        torch.cuda.current_stream(dev).wait_stream(self.stream)

    def replay(self):
        self.graph.replay()
        return self.layer.O, self.layer.dQ, self.layer.dK, self.layer.dV
