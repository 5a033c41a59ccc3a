"""paper_2509_01085_b200 — B200-native BSA (Bidirectional Sparse Attention, arXiv 2509.01085).

Thin Python binding over the C ABI of libbsa.so (include/bsa.h). The functions below have the
same names as the C entry points and only marshal arguments: every step of the hot path runs in
the library's sm_100a kernels. PyTorch provides device memory and the current CUDA stream.
There is no CPU fallback: if libbsa.so is missing or the device is not sm_100, calls raise.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

__all__ = [
    "BSAError", "Geometry", "lib", "bsa_sizes", "bsa_workspace_bytes", "bsa_block_partition", "bsa_select_queries",
    "bsa_select_kv_blocks", "bsa_attn_fwd", "bsa_attn_bwd", "bsa_sp_relayout", "Selection", "select", "resolve_k",
    "kv_quantile", "tensor_desc",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BSA_LIB_PATH") or os.path.join(_HERE, "libbsa.so")  # override: debug builds only

OP_SELECT_KV, OP_ATTN_FWD, OP_ATTN_BWD = 1, 2, 3


class BSAError(RuntimeError):
    pass


class _CGeom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("T", "H", "W", "ct", "ch", "cw", "ut", "uh", "uw")]


class _CTensor(ctypes.Structure):
    """include/bsa.h bsa_tensor: bf16 [B, Hh, L, d], element (b, h, n, c) at ptr[b sb + h sh + n sl + c]."""
    _fields_ = [("ptr", ctypes.c_void_p), ("sb", ctypes.c_int64), ("sh", ctypes.c_int64), ("sl", ctypes.c_int64)]


def tensor_desc(t) -> _CTensor:
    """bsa_tensor of a bf16 CUDA tensor shaped [B, Hh, L, d] with contiguous channels (any batch / head / token
    strides, e.g. x.transpose(1, 2) of a model's [B, L, Hh, d]); a NULL descriptor for None. Marshalling only."""
    if t is None:
        return _CTensor(None, 0, 0, 0)
    if t.dim() != 4 or t.dtype != torch.bfloat16 or not t.is_cuda:
        raise BSAError(f"expected a bf16 CUDA tensor [B, Hh, L, d], got {tuple(t.shape)} {t.dtype} {t.device}")
    if t.stride(3) != 1:
        raise BSAError("the d channels of each row must be contiguous (stride(-1) == 1)")
    return _CTensor(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2))


@dataclass(frozen=True)
class Geometry:
    """Latent grid (T,H,W), cuboid block (ct,ch,cw), selection unit/window (
    0 = whole block, the north_star's block-centre selection)."""
    T: int
    H: int
    W: int
    ct: int = 4
    ch: int = 4
    cw: int = 4
    ut: int = 0
    uh: int = 0
    uw: int = 0

    @property
    def L(self) -> int:
        return self.T * self.H * self.W

    def c(self) -> _CGeom:
        return _CGeom(self.T, self.H, self.W, self.ct, self.ch, self.cw, self.ut, self.uh, self.uw)


_lib = None
_P = ctypes.c_void_p
_I = ctypes.c_int32
_D = ctypes.c_double
_F = ctypes.c_float
_S = ctypes.c_size_t


def lib() -> ctypes.CDLL:
    """Load libbsa.so (built by paper_2509_01085_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BSAError(f"{LIB_PATH} is missing: run `python -m paper_2509_01085_b200.build` (no fallback path)")
        L = ctypes.CDLL(LIB_PATH)
        gp = ctypes.POINTER(_CGeom)
        _T = _CTensor
        L.bsa_version.restype = _I
        L.bsa_strerror.restype = ctypes.c_char_p
        L.bsa_strerror.argtypes = [_I]
        L.bsa_last_error.restype = ctypes.c_char_p
        L.bsa_sizes.argtypes = [gp, _D, _P, _P, _P]
        L.bsa_workspace_bytes.argtypes = [_I, gp, _D, _I, _I, _I, ctypes.POINTER(_S)]
        L.bsa_block_partition.argtypes = [gp, _D, _P, _P, _P, _P, _P]
        L.bsa_select_queries.argtypes = [gp, _D, _I, _I, _I, _T, _P, _P, _P, _P, _P, _P]
        L.bsa_select_kv_blocks.argtypes = [gp, _I, _I, _I, _T, _P, _T, _I, _D, _P, _P, _P, _P, _P, _P, _S, _P]
        L.bsa_attn_fwd.argtypes = [gp, _D, _I, _I, _I, _T, _T, _T, _P, _P, _P, _P, _P, _P, _F, _T, _P, _P, _S, _P]
        L.bsa_attn_bwd.argtypes = [gp, _D, _I, _I, _I, _T, _T, _T, _T, _T, _P, _P, _P, _P, _P, _P, _P, _P, _P, _F,
                                   _T, _T, _T, _P, _S, _P]
        L.bsa_sp_relayout.argtypes = [_I, _I, _I, _I, _I, _I, _P, _P, _P]
        L.bsa_sp_relayout_group.argtypes = [_I, _I, _I, _I, _I, _I, _I, _P, _P, _P]
        L.bsa_select_kv_blocks_ex.argtypes = [gp, _I, _I, _I, _T, _P, _T, _I, _D, _I, _P, _P, _P, _P, _P, _P, _S, _P]
        L.bsa_resolve_k.argtypes = [_D, _I, _P]
        L.bsa_kv_quantile.argtypes = [_I, _I, _P]
        L.bsa_launch_count.restype = ctypes.c_int64
        L.bsa_launch_count.argtypes = []
        L.bsa_timing_enable.argtypes = [_I]
        L.bsa_timing_read.argtypes = [_P, _P, _I]
        L.bsa_set_bwd_path.argtypes = [_I]
        L.bsa_set_fwd_tiling.argtypes = [_I, _I]
        L.bsa_bwd_ds_capacity.argtypes = [gp, _D, _I, _I, _I, _P]
        for f in ("bsa_timing_enable", "bsa_timing_read",
                  "bsa_sizes", "bsa_workspace_bytes", "bsa_block_partition", "bsa_select_queries",
                  "bsa_select_kv_blocks", "bsa_attn_fwd", "bsa_attn_bwd", "bsa_sp_relayout",
                  "bsa_select_kv_blocks_ex", "bsa_resolve_k", "bsa_kv_quantile", "bsa_set_bwd_path", "bsa_bwd_ds_capacity",
                  "bsa_sp_relayout_group", "bsa_set_fwd_tiling"):
            getattr(L, f).restype = _I
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        L = lib()
        raise BSAError(f"{what}: {L.bsa_strerror(rc).decode()} — {L.bsa_last_error().decode()}")


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise BSAError("libbsa expects contiguous CUDA tensors")


def _need_rows(shape, *ts):
    """Strided [B, Hh, L, d] bf16 operands: shape and channel contiguity (strides are checked by the library)."""
    for t in ts:
        if t is not None and (tuple(t.shape) != tuple(shape) or t.dtype != torch.bfloat16 or not t.is_cuda
                              or t.stride(-1) != 1):
            raise BSAError(f"expected a bf16 CUDA [B, Hh, L, d] = {tuple(shape)} tensor with contiguous channels, got "
                           f"{tuple(t.shape)} {t.dtype} stride {t.stride()}")


def _need_i32(name, t, shape):
    if t is None or tuple(t.shape) != tuple(shape) or t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
        got = None if t is None else (tuple(t.shape), t.dtype)
        raise BSAError(f"{name}: expected a contiguous int32 CUDA tensor of shape {tuple(shape)}, got {got}")


def bsa_sizes(g: Geometry, r: float):
    """(N, Lq, max_block_kept) for geometry g and keep ratio r (host only)."""
    N, Lq, mk = _I(), _I(), _I()
    _check(lib().bsa_sizes(ctypes.byref(g.c()), r, ctypes.byref(N), ctypes.byref(Lq), ctypes.byref(mk)), "bsa_sizes")
    return N.value, Lq.value, mk.value


def bsa_workspace_bytes(op: int, g: Geometry, r: float, B: int, Hh: int, d: int) -> int:
    n = _S()
    _check(lib().bsa_workspace_bytes(op, ctypes.byref(g.c()), r, B, Hh, d, ctypes.byref(n)), "bsa_workspace_bytes")
    return n.value


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


def bsa_block_partition(g: Geometry, r: float, device="cuda"):
    """a1: dict of device int32 tensors block_off[N+1], block_tok[L], block_ext[N,3], kept_off[N+1]."""
    N, Lq, _ = bsa_sizes(g, r)
    dev = torch.device(device)
    out = dict(
        block_off=torch.empty(N + 1, dtype=torch.int32, device=dev),
        block_tok=torch.empty(g.L, dtype=torch.int32, device=dev),
        block_ext=torch.empty(N, 3, dtype=torch.int32, device=dev),
        kept_off=torch.empty(N + 1, dtype=torch.int32, device=dev),
    )
    _check(lib().bsa_block_partition(ctypes.byref(g.c()), r, _ptr(out["block_off"]), _ptr(out["block_tok"]),
                                     _ptr(out["block_ext"]), _ptr(out["kept_off"]), _stream(dev)),
           "bsa_block_partition")
    out["N"], out["Lq"] = N, Lq
    return out


def bsa_select_queries(g: Geometry, r: float, Q: torch.Tensor, kept_off: torch.Tensor, pooled: bool = True,
                       packed: bool = True):
    """a2+a3 (Eq.2): returns kept_tok [B,Hh,Lq], donor [B,Hh,L], q_pooled [B,Hh,N,d] fp64 or None,
    q_packed [B,Hh,Lq,d] bf16 or None."""
    B, Hh, L, d = Q.shape
    _need_rows((B, Hh, g.L, d), Q)
    N, Lq, _ = bsa_sizes(g, r)
    _need_i32("kept_off", kept_off, (N + 1,))
    dev = Q.device
    kept = torch.empty(B, Hh, Lq, dtype=torch.int32, device=dev)
    donor = torch.empty(B, Hh, L, dtype=torch.int32, device=dev)
    qp = torch.empty(B, Hh, N, d, dtype=torch.float64, device=dev) if pooled else None
    qs = torch.empty(B, Hh, Lq, d, dtype=torch.bfloat16, device=dev) if packed else None
    _check(lib().bsa_select_queries(ctypes.byref(g.c()), r, B, Hh, d, tensor_desc(Q), _ptr(kept_off), _ptr(kept), _ptr(donor),
                                    _ptr(qp), _ptr(qs), _stream(dev)), "bsa_select_queries")
    return kept, donor, qp, qs


KV_TWO_STAGE, KV_UNIFIED_PROB = 0, 1


def bsa_select_kv_blocks(g: Geometry, Q: torch.Tensor, K: torch.Tensor, k: int, tau: float, q_pooled=None,
                         with_k2q: bool = True, with_thresh: bool = False, mode: int = KV_TWO_STAGE):
    """a4-a6 (Eq.3, Eq.4): returns q2k_num [B,Hh,N], q2k_idx [B,Hh,N,N] (row i valid up to q2k_num),
    k2q_num, k2q_idx (or None), thresh (or None). mode = KV_UNIFIED_PROB selects SPEC's unified_prob reading
    (bsa_select_kv_blocks_ex; tau unused)."""
    B, Hh, L, d = K.shape
    _need_rows((B, Hh, g.L, d), Q, K)
    _need_cuda(q_pooled)
    N = bsa_sizes(g, 1.0)[0]
    dev = K.device
    num = torch.empty(B, Hh, N, dtype=torch.int32, device=dev)
    idx = torch.empty(B, Hh, N, N, dtype=torch.int32, device=dev)
    knum = torch.empty(B, Hh, N, dtype=torch.int32, device=dev) if with_k2q else None
    kidx = torch.empty(B, Hh, N, N, dtype=torch.int32, device=dev) if with_k2q else None
    th = torch.empty(B, Hh, N, dtype=torch.float64, device=dev) if with_thresh else None
    nb = bsa_workspace_bytes(OP_SELECT_KV, g, 1.0, B, Hh, d)
    ws = _ws(nb, dev)
    _check(lib().bsa_select_kv_blocks_ex(ctypes.byref(g.c()), B, Hh, d, tensor_desc(Q), _ptr(q_pooled), tensor_desc(K), int(k),
                                         float(tau), int(mode), _ptr(num), _ptr(idx), _ptr(knum), _ptr(kidx), _ptr(th),
                                         _ptr(ws), nb, _stream(dev)), "bsa_select_kv_blocks_ex")
    return num, idx, knum, kidx, th


def bsa_attn_fwd(g: Geometry, r: float, Q, K, V, kept_off, kept_tok, donor, q2k_num, q2k_idx, scale=None,
                 q_packed=None, out=None, lse=None):
    """a7 (Eq.5) + fill: returns O [B,Hh,L,d] bf16 and lse [B,Hh,Lq] fp32. Q, K, V, out may be strided
    [B, Hh, L, d] views (contiguous channels)."""
    B, Hh, L, d = K.shape
    N, Lq, _ = bsa_sizes(g, r)
    dev = K.device
    O = torch.empty(B, Hh, L, d, dtype=torch.bfloat16, device=dev) if out is None else out
    _need_rows((B, Hh, g.L, d), Q, K, V, O)
    _need_i32("kept_off", kept_off, (N + 1,))
    _need_i32("kept_tok", kept_tok, (B, Hh, Lq))
    _need_i32("donor", donor, (B, Hh, L))
    _need_i32("q2k_num", q2k_num, (B, Hh, N))
    _need_i32("q2k_idx", q2k_idx, (B, Hh, N, N))
    if q_packed is not None and (tuple(q_packed.shape) != (B, Hh, Lq, d) or not q_packed.is_contiguous()):
        raise BSAError("q_packed must be a contiguous [B, Hh, Lq, d] bf16 tensor")
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    lse = torch.empty(B, Hh, Lq, dtype=torch.float32, device=dev) if lse is None else lse
    if tuple(lse.shape) != (B, Hh, Lq) or lse.dtype != torch.float32 or not lse.is_contiguous():
        raise BSAError("lse must be a contiguous fp32 [B, Hh, Lq] tensor")
    nb = bsa_workspace_bytes(OP_ATTN_FWD, g, r, B, Hh, d)
    ws = _ws(nb, dev)
    _check(lib().bsa_attn_fwd(ctypes.byref(g.c()), r, B, Hh, d, tensor_desc(Q), tensor_desc(K), tensor_desc(V),
                              _ptr(q_packed), _ptr(kept_off), _ptr(kept_tok), _ptr(donor), _ptr(q2k_num), _ptr(q2k_idx),
                              float(scale), tensor_desc(O), _ptr(lse), _ptr(ws), nb, _stream(dev)), "bsa_attn_fwd")
    return O, lse


def bsa_attn_bwd(g: Geometry, r: float, Q, K, V, O, dO, kept_off, kept_tok, donor, q2k_num, q2k_idx, k2q_num,
                 k2q_idx, lse, scale=None, q_packed=None, ws=None, out=None):
    """a8: returns dQ, dK, dV [B,Hh,L,d] bf16 (into `out` = (dQ, dK, dV) if given; strided views allowed)."""
    B, Hh, L, d = K.shape
    N, Lq, _ = bsa_sizes(g, r)
    dev = K.device
    mk = lambda: torch.empty(B, Hh, L, d, dtype=torch.bfloat16, device=dev)  # noqa: E731
    dQ, dK, dV = (mk(), mk(), mk()) if out is None else out
    _need_rows((B, Hh, g.L, d), Q, K, V, O, dO, dQ, dK, dV)
    _need_i32("kept_off", kept_off, (N + 1,))
    _need_i32("kept_tok", kept_tok, (B, Hh, Lq))
    _need_i32("donor", donor, (B, Hh, L))
    _need_i32("q2k_num", q2k_num, (B, Hh, N))
    _need_i32("q2k_idx", q2k_idx, (B, Hh, N, N))
    _need_i32("k2q_num", k2q_num, (B, Hh, N))
    _need_i32("k2q_idx", k2q_idx, (B, Hh, N, N))
    if tuple(lse.shape) != (B, Hh, Lq) or lse.dtype != torch.float32 or not lse.is_contiguous():
        raise BSAError("lse must be a contiguous fp32 [B, Hh, Lq] tensor")
    if q_packed is not None and (tuple(q_packed.shape) != (B, Hh, Lq, d) or not q_packed.is_contiguous()):
        raise BSAError("q_packed must be a contiguous [B, Hh, Lq, d] bf16 tensor")
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    nb = bsa_workspace_bytes(OP_ATTN_BWD, g, r, B, Hh, d)
    if ws is None or ws.numel() < nb:
        ws = _ws(nb, dev)
    T = tensor_desc
    _check(lib().bsa_attn_bwd(ctypes.byref(g.c()), r, B, Hh, d, T(Q), T(K), T(V), T(O), T(dO), _ptr(q_packed),
                              _ptr(kept_off), _ptr(kept_tok), _ptr(donor), _ptr(q2k_num), _ptr(q2k_idx),
                              _ptr(k2q_num), _ptr(k2q_idx), _ptr(lse), float(scale), T(dQ), T(dK), T(dV), _ptr(ws), nb,
                              _stream(dev)), "bsa_attn_bwd")
    return dQ, dK, dV


BWD_REDUCE, BWD_DS = 0, 1


def bwd_ds_capacity(g: Geometry, r: float, B: int, Hh: int, d: int) -> int:
    """Admitted-pair capacity of the backward's dS path (-1 unless BWD_DS is set); include/bsa.h."""
    out = ctypes.c_int64(0)
    _check(lib().bsa_bwd_ds_capacity(ctypes.byref(g.c()), r, B, Hh, d, ctypes.byref(out)), "bsa_bwd_ds_capacity")
    return int(out.value)


def set_bwd_path(mode: int):
    """Backward dQ path, process-wide (include/bsa.h bsa_set_bwd_path): BWD_REDUCE (default) or BWD_DS."""
    _check(lib().bsa_set_bwd_path(int(mode)), "bsa_set_bwd_path")


FWD_SMALL_FIRST, FWD_LARGE_FIRST = 0, 1


def set_fwd_tiling(min_slot_rows: int = 0, order: int = FWD_SMALL_FIRST):
    """Forward query tiling, process-wide (include/bsa.h bsa_set_fwd_tiling): a block's slot is its kept count
    rounded up to a power of two >= min_slot_rows (0 = default 16; >= SR = one slot per block)."""
    _check(lib().bsa_set_fwd_tiling(int(min_slot_rows), int(order)), "bsa_set_fwd_tiling")


SP_SEQ_TO_SEND, SP_RECV_TO_HEADS, SP_HEADS_TO_SEND, SP_RECV_TO_SEQ, SP_SEQ_TO_SEND_T, SP_RECV_T_TO_SEQ = 0, 1, 2, 3, 4, 5


def bsa_sp_relayout(mode: int, src: torch.Tensor, dst: torch.Tensor, B: int, Ls: int, Hh: int, d: int, P: int):
    """Row reorder around the Ulysses all-to-all (include/bsa.h, bsa_sp_relayout); writes dst."""
    _need_cuda(src, dst)
    if src.dtype != torch.bfloat16 or dst.dtype != torch.bfloat16 or not src.is_contiguous() or not dst.is_contiguous():
        raise BSAError("bsa_sp_relayout: src and dst must be contiguous bf16")
    if src.numel() != B * Ls * Hh * d or dst.numel() != src.numel():
        raise BSAError("bsa_sp_relayout: src/dst must hold B*Ls*Hh*d elements")
    _check(lib().bsa_sp_relayout(mode, B, Ls, Hh, d, P, _ptr(src), _ptr(dst), _stream(src.device)), "bsa_sp_relayout")
    return dst


SP_GROUP_SEND, SP_GROUP_RECV = 0, 1


def bsa_sp_relayout_group(mode: int, src: torch.Tensor, dst: torch.Tensor, Ls: int, Hh: int, d: int, P: int,
                          hoff: int, Hs: int):
    """Head-group token-major reorder (include/bsa.h, bsa_sp_relayout_group); writes dst."""
    _need_cuda(src, dst)
    if src.dtype != torch.bfloat16 or dst.dtype != torch.bfloat16 or not src.is_contiguous() or not dst.is_contiguous():
        raise BSAError("bsa_sp_relayout_group: src and dst must be contiguous bf16")
    big, small = Ls * Hh * d, P * Ls * Hs * d
    if (src.numel(), dst.numel()) != ((big, small) if mode == SP_GROUP_SEND else (small, big)):
        raise BSAError("bsa_sp_relayout_group: src/dst sizes do not match the mode")
    _check(lib().bsa_sp_relayout_group(mode, Ls, Hh, d, P, hoff, Hs, _ptr(src), _ptr(dst), _stream(src.device)),
           "bsa_sp_relayout_group")
    return dst


def resolve_k(f: float, N: int) -> int:
    """Eq.3 key count from a fraction: clamp(ceil(f*N - 1e-9), 1, N) (reading C6), computed by the library
    (bsa_resolve_k, host only)."""
    k = _I()
    _check(lib().bsa_resolve_k(float(f), int(N), ctypes.byref(k)), "bsa_resolve_k")
    return k.value


def kv_quantile(k: int, N: int) -> float:
    """Eq.3's z = U(1 - k/N) (argument clamped to [1/(2N), 1 - 1/(2N)]) exactly as bsa_select_kv_blocks uses it
    (bsa_kv_quantile, host only)."""
    z = _D()
    _check(lib().bsa_kv_quantile(int(k), int(N), ctypes.byref(z)), "bsa_kv_quantile")
    return z.value


@dataclass
class Selection:
    """Everything the attention kernels consume, produced by `select` on the device."""
    geom: Geometry
    r: float
    k: int
    tau: float
    part: dict
    kept_tok: torch.Tensor
    donor: torch.Tensor
    q_pooled: torch.Tensor
    q_packed: torch.Tensor
    q2k_num: torch.Tensor
    q2k_idx: torch.Tensor
    k2q_num: torch.Tensor
    k2q_idx: torch.Tensor


def select(g: Geometry, r: float, k: int, tau: float, Q: torch.Tensor, K: torch.Tensor, part=None) -> Selection:
    """a1-a6 on the device: partition, query pruning, KV-block admission (and its transpose)."""
    part = part if part is not None else bsa_block_partition(g, r, Q.device)
    kept, donor, qp, qs = bsa_select_queries(g, r, Q, part["kept_off"])
    num, idx, knum, kidx, _ = bsa_select_kv_blocks(g, Q, K, k, tau, q_pooled=qp)
    return Selection(g, r, k, tau, part, kept, donor, qp, qs, num, idx, knum, kidx)
