"""CPU fp64 oracle for BSA — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this package. It wraps oracle/bsa_oracle.c (plain C, OpenMP, fp64) with ctypes and shares
no code with the CUDA product path in paper_2509_01085_b200/.

See bsa_oracle.c for the per-function citations of PAPER.md / SPEC.md and the pin status.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bsa_oracle.c")
_LIB = os.path.join(_HERE, "libbsa_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call([
            "gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
            "-std=c11", "-o", _LIB, _SRC, "-lm",
        ])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        _lib.or_normal_quantile.restype = ctypes.c_double
        _lib.or_normal_quantile.argtypes = [ctypes.c_double]
        _lib.or_keep_count.restype = ctypes.c_int
        _lib.or_keep_count.argtypes = [ctypes.c_double, ctypes.c_int]
        _lib.or_flatten.restype = ctypes.c_int
    return _lib


class _G(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("T", "H", "W", "ct", "ch", "cw", "ut", "uh", "uw")]


@dataclass(frozen=True)
class Geom:
    T: int
    H: int
    W: int
    ct: int
    ch: int
    cw: int
    ut: int = 0
    uh: int = 0
    uw: int = 0

    @property
    def unit(self):
        return (self.ut or self.ct, self.uh or self.ch, self.uw or self.cw)

    @property
    def L(self):
        return self.T * self.H * self.W

    def c(self) -> _G:
        u = self.unit
        return _G(self.T, self.H, self.W, self.ct, self.ch, self.cw, u[0], u[1], u[2])


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


_D = ctypes.c_double
_I = ctypes.c_int


def set_threads(n: int):
    lib().or_set_threads(int(n))


def max_threads() -> int:
    return int(lib().or_max_threads())


def sizes(g: Geom, r: float):
    N, Lq = _I(), _I()
    lib().or_sizes(ctypes.byref(g.c()), _D(r), ctypes.byref(N), ctypes.byref(Lq))
    return N.value, Lq.value


def keep_count(r: float, n: int) -> int:
    return int(lib().or_keep_count(r, n))


def normal_quantile(u: float) -> float:
    return float(lib().or_normal_quantile(u))


def partition(g: Geom, r: float):
    N, Lq = sizes(g, r)
    bo = np.zeros(N + 1, np.int32)
    bt = np.zeros(g.L, np.int32)
    be = np.zeros(3 * N, np.int32)
    ko = np.zeros(N + 1, np.int32)
    lib().or_partition(ctypes.byref(g.c()), _D(r), _p(bo, _I), _p(bt, _I), _p(be, _I), _p(ko, _I))
    return dict(N=N, Lq=Lq, block_off=bo, block_tok=bt, block_ext=be.reshape(N, 3), kept_off=ko)


def _f64(x) -> np.ndarray:
    """torch bf16/fp32 or numpy -> contiguous fp64 numpy [BH, L, d] (exact widening)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            x = x.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return x.reshape(-1, x.shape[-2], x.shape[-1]) if x.ndim >= 3 else x


def pool(g: Geom, X) -> np.ndarray:
    X = _f64(X)
    BH, L, d = X.shape
    N = sizes(g, 1.0)[0]
    out = np.zeros((BH, N, d), np.float64)
    lib().or_pool(ctypes.byref(g.c()), _I(BH), _I(d), _p(X, _D), _p(out, _D))
    return out


def select_queries(g: Geom, r: float, Q):
    Q = _f64(Q)
    BH, L, d = Q.shape
    N, Lq = sizes(g, r)
    kept = np.zeros((BH, Lq), np.int32)
    donor = np.zeros((BH, L), np.int32)
    um = np.zeros((BH, L), np.float64)
    dm = np.zeros((BH, L), np.float64)
    lib().or_select_queries(ctypes.byref(g.c()), _D(r), _I(BH), _I(d), _p(Q, _D), _p(kept, _I), _p(donor, _I),
                            _p(um, _D), _p(dm, _D))
    return dict(kept_tok=kept, donor=donor, unit_margin=um, donor_margin=dm)


def select_kv_from_pooled(Qc: np.ndarray, Kc: np.ndarray, k: int, tau: float):
    Qc = np.ascontiguousarray(Qc, np.float64)
    Kc = np.ascontiguousarray(Kc, np.float64)
    BH, N, d = Qc.shape
    num = np.zeros((BH, N), np.int32)
    idx = np.zeros((BH, N, N), np.int32)
    th = np.zeros((BH, N), np.float64)
    sc = np.zeros((BH, N, N), np.float64)
    tm = np.zeros((BH, N), np.float64)
    mm = np.zeros((BH, N), np.float64)
    om = np.zeros((BH, N), np.float64)
    lib().or_select_kv(_I(N), _I(BH), _I(d), _p(Qc, _D), _p(Kc, _D), _I(k), _D(tau), _p(num, _I), _p(idx, _I),
                       _p(th, _D), _p(sc, _D), _p(tm, _D), _p(mm, _D), _p(om, _D))
    return dict(q2k_num=num, q2k_idx=idx, thresh=th, scores=sc, thr_margin=tm, mass_margin=mm,
                order_margin=om)


def select_kv(g: Geom, Q, K, k: int, tau: float):
    return select_kv_from_pooled(pool(g, Q), pool(g, K), k, tau)


def select_kv_unified_from_pooled(Qc: np.ndarray, Kc: np.ndarray, k: int):
    """SPEC's unified_prob reading (C28): Eq.3 over the softmax-normalised row gives
    a probability-mass target p, Eq.4 admits the shortest prefix reaching it."""
    Qc = np.ascontiguousarray(Qc, np.float64)
    Kc = np.ascontiguousarray(Kc, np.float64)
    BH, N, d = Qc.shape
    num = np.zeros((BH, N), np.int32)
    idx = np.zeros((BH, N, N), np.int32)
    th = np.zeros((BH, N), np.float64)
    mm = np.zeros((BH, N), np.float64)
    lib().or_select_kv_unified(_I(N), _I(BH), _I(d), _p(Qc, _D), _p(Kc, _D), _I(k), _p(num, _I), _p(idx, _I),
                               _p(th, _D), _p(mm, _D))
    return dict(q2k_num=num, q2k_idx=idx, thresh=th, mass_margin=mm)


def select_kv_unified(g: Geom, Q, K, k: int):
    return select_kv_unified_from_pooled(pool(g, Q), pool(g, K), k)


def attn_fwd(g: Geom, r: float, Q, K, V, kept_tok, donor, q2k_num, q2k_idx, scale: float):
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    BH, L, d = Q.shape
    N, Lq = sizes(g, r)
    O = np.zeros((BH, L, d), np.float64)
    lse = np.zeros((BH, Lq), np.float64)
    kt, dn = np.ascontiguousarray(kept_tok, np.int32), np.ascontiguousarray(donor, np.int32)
    qn, qi = np.ascontiguousarray(q2k_num, np.int32), np.ascontiguousarray(q2k_idx, np.int32)
    lib().or_attn_fwd(ctypes.byref(g.c()), _D(r), _I(BH), _I(d), _p(Q, _D), _p(K, _D), _p(V, _D), _p(kt, _I),
                      _p(dn, _I), _p(qn, _I), _p(qi, _I), _D(scale), _p(O, _D), _p(lse, _D))
    return O, lse


def attn_fwd_rows(g: Geom, r: float, Q, K, V, kept_tok, q2k_num, q2k_idx, scale: float, rows):
    Q, K, V = _f64(Q), _f64(K), _f64(V)
    BH, L, d = Q.shape
    rows = np.ascontiguousarray(rows, np.int32)
    Os = np.zeros((len(rows), d), np.float64)
    lse = np.zeros(len(rows), np.float64)
    kt = np.ascontiguousarray(kept_tok, np.int32)
    qn, qi = np.ascontiguousarray(q2k_num, np.int32), np.ascontiguousarray(q2k_idx, np.int32)
    lib().or_attn_fwd_rows(ctypes.byref(g.c()), _D(r), _I(BH), _I(d), _p(Q, _D), _p(K, _D), _p(V, _D),
                           _p(kt, _I), _p(qn, _I), _p(qi, _I), _D(scale), _I(len(rows)), _p(rows, _I),
                           _p(Os, _D), _p(lse, _D))
    return Os, lse


def attn_bwd(g: Geom, r: float, Q, K, V, dO, kept_tok, donor, q2k_num, q2k_idx, scale: float):
    Q, K, V, dO = _f64(Q), _f64(K), _f64(V), _f64(dO)
    BH, L, d = Q.shape
    dQ = np.zeros((BH, L, d), np.float64)
    dK = np.zeros_like(dQ)
    dV = np.zeros_like(dQ)
    kt, dn = np.ascontiguousarray(kept_tok, np.int32), np.ascontiguousarray(donor, np.int32)
    qn, qi = np.ascontiguousarray(q2k_num, np.int32), np.ascontiguousarray(q2k_idx, np.int32)
    lib().or_attn_bwd(ctypes.byref(g.c()), _D(r), _I(BH), _I(d), _p(Q, _D), _p(K, _D), _p(V, _D), _p(dO, _D),
                      _p(kt, _I), _p(dn, _I), _p(qn, _I), _p(qi, _I), _D(scale), _p(dQ, _D), _p(dK, _D),
                      _p(dV, _D))
    return dQ, dK, dV


def run_selection(g: Geom, r: float, k: int, tau: float, Q, K):
    qs = select_queries(g, r, Q)
    kv = select_kv(g, Q, K, k, tau)
    return qs, kv


def resolve_k(f: float, N: int) -> int:
    """k = clamp(ceil(f*N - 1e-9), 1, N) (C6 rule applied to the Eq.3 key count)."""
    return keep_count(f, N)
