"""C-ABI library checks that need no GPU (`-m "not gpu"`): libbsa.so loads, exports every symbol
include/bsa.h declares, and its host-only logic (sizes, workspace sizing, validation) is right."""

import ctypes
import math
import os
import re

import pytest

import oracle as orc
import paper_2509_01085_b200 as bsa
from paper_2509_01085_b200 import build as bsa_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    bsa_build.build()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "bsa.h")).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(bsa_[a-z_0-9]+)\s*\(", text, re.M)))


def test_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 10
    L = ctypes.CDLL(bsa.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), s
    # the five hot-path entry points of SURVEY.md §8(b)
    for s in ("bsa_block_partition", "bsa_select_queries", "bsa_select_kv_blocks", "bsa_attn_fwd", "bsa_attn_bwd"):
        assert s in syms


def test_library_has_no_cpu_fallback_and_no_libcuda_link():
    # libbsa links the CUDA runtime statically and resolves the driver lazily; the oracle is not linked in
    import subprocess
    out = subprocess.run(["nm", "-D", bsa.LIB_PATH], capture_output=True, text=True).stdout
    assert "or_attn_fwd" not in out and "or_select_kv" not in out
    ldd = subprocess.run(["ldd", bsa.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcuda.so" not in ldd


@pytest.mark.parametrize("grid,block,unit,r", [((4, 8, 8), (2, 4, 4), (0, 0, 0), 0.5),
                                               ((21, 30, 52), (4, 4, 4), (0, 0, 0), 0.5),
                                               ((21, 45, 80), (4, 4, 4), (0, 0, 0), 0.5),
                                               ((41, 45, 80), (4, 4, 4), (0, 0, 0), 0.25),
                                               ((21, 30, 52), (4, 4, 4), (2, 2, 2), 0.5),
                                               ((5, 7, 9), (2, 3, 4), (1, 3, 2), 0.3)])
def test_sizes_match_oracle(grid, block, unit, r):
    g = bsa.Geometry(*grid, *block, *unit)
    N, Lq, mk = bsa.bsa_sizes(g, r)
    og = orc.Geom(*grid, *block, *unit)
    assert (N, Lq) == orc.sizes(og, r)
    p = orc.partition(og, r)
    import numpy as np
    assert mk == int(np.diff(p["kept_off"]).max())


def test_baseline_sizes():
    """N = 8 / 624 / 1440 / 2640 and L_q = r L exactly at r in {1, .5, .25}."""
    for grid, N in (((4, 8, 8), 8), ((21, 30, 52), 624), ((21, 45, 80), 1440), ((41, 45, 80), 2640)):
        block = (2, 4, 4) if grid == (4, 8, 8) else (4, 4, 4)
        g = bsa.Geometry(*grid, *block)
        for r in (1.0, 0.5, 0.25):
            n, lq, _ = bsa.bsa_sizes(g, r)
            assert n == N and lq == round(r * g.L)


def test_validation_errors_before_any_launch():
    L = bsa.lib()
    g = bsa.Geometry(4, 8, 8, 2, 4, 4)
    N = ctypes.c_int32()
    assert L.bsa_sizes(ctypes.byref(g.c()), 0.0, ctypes.byref(N), None, None) == 2  # r out of range
    assert L.bsa_sizes(ctypes.byref(g.c()), 1.5, None, None, None) == 2
    bad = bsa.Geometry(4, 8, 8, 2, 4, 4, 2, 3, 2)  # unit does not divide the block
    assert L.bsa_sizes(ctypes.byref(bad.c()), 0.5, None, None, None) == 2
    assert b"divide" in L.bsa_last_error()
    zero = bsa.Geometry(0, 8, 8, 2, 4, 4)
    assert L.bsa_sizes(ctypes.byref(zero.c()), 0.5, None, None, None) == 1
    n = ctypes.c_size_t()
    assert L.bsa_workspace_bytes(2, ctypes.byref(g.c()), 0.5, 1, 2, 96, ctypes.byref(n)) == 1  # d unsupported
    T = bsa._CTensor
    t16 = T(256, 2 * 256 * 64, 256 * 64, 64)  # a well-formed contiguous [1, 2, 256, 64] descriptor (never read)
    # select_kv: k out of range -> CONFIG before any device access
    rc = L.bsa_select_kv_blocks(ctypes.byref(g.c()), 1, 2, 64, t16, None, t16, 0, 0.9,
                                ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, None, ctypes.c_void_p(16), 1 << 30,
                                None)
    assert rc == 2 and b"k must be" in L.bsa_last_error()
    rc = L.bsa_select_kv_blocks(ctypes.byref(g.c()), 1, 2, 64, t16, None, t16, 3, 1.5,
                                ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, None, ctypes.c_void_p(16), 1 << 30,
                                None)
    assert rc == 2 and b"tau" in L.bsa_last_error()
    # attention with an unsupported block size
    g3 = bsa.Geometry(4, 8, 8, 1, 2, 2)
    rc = L.bsa_attn_fwd(ctypes.byref(g3.c()), 0.5, 1, 1, 64, t16, t16, t16, *([ctypes.c_void_p(256)] * 6),
                        ctypes.c_float(0.1), t16, ctypes.c_void_p(256), None, 0, None)
    assert rc == 1 and b"ct*ch*cw" in L.bsa_last_error()
    assert L.bsa_strerror(4) == b"unsupported device (needs sm_100a)"
    # selection variant: unknown KV mode -> CONFIG
    rc = L.bsa_select_kv_blocks_ex(ctypes.byref(g.c()), 1, 2, 64, t16, None, t16, 3,
                                   0.9, 7, ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, None,
                                   ctypes.c_void_p(16), 1 << 30, None)
    assert rc == 2 and b"KV mode" in L.bsa_last_error()
    # Ulysses reorders: heads not divisible by P -> CONFIG; d not a multiple of 8 / misaligned -> INVALID_SHAPE
    assert L.bsa_sp_relayout(0, 1, 16, 6, 128, 4, ctypes.c_void_p(256), ctypes.c_void_p(512), None) == 2
    assert b"split" in L.bsa_last_error()
    assert L.bsa_sp_relayout(0, 1, 16, 8, 12, 4, ctypes.c_void_p(256), ctypes.c_void_p(512), None) == 1
    assert L.bsa_sp_relayout(0, 1, 16, 8, 128, 4, ctypes.c_void_p(258), ctypes.c_void_p(512), None) == 1
    assert L.bsa_sp_relayout(9, 1, 16, 8, 128, 4, ctypes.c_void_p(256), ctypes.c_void_p(512), None) == 2


def test_strided_tensor_validation():
    """bsa_tensor checks (include/bsa.h): 16-byte aligned pointer, strides non-negative multiples of 8 elements,
    token stride >= d -> BSA_ERR_INVALID_SHAPE before any device access; a NULL required tensor -> SELECTION_MISMATCH."""
    L = bsa.lib()
    T = bsa._CTensor
    g = bsa.Geometry(4, 8, 8, 2, 4, 4)
    out = (ctypes.c_int32 * 16)()
    ok = T(256, 2 * 256 * 64, 256 * 64, 64)
    bshd = T(256, 256 * 2 * 64, 64, 2 * 64)  # a model's [B, L, Hh, d] layout: accepted
    bad = {"misaligned": T(258, 2 * 256 * 64, 256 * 64, 64), "stride_not_8": T(256, 2 * 256 * 64, 256 * 64, 68),
           "sl_lt_d": T(256, 2 * 256 * 64, 256 * 64, 32), "negative": T(256, -8, 256 * 64, 64)}
    for name, t in bad.items():
        rc = L.bsa_select_queries(ctypes.byref(g.c()), 0.5, 1, 2, 64, t, out, out, out, None, None, None)
        assert rc == 1, name
    rc = L.bsa_select_queries(ctypes.byref(g.c()), 0.5, 1, 2, 64, T(None, 0, 0, 0), out, out, out, None, None, None)
    assert rc == 3 and b"NULL" in L.bsa_last_error()
    # well-formed descriptors pass validation (the call then fails on the missing device, not on the shapes)
    for t in (ok, bshd):
        rc = L.bsa_select_queries(ctypes.byref(g.c()), 0.5, 1, 2, 64, t, out, out, out, None, None, None)
        assert rc not in (1, 2, 3), L.bsa_last_error()


def test_tensor_desc_strides():
    """The binding's descriptor of a [B, L, Hh, d] tensor viewed as [B, Hh, L, d] carries the model layout's strides."""
    import torch
    x = torch.empty(2, 100, 3, 64, dtype=torch.bfloat16)  # [B, L, Hh, d]
    v = x.transpose(1, 2)
    assert (v.stride(0), v.stride(1), v.stride(2), v.stride(3)) == (100 * 3 * 64, 64, 3 * 64, 1)
    qkv = torch.empty(1, 100, 3, 4, 64, dtype=torch.bfloat16)  # fused [B, L, 3, Hh, d] projection
    q = qkv[:, :, 0].transpose(1, 2)
    assert (q.stride(0), q.stride(1), q.stride(2)) == (100 * 3 * 4 * 64, 64, 3 * 4 * 64)


def test_workspace_sizes_monotone():
    g = bsa.Geometry(21, 30, 52)
    a = bsa.bsa_workspace_bytes(bsa.OP_SELECT_KV, g, 0.5, 1, 12, 128)
    b = bsa.bsa_workspace_bytes(bsa.OP_SELECT_KV, g, 0.5, 1, 24, 128)
    assert b > a > 624 * 624 * 8 * 12
    f = bsa.bsa_workspace_bytes(bsa.OP_ATTN_BWD, g, 0.5, 1, 12, 128)
    assert f >= 12 * 16380 * 128 * (2 + 2 + 4)


def test_host_quantile_matches_stdlib():
    """The library's own Eq.3 quantile (bsa_kv_quantile: Acklam + Halley on the host, reading C14) against
    statistics.NormalDist, an independent stdlib routine, at every k of the BASELINE geometries' N and at the
    clamped ends 1/(2N), 1 - 1/(2N)."""
    import statistics
    nd = statistics.NormalDist()
    for N in (8, 100, 624, 1440, 2640, 4096):
        ks = sorted(set([1, 2, N // 2, N - 1, N] + list(range(1, N + 1, max(1, N // 97)))))
        for k in ks:
            u = min(max(1 - k / N, 1 / (2 * N)), 1 - 1 / (2 * N))
            z = bsa.kv_quantile(k, N)
            ref = nd.inv_cdf(u)
            assert abs(z - ref) <= 1e-12 * max(1.0, abs(ref)), (k, N, z, ref)
    assert bsa.kv_quantile(312, 624) == 0.0  # u = 1/2 exactly
    with pytest.raises(bsa.BSAError):
        bsa.kv_quantile(0, 8)
    with pytest.raises(bsa.BSAError):
        bsa.kv_quantile(9, 8)


def test_resolve_k_rounding_rule():
    """Reading C6 behind the ABI (bsa_resolve_k): k = clamp(ceil(f N - 1e-9), 1, N), checked against exact rational
    arithmetic (fractions.Fraction) where plain float ceil goes wrong (0.07 * 100, 0.55 * 1440)."""
    from fractions import Fraction
    assert bsa.resolve_k(0.07, 100) == 7 and math.ceil(0.07 * 100) == 8
    assert bsa.resolve_k(0.55, 1440) == 792
    assert bsa.resolve_k(0.1, 624) == 63 and bsa.resolve_k(0.1, 1440) == 144 and bsa.resolve_k(0.1, 2640) == 264
    assert bsa.resolve_k(1e-9, 624) == 1 and bsa.resolve_k(1.0, 624) == 624
    for N in (8, 624, 1440, 2640):
        for num in range(1, 100):
            f = num / 100
            exact = -((-Fraction(num, 100) * N) // 1)  # ceil of the exact rational f N
            assert bsa.resolve_k(f, N) == max(1, min(N, exact)), (f, N)
    for bad in (0.0, -0.1, 1.5):
        with pytest.raises(bsa.BSAError):
            bsa.resolve_k(bad, 624)


def test_selection_rejects_more_than_4096_blocks():
    """N > 4096 is rejected by bsa_select_kv_blocks(_ex) with BSA_ERR_INVALID_SHAPE before any device access
    (the admission bitmaps and the attention kernels' lists are sized for N <= 4096; include/bsa.h)."""
    L = bsa.lib()
    g = bsa.Geometry(41, 45, 80, 2, 2, 4)  # 21 x 23 x 20 = 9660 blocks
    assert bsa.bsa_sizes(g, 0.5)[0] > 4096
    for fn in ("bsa_select_kv_blocks", "bsa_select_kv_blocks_ex"):
        t = bsa._CTensor(256, 2 * g.L * 64, g.L * 64, 64)
        args = [ctypes.byref(g.c()), 1, 2, 64, t, None, t, 3, 0.9]
        if fn.endswith("_ex"):
            args.append(0)
        args += [ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, None, ctypes.c_void_p(16), 1 << 40, None]
        rc = getattr(L, fn)(*args)
        assert rc == 1 and b"4096" in L.bsa_last_error(), fn


def test_bwd_path_switch_and_ds_capacity():
    """bsa_set_bwd_path / bsa_bwd_ds_capacity (include/bsa.h): the reduce path is the default (capacity -1);
    BSA_BWD_DS gives the dS capacity (a pair density of 1/8, at most 24 GiB of SR x 128-byte tiles) and a larger
    backward workspace; an unknown mode is BSA_ERR_CONFIG."""
    L = bsa.lib()
    g = bsa.Geometry(21, 30, 52)
    assert bsa.bwd_ds_capacity(g, 0.5, 1, 12, 128) == -1
    ws_reduce = bsa.bsa_workspace_bytes(bsa.OP_ATTN_BWD, g, 0.5, 1, 12, 128)
    try:
        bsa.set_bwd_path(bsa.BWD_DS)
        cap = bsa.bwd_ds_capacity(g, 0.5, 1, 12, 128)
        N = 624
        assert cap == 12 * N * ((N + 7) // 8)  # 1/8 density, far below the 24 GiB bound
        ws_ds = bsa.bsa_workspace_bytes(bsa.OP_ATTN_BWD, g, 0.5, 1, 12, 128)
        assert ws_ds >= ws_reduce + cap * 32 * 128 + 12 * N * N * 4  # dS tiles (SR = 32) + the pair-slot table
        big = bsa.Geometry(41, 45, 80)  # 147k: capped by the 24 GiB bound
        assert bsa.bwd_ds_capacity(big, 0.5, 1, 40, 128) == (24 << 30) // (32 * 128)
    finally:
        bsa.set_bwd_path(bsa.BWD_REDUCE)
    assert L.bsa_set_bwd_path(7) == 2 and b"backward path" in L.bsa_last_error()


def test_fwd_tiling_validation():
    """bsa_set_fwd_tiling (include/bsa.h): min slot rows in {0, 8, 16, 32, 64, 128} and a known order, else
    BSA_ERR_CONFIG with the setting unchanged; valid settings leave the forward workspace size unchanged."""
    L = bsa.lib()
    g = bsa.Geometry(21, 30, 52)
    ws = bsa.bsa_workspace_bytes(bsa.OP_ATTN_FWD, g, 0.5, 1, 12, 128)
    assert L.bsa_set_fwd_tiling(12, 0) == 2 and b"min slot" in L.bsa_last_error()
    assert L.bsa_set_fwd_tiling(8, 5) == 2 and b"order" in L.bsa_last_error()
    try:
        for m in (0, 8, 16, 32, 64, 128):
            bsa.set_fwd_tiling(m, bsa.FWD_LARGE_FIRST)
            assert bsa.bsa_workspace_bytes(bsa.OP_ATTN_FWD, g, 0.5, 1, 12, 128) == ws
    finally:
        bsa.set_fwd_tiling(0, bsa.FWD_SMALL_FIRST)


def test_sp_relayout_group_validation():
    """bsa_sp_relayout_group: a head group outside [0, Hh/P) or an unknown mode -> BSA_ERR_CONFIG, d not a
    multiple of 8 or a misaligned buffer -> BSA_ERR_INVALID_SHAPE, all before any device access."""
    L = bsa.lib()
    a, b = ctypes.c_void_p(256), ctypes.c_void_p(512)
    assert L.bsa_sp_relayout_group(0, 16, 8, 128, 2, 3, 2, a, b, None) == 2  # [3, 5) outside Hp = 4
    assert b"head group" in L.bsa_last_error()
    assert L.bsa_sp_relayout_group(0, 16, 8, 128, 2, 0, 0, a, b, None) == 2
    assert L.bsa_sp_relayout_group(5, 16, 8, 128, 2, 0, 2, a, b, None) == 2
    assert L.bsa_sp_relayout_group(0, 16, 8, 12, 2, 0, 2, a, b, None) == 1
    assert L.bsa_sp_relayout_group(1, 16, 8, 128, 2, 0, 2, ctypes.c_void_p(258), b, None) == 1
    assert L.bsa_sp_relayout_group(0, 16, 6, 128, 4, 0, 1, a, b, None) == 2  # heads do not split over P
