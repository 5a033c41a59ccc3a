"""C-ABI library checks that need no GPU (`-m "not gpu"`): libbsa.so loads, exports every symbol
include/bsa.h declares, and its host-only logic (sizes, workspace sizing, validation) is right."""

import ctypes
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
    return sorted(set(re.findall(r"\b(bsa_[a-z_0-9]+)\s*\(", text)))


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
    # select_kv: k out of range -> CONFIG before any device access
    rc = L.bsa_select_kv_blocks(ctypes.byref(g.c()), 1, 2, 64, ctypes.c_void_p(16), None, ctypes.c_void_p(16), 0, 0.9,
                                ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, None, ctypes.c_void_p(16), 1 << 30,
                                None)
    assert rc == 2 and b"k must be" in L.bsa_last_error()
    rc = L.bsa_select_kv_blocks(ctypes.byref(g.c()), 1, 2, 64, ctypes.c_void_p(16), None, ctypes.c_void_p(16), 3, 1.5,
                                ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, None, ctypes.c_void_p(16), 1 << 30,
                                None)
    assert rc == 2 and b"tau" in L.bsa_last_error()
    # attention with an unsupported block size
    g3 = bsa.Geometry(4, 8, 8, 1, 2, 2)
    rc = L.bsa_attn_fwd(ctypes.byref(g3.c()), 0.5, 1, 1, 64, *([ctypes.c_void_p(256)] * 9), ctypes.c_float(0.1),
                        ctypes.c_void_p(256), ctypes.c_void_p(256), None, 0, None)
    assert rc == 1 and b"ct*ch*cw" in L.bsa_last_error()
    assert L.bsa_strerror(4) == b"unsupported device (needs sm_100a)"
    # selection variant: unknown KV mode -> CONFIG
    rc = L.bsa_select_kv_blocks_ex(ctypes.byref(g.c()), 1, 2, 64, ctypes.c_void_p(16), None, ctypes.c_void_p(16), 3,
                                   0.9, 7, ctypes.c_void_p(16), ctypes.c_void_p(16), None, None, None,
                                   ctypes.c_void_p(16), 1 << 30, None)
    assert rc == 2 and b"KV mode" in L.bsa_last_error()
    # Ulysses reorders: heads not divisible by P -> CONFIG; d not a multiple of 8 / misaligned -> INVALID_SHAPE
    assert L.bsa_sp_relayout(0, 1, 16, 6, 128, 4, ctypes.c_void_p(256), ctypes.c_void_p(512), None) == 2
    assert b"split" in L.bsa_last_error()
    assert L.bsa_sp_relayout(0, 1, 16, 8, 12, 4, ctypes.c_void_p(256), ctypes.c_void_p(512), None) == 1
    assert L.bsa_sp_relayout(0, 1, 16, 8, 128, 4, ctypes.c_void_p(258), ctypes.c_void_p(512), None) == 1
    assert L.bsa_sp_relayout(9, 1, 16, 8, 128, 4, ctypes.c_void_p(256), ctypes.c_void_p(512), None) == 2


def test_workspace_sizes_monotone():
    g = bsa.Geometry(21, 30, 52)
    a = bsa.bsa_workspace_bytes(bsa.OP_SELECT_KV, g, 0.5, 1, 12, 128)
    b = bsa.bsa_workspace_bytes(bsa.OP_SELECT_KV, g, 0.5, 1, 24, 128)
    assert b > a > 624 * 624 * 8 * 12
    f = bsa.bsa_workspace_bytes(bsa.OP_ATTN_BWD, g, 0.5, 1, 12, 128)
    assert f >= 12 * 16380 * 128 * (2 + 2 + 4)


def test_host_quantile_matches_stdlib():
    """The library's host Phi^-1 (Acklam + Halley) agrees with statistics.NormalDist; exercised
    through bsa_select_kv_blocks' thresholds on the GPU, checked here via a tiny C shim-free path:
    the oracle's bisection and the stdlib agree (pinned in test_oracle_pins), so we compare the
    threshold the GPU reports in the gpu tests. Here: stdlib vs oracle at the BASELINE k fractions."""
    import statistics
    for N in (8, 624, 1440, 2640):
        for f in (0.1, 0.5, 0.9):
            k = bsa.resolve_k(f, N)
            if k >= N:
                continue
            u = 1 - k / N
            assert abs(orc.normal_quantile(u) - statistics.NormalDist().inv_cdf(u)) < 1e-12
