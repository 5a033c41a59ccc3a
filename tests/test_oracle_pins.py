"""Pins the CPU oracle to things other than itself (CPU only, `-m "not gpu"`).

Each test names the passage it pins. Independent references used: hand-derived worked examples
(tests/golden/worked_examples.json), closed forms, brute-force enumeration written here in numpy,
Python's statistics.NormalDist, torch.nn.functional.scaled_dot_product_attention and torch
autograd in float64 — none of them shares code with oracle/bsa_oracle.c.
"""

import itertools
import json
import math
import os
import statistics

import numpy as np
import pytest
import torch

import bsa_gen
import oracle as orc

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


# ----------------------------------------------------------------------------- generator
def test_splitmix64_golden():
    """SPEC.md S:50-51."""
    out = bsa_gen.splitmix64(0, 2)
    assert [hex(int(x)).upper().replace("0X", "0x") for x in out] == GOLD["splitmix64_seed0"]["outputs_hex"]


def test_gaussian_moments():
    g = bsa_gen.gaussian(7, 200_000)
    assert abs(g.mean()) < 0.01 and abs(g.std() - 1.0) < 0.01


# ----------------------------------------------------------------------------- geometry
def test_flatten_example():
    """P:105 n = tHW + hW + w."""
    f = GOLD["flatten"]
    assert orc.lib().or_flatten(f["t"], f["h"], f["w"], f["H"], f["W"]) == f["n"]


@pytest.mark.parametrize("grid,block", [((4, 8, 8), (2, 4, 4)), ((21, 30, 52), (4, 4, 4)), ((5, 7, 9), (2, 3, 4)),
                                        ((21, 45, 80), (4, 4, 4))])
def test_partition_is_a_partition(grid, block):
    """Every token in exactly one block; blocks in row-major order with ascending tokens (C1, C2)."""
    g = orc.Geom(*grid, *block)
    p = orc.partition(g, 1.0)
    tok = p["block_tok"]
    assert sorted(tok.tolist()) == list(range(g.L))
    T, H, W = grid
    for b in range(p["N"]):
        seg = tok[p["block_off"][b]:p["block_off"][b + 1]]
        assert np.all(np.diff(seg) > 0)
        t, h, w = seg // (H * W), (seg // W) % H, seg % W
        assert len(set((t // block[0]).tolist())) == 1 and len(set((h // block[1]).tolist())) == 1
        assert len(set((w // block[2]).tolist())) == 1
        e = p["block_ext"][b]
        assert len(seg) == e[0] * e[1] * e[2]
    # blocks ordered row-major by (bt, bh, bw)
    firsts = tok[p["block_off"][:-1]]
    bt, bh, bw = firsts // (H * W) // block[0], (firsts // W) % H // block[1], firsts % W // block[2]
    Nh, Nw = -(-H // block[1]), -(-W // block[2])
    assert np.array_equal((bt * Nh + bh) * Nw + bw, np.arange(p["N"]))


def test_geometry_32k_histogram_and_last_block():
    """E_geo (golden): ragged 32k grid."""
    e = GOLD["E_geo"]
    g = orc.Geom(*e["grid"], *e["block"])
    p = orc.partition(g, 0.5)
    assert p["N"] == e["N"]
    hist = {str(k): int(v) for k, v in zip(*np.unique(np.diff(p["block_off"]), return_counts=True))}
    assert hist == e["block_size_histogram"]
    b = e["last_block"]
    assert p["block_ext"][b].tolist() == e["last_block_extent"]
    assert p["block_tok"][p["block_off"][b]:p["block_off"][b + 1]].tolist() == e["last_block_tokens"]


def _unit_vectors(angles_deg):
    return np.array([[math.cos(math.radians(a)), math.sin(math.radians(a))] for a in angles_deg])


def test_worked_example_Eq_and_centre():
    """E_q: Eq.2 P:160-164 literal (keep the most dissimilar), centre offset 7 of a 2x2x2 unit."""
    e = GOLD["E_q"]
    g = orc.Geom(2, 2, 2, 2, 2, 2)
    Q = np.zeros((1, 8, 2))
    Q[0, :7] = _unit_vectors(e["angles_deg_offsets_0_to_6"])
    Q[0, e["centre_offset"]] = [1.0, 0.0]
    s = orc.select_queries(g, e["r"], Q)
    assert s["kept_tok"][0].tolist() == e["kept"]
    for t in e["pruned"]:
        assert s["donor"][0, t] == e["donor_of_pruned"]
    for t in e["kept"]:
        assert s["donor"][0, t] == t


def test_worked_example_last_block_centre():
    """E_geo: centre of the (1,2,4) edge block of the 32k grid is token 32758 (C3 on the actual extent)."""
    e = GOLD["E_geo"]
    g = orc.Geom(*e["grid"], *e["block"])
    Q = np.zeros((1, g.L, 2))
    Q[0, :, 0] = 1.0
    toks = e["last_block_tokens"]
    others = [t for t in toks if t != e["last_block_centre"]]
    Q[0, others] = _unit_vectors(GOLD["E_q"]["angles_deg_offsets_0_to_6"])
    Q[0, e["last_block_centre"]] = [1.0, 0.0]
    s = orc.select_queries(g, 0.5, Q)
    p = orc.partition(g, 0.5)
    b = e["last_block"]
    kept = s["kept_tok"][0, p["kept_off"][b]:p["kept_off"][b + 1]].tolist()
    assert kept == [others[i] for i in GOLD["E_q"]["kept"]]


def test_tie_rule_lower_index_first():
    """SPEC.md S:219 tie example: equal dissimilarity -> lower global index retained (C7)."""
    g = orc.Geom(1, 1, 4, 1, 1, 4)  # one unit of 4 tokens, centre local offset 2
    Q = np.array([[[1.0, 3.0], [1.0, -3.0], [1.0, 0.0], [1.0, 3.0]]])
    s = orc.select_queries(g, 0.5, Q)
    assert s["kept_tok"][0].tolist() == [0, 1]
    assert s["donor"][0].tolist() == [0, 1, 0, 0]  # 2: cos(c, q0) == cos(c, q1) -> lowest j; 3 == q0


def _brute_select(Qu, centre_local, m):
    """Brute force: among all m-subsets maximise sum(1 - cos) then take the lexicographically smallest."""
    c = Qu[centre_local]
    nc = np.linalg.norm(c)
    cos = np.array([1.0 if i == centre_local else (0.0 if nc == 0 or np.linalg.norm(q) == 0 else
                                                   float(c @ q) / (nc * np.linalg.norm(q))) for i, q in enumerate(Qu)])
    best, best_set = -1e300, None
    for sub in itertools.combinations(range(len(Qu)), m):  # lexicographic order
        v = sum(1.0 - cos[i] for i in sub)
        if v > best + 1e-12:
            best, best_set = v, sub
    return list(best_set)


@pytest.mark.parametrize("seed", range(4))
def test_query_selection_brute_force(seed):
    """Eq.2: kept set == brute-force argmax subset; donors == brute-force argmax cosine."""
    # units of <= 16 tokens keep the C(|u|, m) enumeration small
    g = orc.Geom(4, 8, 8, 2, 4, 4, 2, 2, 2) if seed % 2 else orc.Geom(4, 8, 8, 2, 2, 4)
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((1, g.L, 5))
    r = [0.5, 0.25, 0.75, 0.4][seed]
    s = orc.select_queries(g, r, Q)
    p = orc.partition(g, r)
    ut, uh, uw = g.unit
    kept_all = set(s["kept_tok"][0].tolist())
    for b in range(p["N"]):
        toks = p["block_tok"][p["block_off"][b]:p["block_off"][b + 1]]
        T, H, W = g.T, g.H, g.W
        t, h, w = toks // (H * W), (toks // W) % H, toks % W
        key = (t % g.ct) // ut * 100 + (h % g.ch) // uh * 10 + (w % g.cw) // uw
        for u in np.unique(key):
            ut_toks = toks[key == u]
            tt, hh, ww = ut_toks // (H * W), (ut_toks // W) % H, ut_toks % W
            et, eh, ew = tt.max() - tt.min() + 1, hh.max() - hh.min() + 1, ww.max() - ww.min() + 1
            centre = (tt.min() + et // 2) * H * W + (hh.min() + eh // 2) * W + (ww.min() + ew // 2)
            m = max(1, min(len(ut_toks), math.ceil(r * len(ut_toks) - 1e-9)))
            sub = _brute_select(Q[0, ut_toks], int(np.where(ut_toks == centre)[0][0]), m)
            want = sorted(ut_toks[sub].tolist())
            got = sorted(t_ for t_ in ut_toks.tolist() if t_ in kept_all)
            assert got == want
            for i in ut_toks:
                if i in want:
                    assert s["donor"][0, i] == i
                    continue
                qi = Q[0, i]
                cs = [float(qi @ Q[0, j]) / (np.linalg.norm(qi) * np.linalg.norm(Q[0, j])) for j in want]
                assert s["donor"][0, i] == want[int(np.argmax(cs))]


def test_query_selection_invariants():
    """Cardinality, nesting in r, scale invariance; r = 1 identity; 32 per (4,4,4) block at r=.5."""
    g = orc.Geom(8, 8, 8, 4, 4, 4)
    Q = bsa_gen.g_iid(3, 1, 1, (8, 8, 8), 16)[0].double().numpy()[0]
    p = orc.partition(g, 0.5)
    assert np.all(np.diff(p["kept_off"]) == 32)
    prev = set()
    for r in (0.1, 0.25, 0.5, 0.75, 1.0):
        s = orc.select_queries(g, r, Q[None])
        cur = set(s["kept_tok"][0].tolist())
        assert prev <= cur
        prev = cur
        s4 = orc.select_queries(g, r, 4.0 * Q[None])  # power-of-two scale: exact in fp64
        assert np.array_equal(s["kept_tok"], s4["kept_tok"]) and np.array_equal(s["donor"], s4["donor"])
    s = orc.select_queries(g, 1.0, Q[None])
    assert s["kept_tok"][0].tolist() == sorted(range(g.L), key=lambda t: t) or len(s["kept_tok"][0]) == g.L
    assert np.array_equal(s["donor"][0], np.arange(g.L))


def test_keep_count_rounding():
    """C6: plain ceil(0.07*100) = 8 is wrong; the guarded rule gives 7."""
    assert math.ceil(0.07 * 100) == 8
    assert orc.keep_count(0.07, 100) == 7
    assert orc.keep_count(0.5, 64) == 32 and orc.keep_count(0.5, 1) == 1 and orc.keep_count(1e-6, 5) == 1


# ----------------------------------------------------------------------------- pooling
def test_pooling_example_and_linearity():
    """P:136 average pooling; S:140 example [1,0],[3,2] -> [2,1]; constant -> constant; linearity."""
    e = GOLD["pool_example"]
    g = orc.Geom(1, 1, 2, 1, 1, 2)
    assert orc.pool(g, np.array([e["rows"]], float))[0, 0].tolist() == e["pooled"]
    g = orc.Geom(5, 7, 9, 2, 3, 4)
    rng = np.random.default_rng(0)
    X, Y = rng.standard_normal((2, 1, g.L, 3))
    assert np.allclose(orc.pool(g, np.full((1, g.L, 3), 2.5)), 2.5, atol=0, rtol=1e-15)
    assert np.allclose(orc.pool(g, 2 * X + 3 * Y), 2 * orc.pool(g, X) + 3 * orc.pool(g, Y), atol=1e-13)
    # brute mean over the block's tokens
    p = orc.partition(g, 1.0)
    P = orc.pool(g, X)
    for b in range(p["N"]):
        toks = p["block_tok"][p["block_off"][b]:p["block_off"][b + 1]]
        assert np.allclose(P[0, b], X[0, toks].mean(0), atol=1e-14)


# ----------------------------------------------------------------------------- quantile / Eq.3 / Eq.4
def test_quantile():
    """Eq.3 U = Phi^-1 (C14): values from statistics.NormalDist (independent), symmetry."""
    nd = statistics.NormalDist()
    assert abs(orc.normal_quantile(0.5)) < 1e-15
    assert abs(orc.normal_quantile(GOLD["quantile"]["u"]) - GOLD["quantile"]["z"]) < 2e-15
    for u in (1e-6, 0.01, 0.1, 0.3, 0.7, 0.9, 0.99, 1 - 1e-6, 1 / (2 * 624), 1 - 1 / (2 * 2640)):
        assert abs(orc.normal_quantile(u) - nd.inv_cdf(u)) < 1e-12 * max(1, abs(nd.inv_cdf(u)))
    for u in (2.0 ** -20, 1 / 1024, 0.125, 0.25, 0.375):  # dyadic: 1 - u is exact
        assert abs(orc.normal_quantile(u) + orc.normal_quantile(1 - u)) < 1e-14


def _kv_from_row(s, k, tau):
    n = len(s)
    Qc = np.ones((1, n, 1))
    Kc = np.asarray(s, float).reshape(1, n, 1)
    return orc.select_kv_from_pooled(Qc, Kc, k, tau)


def test_worked_example_E_kv():
    """E_kv (golden): Eq.3 threshold and Eq.4 admission on s = (2,1,0,-1)."""
    e = GOLD["E_kv"]
    for case in e["cases"]:
        for tau_s, S in case["tau"].items():
            out = _kv_from_row(e["s"], case["k"], float(tau_s))
            assert out["q2k_idx"][0, 0, :out["q2k_num"][0, 0]].tolist() == S, (case["k"], tau_s)
            if case["p"] is not None:
                assert abs(out["thresh"][0, 0] - case["p"]) < 1e-12


def test_S315_example():
    """probs (.5,.3,.15,.05), target .7 -> {0,1} (threshold off, k = n)."""
    e = GOLD["S315"]
    out = _kv_from_row(np.log(e["probs"]), 4, e["tau"])
    assert out["q2k_idx"][0, 0, :out["q2k_num"][0, 0]].tolist() == e["S"]


def test_threshold_special_cases():
    """k = n/2 -> p = mean; constant row -> p = mean; k = N bypass admits all at tau=1 (C15)."""
    rng = np.random.default_rng(1)
    s = rng.standard_normal(8)
    out = _kv_from_row(s, 4, 1.0)
    assert abs(out["thresh"][0, 0] - s.mean()) < 1e-12
    out = _kv_from_row(np.full(8, 0.3), 3, 1.0)
    assert abs(out["thresh"][0, 0] - 0.3) < 1e-15 and out["q2k_num"][0, 0] == 8
    out = _kv_from_row(s, 8, 1.0)
    assert out["q2k_num"][0, 0] == 8


def _brute_kv_row(s, k, tau):
    """Independent: candidates by Eq.3 with statistics.NormalDist, then exhaustive subset search:
    minimal cardinality reaching tau*E, then maximal mass, then lexicographic."""
    n = len(s)
    if k >= n:
        C = list(range(n))
    else:
        mu = sum(s) / n
        sig = math.sqrt(sum((x - mu) ** 2 for x in s) / n)
        u = min(max(1 - k / n, 1 / (2 * n)), 1 - 1 / (2 * n))
        p = mu + sig * statistics.NormalDist().inv_cdf(u)
        C = [j for j in range(n) if s[j] >= p] or [int(np.argmax(s))]
    if tau >= 1:
        return sorted(C)
    m = max(s[j] for j in C)
    e = {j: math.exp(s[j] - m) for j in C}
    E = sum(e.values())
    for size in range(1, len(C) + 1):
        cands = [sub for sub in itertools.combinations(sorted(C), size) if sum(e[j] for j in sub) >= tau * E]
        if cands:
            best = max(sum(e[j] for j in sub) for sub in cands)
            return list(min(sub for sub in cands if sum(e[j] for j in sub) >= best - 1e-15))
    return sorted(C)


@pytest.mark.parametrize("seed", range(6))
def test_kv_selection_brute_force_tiny(seed):
    """Tiny grid N=8 (BASELINE configs[0]): oracle q2k == exhaustive 2^|C| search for several (k, tau)."""
    g = orc.Geom(4, 8, 8, 2, 4, 4)
    kind = "video" if seed % 2 else "iid"
    Q, K, _ = bsa_gen.make_inputs(kind, seed, 1, 2, (4, 8, 8), 64)
    Qc, Kc = orc.pool(g, Q), orc.pool(g, K)
    for k in (1, 2, 4, 8):
        for tau in (0.5, 0.9, 1.0):
            out = orc.select_kv_from_pooled(Qc, Kc, k, tau)
            for bh in range(2):
                for i in range(8):
                    s = [float(Qc[bh, i] @ Kc[bh, j]) / 8.0 for j in range(8)]
                    want = _brute_kv_row(s, k, tau)
                    got = out["q2k_idx"][bh, i, :out["q2k_num"][bh, i]].tolist()
                    assert got == want, (k, tau, bh, i)


def test_admission_monotone_in_tau():
    """Eq.4: larger target never admits fewer blocks."""
    rng = np.random.default_rng(5)
    Qc, Kc = rng.standard_normal((2, 1, 40, 8))
    prev = None
    for tau in (0.3, 0.5, 0.7, 0.9, 0.95, 1.0):
        out = orc.select_kv_from_pooled(Qc, Kc, 12, tau)
        sets = [set(out["q2k_idx"][0, i, :out["q2k_num"][0, i]].tolist()) for i in range(40)]
        if prev:
            assert all(a <= b for a, b in zip(prev, sets))
        prev = sets


# ----------------------------------------------------------------------------- attention
def _selection(g, r, k, tau, Q, K):
    qs = orc.select_queries(g, r, Q)
    kv = orc.select_kv(g, Q, K, k, tau)
    return qs, kv


def _masked_sdpa(g, r, Q, K, V, qs, kv, scale):
    """Independent reference: torch SDPA (fp64) with a boolean token mask built from (kept, q2k), then the fill."""
    p = orc.partition(g, r)
    BH, L, d = Q.shape
    blk_of = np.empty(L, np.int64)
    for b in range(p["N"]):
        blk_of[p["block_tok"][p["block_off"][b]:p["block_off"][b + 1]]] = b
    out = np.zeros((BH, L, d))
    lse = np.zeros((BH, p["Lq"]))
    for bh in range(BH):
        kept = qs["kept_tok"][bh]
        adm = np.zeros((p["N"], p["N"]), bool)
        for i in range(p["N"]):
            adm[i, kv["q2k_idx"][bh, i, :kv["q2k_num"][bh, i]]] = True
        mask = adm[blk_of[kept]][:, blk_of]  # [Lq, L]
        q = torch.from_numpy(Q[bh, kept])
        kk, vv = torch.from_numpy(K[bh]), torch.from_numpy(V[bh])
        o = torch.nn.functional.scaled_dot_product_attention(q[None], kk[None], vv[None], attn_mask=torch.from_numpy(mask)[None],
                                                             scale=scale)[0]
        logits = (q @ kk.T) * scale
        logits[~torch.from_numpy(mask)] = -float("inf")
        lse[bh] = torch.logsumexp(logits, -1).numpy()
        out[bh, kept] = o.numpy()
        out[bh] = out[bh, qs["donor"][bh]]
    return out, lse


@pytest.mark.parametrize("kind,r,f,tau", [("iid", 0.5, 0.5, 0.9), ("video", 0.5, 1.0, 0.9), ("video", 0.25, 0.5, 0.95),
                                          ("iid", 1.0, 1.0, 1.0)])
def test_attention_forward_vs_sdpa(kind, r, f, tau):
    """Eq.5 P:194-197 + fill P:155: oracle == SDPA(fp64, boolean mask) + donor copy."""
    g = orc.Geom(4, 8, 8, 2, 4, 4)
    Q, K, V = (x.double().numpy().reshape(-1, 256, 64) for x in bsa_gen.make_inputs(kind, 11, 1, 2, (4, 8, 8), 64))
    N = 8
    k = orc.resolve_k(f, N)
    qs, kv = _selection(g, r, k, tau, Q, K)
    scale = 1 / 8.0
    O, lse = orc.attn_fwd(g, r, Q, K, V, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], scale)
    Oref, lseref = _masked_sdpa(g, r, Q, K, V, qs, kv, scale)
    assert np.max(np.abs(O - Oref)) < 1e-12
    assert np.max(np.abs(lse - lseref)) < 1e-12
    if r == 1.0 and k == N and tau == 1.0:  # dense equivalence
        dense = torch.nn.functional.scaled_dot_product_attention(torch.from_numpy(Q), torch.from_numpy(K),
                                                                 torch.from_numpy(V), scale=scale).numpy()
        assert np.max(np.abs(O - dense)) < 1e-12
    # rows from sampled API agree
    rows = np.arange(0, 2 * qs["kept_tok"].shape[1], 7)
    Os, ls = orc.attn_fwd_rows(g, r, Q, K, V, qs["kept_tok"], kv["q2k_num"], kv["q2k_idx"], scale, rows)
    Lq = qs["kept_tok"].shape[1]
    for n, rw in enumerate(rows):
        assert np.allclose(Os[n], O[rw // Lq, qs["kept_tok"][rw // Lq, rw % Lq]], atol=0, rtol=0)
        assert ls[n] == lse[rw // Lq, rw % Lq]


def test_attention_special_cases():
    """L=1 -> O = V; identical K rows -> mean of V; linear in V; convex hull."""
    g = orc.Geom(1, 1, 1, 1, 1, 1)
    one = lambda x: np.array(x, float).reshape(1, 1, -1)
    O, lse = orc.attn_fwd(g, 1.0, one([0.3, -1]), one([2, 1]), one([5, 7]), [[0]], [[0]], [[1]], [[0]], 0.7)
    assert O[0, 0].tolist() == [5.0, 7.0]
    g = orc.Geom(2, 4, 4, 2, 2, 2)
    rng = np.random.default_rng(2)
    Q = rng.standard_normal((1, 32, 4))
    K = np.tile(rng.standard_normal((1, 1, 4)), (1, 32, 1))
    V = rng.standard_normal((1, 32, 4))
    qs = orc.select_queries(g, 1.0, Q)
    N = 4
    num = np.full((1, N), N, np.int32)
    idx = np.tile(np.arange(N, dtype=np.int32), (1, N, 1))
    O, _ = orc.attn_fwd(g, 1.0, Q, K, V, qs["kept_tok"], qs["donor"], num, idx, 0.5)
    assert np.allclose(O[0], V[0].mean(0), atol=1e-14)
    V2 = rng.standard_normal((1, 32, 4))
    K = rng.standard_normal((1, 32, 4))
    O1, _ = orc.attn_fwd(g, 1.0, Q, K, V, qs["kept_tok"], qs["donor"], num, idx, 0.5)
    O2, _ = orc.attn_fwd(g, 1.0, Q, K, V2, qs["kept_tok"], qs["donor"], num, idx, 0.5)
    O3, _ = orc.attn_fwd(g, 1.0, Q, K, 2 * V - 3 * V2, qs["kept_tok"], qs["donor"], num, idx, 0.5)
    assert np.allclose(O3, 2 * O1 - 3 * O2, atol=1e-13)
    assert np.all(O1 <= V.max(1, keepdims=True) + 1e-14) and np.all(O1 >= V.min(1, keepdims=True) - 1e-14)


def test_key_shift_invariance():
    """K -> K + 1 c^T shifts every pooled score row by a constant: selection and O unchanged."""
    g = orc.Geom(4, 8, 8, 2, 4, 4)
    Q, K, V = (x.double().numpy().reshape(-1, 256, 64) for x in bsa_gen.make_inputs("video", 4, 1, 2, (4, 8, 8), 64))
    c = np.random.default_rng(9).standard_normal(64) * 0.25
    qs, kv = _selection(g, 0.5, 4, 0.9, Q, K)
    qs2, kv2 = _selection(g, 0.5, 4, 0.9, Q, K + c)
    assert np.array_equal(kv["q2k_idx"], kv2["q2k_idx"])
    O, _ = orc.attn_fwd(g, 0.5, Q, K, V, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], 0.125)
    O2, _ = orc.attn_fwd(g, 0.5, Q, K + c, V, qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], 0.125)
    assert np.max(np.abs(O - O2)) < 1e-12


# ----------------------------------------------------------------------------- backward
def _torch_sparse_loss_grads(g, r, Q, K, V, dO, qs, kv, scale):
    """Independent: torch autograd (fp64) through masked SDPA + donor gather; loss = <O, dO>."""
    p = orc.partition(g, r)
    BH, L, d = Q.shape
    blk_of = np.empty(L, np.int64)
    for b in range(p["N"]):
        blk_of[p["block_tok"][p["block_off"][b]:p["block_off"][b + 1]]] = b
    Qt, Kt, Vt = (torch.tensor(x, requires_grad=True) for x in (Q, K, V))
    loss = 0
    for bh in range(BH):
        kept = torch.from_numpy(qs["kept_tok"][bh].astype(np.int64))
        adm = np.zeros((p["N"], p["N"]), bool)
        for i in range(p["N"]):
            adm[i, kv["q2k_idx"][bh, i, :kv["q2k_num"][bh, i]]] = True
        mask = torch.from_numpy(adm[blk_of[qs["kept_tok"][bh]]][:, blk_of])
        Os = torch.nn.functional.scaled_dot_product_attention(Qt[bh, kept][None], Kt[bh][None], Vt[bh][None],
                                                              attn_mask=mask[None], scale=scale)[0]
        pos = torch.empty(L, dtype=torch.long)
        pos[kept] = torch.arange(len(kept))
        O = Os[pos[torch.from_numpy(qs["donor"][bh].astype(np.int64))]]
        loss = loss + (O * torch.from_numpy(dO[bh])).sum()
    loss.backward()
    return Qt.grad.numpy(), Kt.grad.numpy(), Vt.grad.numpy()


@pytest.mark.parametrize("kind,r,f,tau", [("video", 0.5, 0.5, 0.9), ("iid", 0.25, 1.0, 0.8), ("iid", 1.0, 1.0, 1.0)])
def test_attention_backward(kind, r, f, tau):
    """a8 (C10): oracle gradients == torch fp64 autograd; sum dK = 0; sum dV = sum dO; dQ[pruned] = 0."""
    g = orc.Geom(4, 8, 8, 2, 4, 4)
    Q, K, V = (x.double().numpy().reshape(-1, 256, 64) for x in bsa_gen.make_inputs(kind, 21, 1, 2, (4, 8, 8), 64))
    dO = bsa_gen.grad_output(21, (2, 256, 64)).double().numpy()
    qs, kv = _selection(g, r, orc.resolve_k(f, 8), tau, Q, K)
    args = (qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], 0.125)
    dQ, dK, dV = orc.attn_bwd(g, r, Q, K, V, dO, *args)
    tQ, tK, tV = _torch_sparse_loss_grads(g, r, Q, K, V, dO, qs, kv, 0.125)
    assert np.max(np.abs(dQ - tQ)) < 1e-11 and np.max(np.abs(dK - tK)) < 1e-11 and np.max(np.abs(dV - tV)) < 1e-11
    assert np.max(np.abs(dK.sum(1))) < 1e-11
    assert np.max(np.abs(dV.sum(1) - dO.sum(1))) < 1e-11
    for bh in range(2):
        pruned = np.setdiff1d(np.arange(256), qs["kept_tok"][bh])
        assert np.all(dQ[bh, pruned] == 0)


def test_attention_backward_finite_differences():
    """Central differences of <O, dO> with the selection frozen (C10)."""
    g = orc.Geom(2, 4, 4, 2, 2, 2)
    rng = np.random.default_rng(3)
    Q, K, V, dO = rng.standard_normal((4, 1, 32, 8))
    qs, kv = _selection(g, 0.5, 2, 0.9, Q, K)
    args = (qs["kept_tok"], qs["donor"], kv["q2k_num"], kv["q2k_idx"], 0.35)
    dQ, dK, dV = orc.attn_bwd(g, 0.5, Q, K, V, dO, *args)

    def loss(Q_, K_, V_):
        O, _ = orc.attn_fwd(g, 0.5, Q_, K_, V_, *args)
        return float((O * dO).sum())

    h = 1e-6
    for X, G, which in ((Q, dQ, 0), (K, dK, 1), (V, dV, 2)):
        for _ in range(6):
            t, c = rng.integers(32), rng.integers(8)
            Xp, Xm = X.copy(), X.copy()
            Xp[0, t, c] += h
            Xm[0, t, c] -= h
            a = [Q, K, V]
            a[which] = Xp
            lp = loss(*a)
            a[which] = Xm
            lm = loss(*a)
            assert abs((lp - lm) / (2 * h) - G[0, t, c]) < 1e-7


def test_sparsity_composition():
    """Table 2: 1 - (1-0.5)(1-0.86) = 0.93."""
    e = GOLD["sparsity_composition"]
    assert abs(1 - (1 - e["s_q"]) * (1 - e["s_kv"]) - e["combined"]) < 1e-12


# ---------------------------------------------------------------- unified_prob variant (C28)
def _unified_reference_row(s, k):
    """Independent statement of the unified_prob rule on one row (numpy softmax, statistics.NormalDist)."""
    import statistics
    N = len(s)
    e = np.exp(s - s.max())
    prob = e / e.sum()
    mu, sigma = prob.mean(), prob.std()
    u = min(max(1 - k / N, 1 / (2 * N)), 1 - 1 / (2 * N))
    p = min(1.0, mu + sigma * statistics.NormalDist().inv_cdf(u))
    return prob, max(p, np.finfo(float).tiny)


def test_unified_uniform_row_admits_one_block():
    # all scores equal: prob = 1/N, sigma = 0, p = 1/N -> exactly one block, the lowest id (C7)
    N, d = 6, 4
    Qc = np.ones((1, N, d))
    Kc = np.tile(np.arange(1.0, d + 1.0), (1, N, 1))
    out = orc.select_kv_unified_from_pooled(Qc, Kc, k=2)
    assert (out["q2k_num"][0] == 1).all() and (out["q2k_idx"][0, :, 0] == 0).all()


@pytest.mark.parametrize("seed", range(6))
def test_unified_brute_force_and_monotone(seed):
    rng = np.random.default_rng(seed)
    N, d = 7, 4
    Qc = rng.normal(size=(1, N, d)) * 2.0
    Kc = rng.normal(size=(1, N, d)) * 2.0
    prev = None
    for k in range(1, N + 1):
        out = orc.select_kv_unified_from_pooled(Qc, Kc, k)
        for i in range(N):
            s = Qc[0, i] @ Kc[0].T / np.sqrt(d)
            prob, p = _unified_reference_row(s, k)
            assert abs(out["thresh"][0, i] - p) <= 1e-12
            got = set(out["q2k_idx"][0, i, :out["q2k_num"][0, i]].tolist())
            # brute force: minimum cardinality reaching mass p; among those the largest mass, then lowest ids
            best = None
            for m in range(1, N + 1):
                cands = [c for c in itertools.combinations(range(N), m) if prob[list(c)].sum() >= p * (1 - 1e-12)]
                if cands:
                    best = max(cands, key=lambda c: (prob[list(c)].sum(), [-x for x in c]))
                    break
            assert got == set(best), (k, i, got, best)
        num = out["q2k_num"][0]
        if prev is not None:  # larger k: smaller quantile, smaller p, never more blocks (C28)
            assert (num <= prev).all()
        prev = num


# ----------------------------------------------------------------------------- near-tie margins (C24)
# The GPU-vs-oracle protocol excuses a selection disagreement only when the oracle's own decision margin is
# below 1e-6. These pins tie the margins to closed forms on the worked examples, so a margin
# that came out ~0 (turning real mismatches into "near-ties") or too large fails here.
def _deg_cos(a):
    return math.cos(math.radians(a))


def test_query_margins_worked_example_E_q():
    """E_q (Eq.2): unit gap at the keep cut = c_(5th) - c_(4th) of the ascending cosines =
    cos 45 - cos 60 = (sqrt 2 - 1)/2 for every token of the unit; donor margin of a pruned token p = best - second
    best of cos(theta_p - theta_j) over the kept j (angles 90, 60, 170, 120); kept tokens: no margin (DBL_MAX)."""
    e = GOLD["E_q"]
    g = orc.Geom(2, 2, 2, 2, 2, 2)
    ang = e["angles_deg_offsets_0_to_6"] + [0.0]  # offset 7 = the centre, at 0 degrees
    Q = _unit_vectors(ang)[None]
    s = orc.select_queries(g, e["r"], Q)
    gap = (math.sqrt(2.0) - 1.0) / 2.0
    assert np.allclose(s["unit_margin"][0], gap, rtol=0, atol=1e-12)
    kept_angles = [ang[t] for t in e["kept"]]
    for t in e["pruned"]:
        c = sorted((_deg_cos(ang[t] - a) for a in kept_angles), reverse=True)
        assert abs(s["donor_margin"][0, t] - (c[0] - c[1])) < 1e-12, t
    for t in e["kept"]:
        assert s["donor_margin"][0, t] > 1e300
    # closed forms spelled out: 10 deg -> cos 50 - cos 80, 30 -> cos 30 - cos 60, 45 -> cos 15 - cos 45, centre -> cos 60
    assert abs(s["donor_margin"][0, 1] - (_deg_cos(50) - _deg_cos(80))) < 1e-12
    assert abs(s["donor_margin"][0, 7] - 0.5) < 1e-12


def test_query_margins_vanish_on_exact_ties():
    """An exact cosine tie at the keep cut (S:219's example) has unit margin 0, and a pruned token equidistant
    from two kept tokens has donor margin 0: both would be counted as near-ties, never as mismatches."""
    g = orc.Geom(1, 1, 4, 1, 1, 4)  # centre local offset 2
    Q = np.array([[[1.0, 3.0], [1.0, -3.0], [1.0, 0.0], [1.0, 3.0]]])
    s = orc.select_queries(g, 0.5, Q)
    # ascending cosines: c0 = c1 = c3 < c2 = 1; the cut between the 2nd and 3rd is a tie
    assert s["unit_margin"][0].tolist() == [0.0] * 4
    assert s["donor_margin"][0, 2] == 0.0  # cos(q2, q0) == cos(q2, q1)
    assert s["donor_margin"][0, 3] > 0.5  # q3 == q0: cos 1 vs cos(q0, q1) = -0.8


def _kv_margins(k, tau):
    out = _kv_from_row(GOLD["E_kv"]["s"], k, tau)
    return out["thr_margin"][0, 0], out["mass_margin"][0, 0], out["order_margin"][0, 0]


def test_kv_margins_worked_example_E_kv():
    """E_kv (Eq.3, Eq.4) on s = (2,1,0,-1), sigma = sqrt(5)/2, p = 1/2 + sigma z_k with z from
    statistics.NormalDist (independent): thr margin = min_j |s_j - p| / max(|s_j|, |p|, sigma); mass margin = the
    smaller distance of the cumulative exp mass to tau E on either side of the cut, / E; order margin =
    (s_(l) - s_(l+1)) / max(sigma, |s_(l+1)|) between the last admitted and the first rejected candidate."""
    s = np.array(GOLD["E_kv"]["s"], float)
    sig = math.sqrt(5.0) / 2.0
    nd = statistics.NormalDist()
    BIG = 1e300
    for k in (1, 2, 3):
        p = 0.5 + sig * nd.inv_cdf(1 - k / 4)
        want = min(abs(sj - p) / max(abs(sj), abs(p), sig) for sj in s)
        assert abs(_kv_margins(k, 0.9)[0] - want) < 1e-12, k
    assert _kv_margins(4, 0.9)[0] > BIG  # k = N: no threshold (C15)
    # closed forms: k = 2 -> p = 1/2, margin 1/(2 sigma) = 1/sqrt 5; k = 1 -> (p - 1)/p
    assert abs(_kv_margins(2, 0.9)[0] - 1 / math.sqrt(5)) < 1e-12
    e = [math.exp(-t) for t in range(4)]  # exp(s - max) in sorted order
    cases = [  # (k, tau, admitted l, candidates)
        (1, 0.7, 1, 1), (1, 0.9, 1, 1), (2, 0.7, 1, 2), (2, 0.9, 2, 2), (3, 0.7, 2, 3), (3, 0.9, 2, 3),
        (4, 0.7, 2, 4), (4, 0.9, 3, 4)]
    for k, tau, ell, nc in cases:
        E = sum(e[:nc])
        cum, prev = sum(e[:ell]), sum(e[:ell - 1])
        mass = abs(cum - tau * E) / E if ell == 1 else min(abs(cum - tau * E), abs(prev - tau * E)) / E
        order = (s[ell - 1] - s[ell]) / max(sig, abs(s[ell])) if ell < nc else None
        thr, mm, om = _kv_margins(k, tau)
        assert abs(mm - mass) < 1e-12, (k, tau, mm, mass)
        if order is None:
            assert om > BIG
        else:
            assert abs(om - order) < 1e-12, (k, tau)
    # tau = 1: the whole candidate set, no mass cut (C18)
    assert _kv_margins(3, 1.0)[1] > BIG and _kv_margins(3, 1.0)[2] > BIG


def test_kv_margins_vanish_on_exact_ties():
    """A score exactly at the threshold p has thr margin 0; two candidates with equal score at the admission cut
    have order margin 0; a cumulative mass exactly at tau E has mass margin 0."""
    # s = (1, -1): mu = 0, k = N/2 -> p = mu = 0 ... make a score sit exactly on p: s = (1, 0, -1), k with z = 0
    # needs k/N = 1/2; use N = 4: s = (1, 0, 0, -1), k = 2 -> p = 0 = s_1 = s_2
    out = _kv_from_row([1.0, 0.0, 0.0, -1.0], 2, 0.9)
    assert out["thr_margin"][0, 0] == 0.0
    # equal scores at the cut: s = (1, 1), k = N (all candidates), tau = 0.5: l = 1, order margin 0
    out = _kv_from_row([1.0, 1.0], 2, 0.5)
    assert out["q2k_num"][0, 0] == 1 and out["order_margin"][0, 0] == 0.0
    assert out["mass_margin"][0, 0] == 0.0  # cum = 1 = 0.5 * 2 exactly
