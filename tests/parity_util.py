"""Parity helpers: compare the CUDA path (through the C ABI) with the fp64 oracle.

Protocol (north_star; SURVEY.md §8(c) "GPU-vs-oracle parity protocol", reading C24):
 * selection (kept_tok, donor, q2k) must be bit-exact; a disagreement is tolerated only when the
   oracle's own decision margin is below 1e-6 (cosine gap, logit margin relative to
   max(|s|,|p|,sigma), or cumulative-mass margin relative to E) — such near-ties are counted and
   reported, anything else fails;
 * attention outputs and gradients X in {O, dQ, dK, dV} (bf16 in, fp32 accumulate, bf16 out): with the
   output scale s = max|X_ref| (reading C26), max|X_gpu - X_ref| / s <= 2e-2 and
   mean|X_gpu - X_ref| / s <= 2e-3 (the north_star tolerance); in addition the mean error must stay
   within 5e-3 of RMS(X_ref) (rounding the output to bf16 alone costs ~1.6e-3 of RMS), which catches
   a wrong minority of rows that the max-normalised mean would hide.
   When near-ties changed the selection, the oracle attention is re-run on the GPU's selection.

Every comparison is also recorded in RECORDS (per case: near-tie counts; per case and tensor: max/max,
mean/max, mean/RMS, max/RMS); conftest.py writes them to $BSA_PARITY_OUT at the end of the session, which is
how profiles/r02_parity.json is produced from a GPU run. The parity tests assert that the near-tie count is 0
(none has been observed; a non-zero count fails with the list instead of passing silently).
"""

from __future__ import annotations

import numpy as np
import torch

import oracle as orc

NEAR = 1e-6
MAX_TOL, MEAN_TOL, MEAN_RMS_TOL = 2e-2, 2e-3, 5e-3

RECORDS: list = []


def record(case, **kw):
    RECORDS.append(dict(case=case, **kw))


def compare_selection(g: orc.Geom, r, gpu_kept, gpu_donor, gpu_num, gpu_idx, oq, okv, case=None):
    """Returns a dict of near-tie counts (and the list of near-tie items under "items"); raises AssertionError on
    a disagreement outside the near-tie band. The counts are recorded under `case`."""
    kept = gpu_kept.cpu().numpy().reshape(oq["kept_tok"].shape)
    donor = gpu_donor.cpu().numpy().reshape(oq["donor"].shape)
    num = gpu_num.cpu().numpy().reshape(okv["q2k_num"].shape)
    idx = gpu_idx.cpu().numpy().reshape(okv["q2k_idx"].shape)
    BH, L = donor.shape
    N = num.shape[1]
    near = dict(kept=0, donor=0, q2k=0)
    items = []
    bad = []
    # kept sets per unit: compare kept flags per token
    kf_gpu = np.zeros((BH, L), bool)
    kf_ref = np.zeros((BH, L), bool)
    for bh in range(BH):
        kf_gpu[bh, kept[bh]] = True
        kf_ref[bh, oq["kept_tok"][bh]] = True
    diff = np.argwhere(kf_gpu != kf_ref)
    for bh, t in diff:
        if oq["unit_margin"][bh, t] < NEAR:
            near["kept"] += 1
            items.append(("kept", int(bh), int(t), float(oq["unit_margin"][bh, t])))
        else:
            bad.append(("kept", bh, t, oq["unit_margin"][bh, t]))
    if len(diff) == 0:
        assert np.array_equal(kept, oq["kept_tok"]), "kept_tok order differs"
    dd = np.argwhere(donor != oq["donor"])
    for bh, t in dd:
        if kf_gpu[bh, t] != kf_ref[bh, t] or oq["unit_margin"][bh, t] < NEAR:
            continue  # consequence of a kept-set near-tie in this unit
        if oq["donor_margin"][bh, t] < NEAR:
            near["donor"] += 1
            items.append(("donor", int(bh), int(t), float(oq["donor_margin"][bh, t])))
        else:
            bad.append(("donor", bh, t, oq["donor_margin"][bh, t]))
    for bh in range(BH):
        for i in range(N):
            a = idx[bh, i, :num[bh, i]]
            b = okv["q2k_idx"][bh, i, :okv["q2k_num"][bh, i]]
            if num[bh, i] == okv["q2k_num"][bh, i] and np.array_equal(a, b):
                continue
            m = min(okv["thr_margin"][bh, i], okv["mass_margin"][bh, i], okv["order_margin"][bh, i])
            if m < NEAR:
                near["q2k"] += 1
                items.append(("q2k", int(bh), int(i), float(m)))
            else:
                bad.append(("q2k", bh, i, m, a.tolist()[:8], b.tolist()[:8]))
    assert not bad, f"selection mismatches outside the near-tie band: {bad[:5]} (total {len(bad)})"
    # rows/tokens compared, for the record
    record(case, kind="selection", heads=int(BH), tokens=int(BH * L), q2k_rows=int(BH * N),
           admitted_blocks=int(num.sum()), near_kept=near["kept"], near_donor=near["donor"], near_q2k=near["q2k"],
           near_items=items[:20])
    near["items"] = items
    return near


def assert_no_near_ties(near, what=""):
    """The parity tests' bar: selection bit-exact with zero near-ties (SURVEY §8(c) protocol; C24 margins)."""
    n = near["kept"] + near["donor"] + near["q2k"]
    assert n == 0, f"{what}: {n} near-tie disagreements with the oracle: {near['items'][:10]}"


def rel_err(x_gpu: torch.Tensor, x_ref: np.ndarray):
    """(max|d|/max|ref|, mean|d|/max|ref|, mean|d|/rms(ref)) with d = gpu - ref."""
    a = x_gpu.detach().double().cpu().numpy().reshape(x_ref.shape)
    smax = float(np.abs(x_ref).max()) or 1.0
    srms = float(np.sqrt(np.mean(x_ref ** 2))) or 1.0
    d = np.abs(a - x_ref)
    return float(d.max() / smax), float(d.mean() / smax), float(d.mean() / srms)


def rel_err_all(x_gpu: torch.Tensor, x_ref: np.ndarray):
    a = x_gpu.detach().double().cpu().numpy().reshape(x_ref.shape)
    smax = float(np.abs(x_ref).max()) or 1.0
    srms = float(np.sqrt(np.mean(x_ref ** 2))) or 1.0
    d = np.abs(a - x_ref)
    return dict(max_over_max=float(d.max() / smax), mean_over_max=float(d.mean() / smax),
                mean_over_rms=float(d.mean() / srms), max_over_rms=float(d.max() / srms), ref_max=smax, ref_rms=srms)


def assert_close(name, x_gpu, x_ref, case=None):
    e = rel_err_all(x_gpu, x_ref)
    record(case, kind="tensor", tensor=name, **e)
    mx, mean, mean_rms = e["max_over_max"], e["mean_over_max"], e["mean_over_rms"]
    assert mx <= MAX_TOL and mean <= MEAN_TOL and mean_rms <= MEAN_RMS_TOL, \
        f"{name}: max/scale={mx:.3e} mean/scale={mean:.3e} mean/rms={mean_rms:.3e}"
    return mx, mean, mean_rms
