"""Seeded synthetic Q/K/V generators shared by the tests, the bench and the oracle harness.

This module holds NO arithmetic of the BSA method (no pooling, similarity, threshold,
admission or attention). It only turns (seed, shape) into bf16 tensors, so that the CUDA
path and the CPU oracle can be fed bit-identical inputs without sharing method code.

Recipes:

* splitmix64: state += 0x9E3779B97F4A7C15; z = state;
  z = (z ^ z>>30)*0xBF58476D1CE4E5B9; z = (z ^ z>>27)*0x94D049BB133111EB; z ^ z>>31.
  It is counter based: the i-th output (i = 0, 1, ...) of seed s is mix(s + (i+1)*gamma),
  which lets numpy/torch draw a whole stream in one vectorised call.
* uniform: top 24 bits of each draw * 2**-24, in [0, 1).
* gaussian: Box-Muller on consecutive uniform pairs (u, v): r = sqrt(-2 ln(1-u)),
  outputs r*cos(2*pi*v) then r*sin(2*pi*v); computed in fp64, rounded to fp32, then to
  bf16 with round-to-nearest-even.
* G_iid(seed): Q, K, V filled in that order from ONE gaussian stream, each [B, Hh, L, d]
  row-major.
* G_video(seed): per (b, h) a shared low-frequency field
  F(t,h,w) = (amp/sqrt(16)) * sum_{m<16} a_m * cos(2*pi*(ft_m t/T + fh_m h/H + fw_m w/W) + phi_m)
  with a_m ~ N(0, I_d), frequencies uniform in {0,1,2,3}^3 and phi_m ~ U[0, 2*pi);
  Q = F + eps_q, K = F + eps_k, V = eps_v with unit gaussian noise; amp = 1.2. It mimics the
  local redundancy the paper relies on.
"""

from __future__ import annotations

import numpy as np
import torch

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """Outputs offset .. offset+n-1 of the splitmix64 stream started at `seed` (uint64)."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform24(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """Top 24 bits of each draw as fp64 in [0,1) (exactly representable in fp32)."""
    return (splitmix64(seed, n, offset) >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)


def gaussian(seed: int, n: int) -> np.ndarray:
    """n standard normals (fp64) by Box-Muller on consecutive uniform pairs."""
    m = (n + 1) // 2
    u = uniform24(seed, 2 * m)
    u1 = 1.0 - u[0::2]
    u2 = u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    out = np.empty(2 * m, dtype=np.float64)
    out[0::2] = r * np.cos(2.0 * np.pi * u2)
    out[1::2] = r * np.sin(2.0 * np.pi * u2)
    return out[:n]


def to_bf16(x: np.ndarray, shape) -> torch.Tensor:
    """fp64 -> fp32 -> bf16 (round to nearest even), as a CPU torch tensor."""
    t = torch.from_numpy(np.ascontiguousarray(x.astype(np.float32))).reshape(shape)
    return t.to(torch.bfloat16)


def g_iid(seed: int, B: int, Hh: int, grid, d: int):
    """G_iid: Q, K, V ~ N(0,1) iid, bf16 [B, Hh, L, d] on CPU."""
    T, H, W = grid
    L = T * H * W
    n = B * Hh * L * d
    g = gaussian(seed, 3 * n)
    shape = (B, Hh, L, d)
    return to_bf16(g[:n], shape), to_bf16(g[n:2 * n], shape), to_bf16(g[2 * n:], shape)


def _field(seed: int, grid, d: int, amp: float, device, n_modes: int = 16) -> torch.Tensor:
    """Low-frequency field F for one (b, h): fp64 [L, d] on `device`."""
    T, H, W = grid
    u = uniform24(seed, 4 * n_modes)
    freq = np.floor(u[: 3 * n_modes] * 4.0).reshape(n_modes, 3)  # {0,1,2,3}
    phi = 2.0 * np.pi * u[3 * n_modes:]
    a = gaussian(seed ^ 0x5EED5EED, n_modes * d).reshape(n_modes, d)
    t = torch.arange(T, dtype=torch.float64, device=device).view(T, 1, 1) / T
    h = torch.arange(H, dtype=torch.float64, device=device).view(1, H, 1) / H
    w = torch.arange(W, dtype=torch.float64, device=device).view(1, 1, W) / W
    F = torch.zeros(T * H * W, d, dtype=torch.float64, device=device)
    for m in range(n_modes):
        ph = 2.0 * np.pi * (freq[m, 0] * t + freq[m, 1] * h + freq[m, 2] * w) + float(phi[m])
        F += torch.cos(ph).reshape(-1, 1) * torch.from_numpy(a[m]).to(device).view(1, d)
    return F * (amp / np.sqrt(n_modes))


def g_video(seed: int, B: int, Hh: int, grid, d: int, amp: float = 1.2, device="cpu"):
    """G_video: Q = F + eps_q, K = F + eps_k, V = eps_v; bf16 [B, Hh, L, d] on `device`.

    The noise is drawn from splitmix streams keyed by (seed, b, h, tensor); the field F by
    (seed, b, h). Deterministic and identical on CPU; on CUDA the fp64 transcendental
    results may differ in the last ulp before rounding to bf16 (perf inputs only).
    """
    T, H, W = grid
    L = T * H * W
    Q = torch.empty(B, Hh, L, d, dtype=torch.bfloat16, device=device)
    K = torch.empty_like(Q)
    V = torch.empty_like(Q)
    for b in range(B):
        for h in range(Hh):
            base = (seed * 1_000_003 + b * 4099 + h * 131) & 0xFFFFFFFFFFFF
            F = _field(base, grid, d, amp, device)
            for which, dst in ((1, Q), (2, K), (3, V)):
                eps = torch.from_numpy(gaussian(base * 8 + which, L * d)).to(device).view(L, d)
                x = eps if which == 3 else F + eps
                dst[b, h] = x.to(torch.float32).to(torch.bfloat16)
    return Q, K, V


def make_inputs(kind: str, seed: int, B: int, Hh: int, grid, d: int, device="cpu"):
    if kind == "iid":
        q, k, v = g_iid(seed, B, Hh, grid, d)
        return q.to(device), k.to(device), v.to(device)
    if kind == "video":
        return g_video(seed, B, Hh, grid, d, device=device)
    raise ValueError(kind)


def grad_output(seed: int, shape, device="cpu") -> torch.Tensor:
    """dO ~ N(0,1) bf16 from its own stream (seed offset so it never aliases Q/K/V)."""
    n = int(np.prod(shape))
    return to_bf16(gaussian(seed + 0x0D0D0D0D, n), shape).to(device)
