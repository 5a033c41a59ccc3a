// geom.cuh — 3D block / unit geometry for the BSA kernels (§3.1, §3.2.1).
// Blocks are row-major over (ceil(T/ct), ceil(H/ch), ceil(W/cw)); edge blocks are truncated
// (reading C1); tokens of a block are in ascending raster order, which is the order
// (lt, lh, lw) lexicographic, i.e. the order a TMA box (w fastest) lays them out in shared memory.
#pragma once
#include <cstdint>

namespace bsa {

struct Geo {
  int T, H, W;
  int ct, ch, cw;
  int ut, uh, uw;  // selection unit (window); equals the block dims when the caller passed 0
  int Nt, Nh, Nw, N;
  int L;
  int BT;  // nominal tokens per block ct*ch*cw
};

__host__ __device__ inline int cdiv_i(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline int min_i(int a, int b) { return a < b ? a : b; }
__host__ __device__ inline int max_i(int a, int b) { return a > b ? a : b; }

inline Geo make_geo(int T, int H, int W, int ct, int ch, int cw, int ut, int uh, int uw) {
  Geo g;
  g.T = T; g.H = H; g.W = W;
  g.ct = ct; g.ch = ch; g.cw = cw;
  g.ut = ut > 0 ? ut : ct; g.uh = uh > 0 ? uh : ch; g.uw = uw > 0 ? uw : cw;
  g.Nt = cdiv_i(T, ct); g.Nh = cdiv_i(H, ch); g.Nw = cdiv_i(W, cw);
  g.N = g.Nt * g.Nh * g.Nw;
  g.L = T * H * W;
  g.BT = ct * ch * cw;
  return g;
}

struct Box {
  int o[3];  // origin (t, h, w) of the block in the grid
  int e[3];  // actual extent
};

__host__ __device__ inline Box block_box(const Geo& g, int b) {
  Box x;
  int bt = b / (g.Nh * g.Nw), bh = (b / g.Nw) % g.Nh, bw = b % g.Nw;
  x.o[0] = bt * g.ct; x.o[1] = bh * g.ch; x.o[2] = bw * g.cw;
  x.e[0] = min_i(g.ct, g.T - x.o[0]);
  x.e[1] = min_i(g.ch, g.H - x.o[1]);
  x.e[2] = min_i(g.cw, g.W - x.o[2]);
  return x;
}

__host__ __device__ inline int box_size(const Box& x) { return x.e[0] * x.e[1] * x.e[2]; }

// Token of the i-th (ascending) element of a block.
__host__ __device__ inline int box_token(const Geo& g, const Box& x, int i) {
  int lw = i % x.e[2], lh = (i / x.e[2]) % x.e[1], lt = i / (x.e[2] * x.e[1]);
  return ((x.o[0] + lt) * g.H + (x.o[1] + lh)) * g.W + (x.o[2] + lw);
}

// Per-unit keep count clamp(ceil(r n - 1e-9), 1, n) (Eq.2 P:166 with the guarded rounding, C6).
__host__ __device__ inline int keep_count(double r, int n) {
  int m = static_cast<int>(ceil(r * static_cast<double>(n) - 1e-9));
  if (m < 1) m = 1;
  if (m > n) m = n;
  return m;
}

// Units (windows) of a block: grid ceil(e/u) per axis, truncated at the block edge (C8).
__host__ __device__ inline int unit_grid(const Geo& g, const Box& x, int* nu) {
  nu[0] = cdiv_i(x.e[0], g.ut); nu[1] = cdiv_i(x.e[1], g.uh); nu[2] = cdiv_i(x.e[2], g.uw);
  return nu[0] * nu[1] * nu[2];
}

// Kept queries of a block = sum over its units of keep_count(r, |unit|).
__host__ __device__ inline int block_kept(const Geo& g, const Box& x, double r) {
  int nu[3];
  unit_grid(g, x, nu);
  int k = 0;
  for (int a = 0; a < nu[0]; ++a) {
    int et = min_i(g.ut, x.e[0] - a * g.ut);
    for (int b = 0; b < nu[1]; ++b) {
      int eh = min_i(g.uh, x.e[1] - b * g.uh);
      for (int c = 0; c < nu[2]; ++c) {
        int ew = min_i(g.uw, x.e[2] - c * g.uw);
        k += keep_count(r, et * eh * ew);
      }
    }
  }
  return k;
}

}  // namespace bsa
