// ARCHIVED EXPERIMENT (not built; needs the tile_blk hook it once added to attn_fwd.cu). Result on
// wan1.3b_32k: union steps -9..16%, attn_fwd 1.02 -> 0.94 ms, but this one-CTA-per-head matching cost
// 0.33 ms (1.67 ms at 75k) -> not adopted (DESIGN.md §5 "Tried").
//
// tiles.cu — which query blocks share a forward tile.
//
// The forward (attn_fwd.cu) packs G = 128/SR query blocks into one 128-row tcgen05 tile and walks the
// UNION of their KV lists (P:210's q2k lists): a step on KV block j costs a full 128-row QK^T + PV even
// if one block of the tile admitted j. The union waste (sum over tiles of G |union| / sum of |lists|)
// is ~2.8 for G = 4 consecutive block ids on the 32k video workload, because Eq.3/Eq.4 pick fairly
// individual sets per query block. Grouping blocks with similar lists lowers it (to ~2.3 with the
// neighbourhood matching below), i.e. fewer forward steps for the same result.
//
// Method: hierarchical matching, log2(G) levels of pairing. At each level every unit (a block, then a
// pair, ...) proposes to the unmatched candidate with the largest Jaccard similarity of their admitted-
// KV bitmaps (ties -> lowest unit id); mutual proposals are matched; a few rounds, then leftovers are
// paired in ascending id order. Candidates are the units owning the 26 spatial neighbour blocks of a
// unit's members (similar lists are local in a smooth video latent; this keeps the cost O(N)).
// Deterministic for a given selection. The grouping only reorders work: the forward computes the same
// rows (up to fp32 summation order), which the parity tests check against the oracle.
#include "kernels.h"

namespace bsa {

// Row bitmaps of the q2k lists: one warp per (bh, query block).
__global__ void __launch_bounds__(256) k_q2k_bits(int N, int rows, const int* __restrict__ q2k_num,
                                                  const int* __restrict__ q2k_idx, uint32_t* __restrict__ bits) {
  __shared__ uint32_t s_b[8][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= rows) return;
  const int NW = (N + 31) >> 5;
  for (int w = lane; w < NW; w += 32) s_b[warp][w] = 0u;
  __syncwarp();
  const int num = q2k_num[row];
  const int* idx = q2k_idx + static_cast<size_t>(row) * N;
  for (int a = lane; a < num; a += 32) {
    const int j = idx[a];
    atomicOr(&s_b[warp][j >> 5], 1u << (j & 31));
  }
  __syncwarp();
  for (int w = lane; w < NW; w += 32) bits[static_cast<size_t>(row) * NW + w] = s_b[warp][w];
}

// Exclusive prefix sum of one int per thread over the CTA (1024 threads), plus the total.
__device__ __forceinline__ int cta_excl_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = s_warp[lane];
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    s_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  const int r = s_warp[warp] + incl - v;
  __syncthreads();
  return r;
}

__device__ __forceinline__ float jaccard(const uint32_t* a, const uint32_t* b, int NW) {
  int in = 0, un = 0;
  for (int w = 0; w < NW; ++w) {
    const uint32_t x = a[w], y = b[w];  // plain loads: the unit bitmaps are written by this kernel
    in += __popc(x & y);
    un += __popc(x | y);
  }
  return un ? static_cast<float>(in) / static_cast<float>(un) : 1.f;
}

struct TileScratch {  // per head
  uint32_t* ubA;  // [N][NW] unit bitmaps (levels >= 1), ping
  uint32_t* ubB;  // pong
  int* memA;      // [N + G] unit members (size per level), ping
  int* memB;      // pong
  int* owner;     // [N] block -> unit
  int* nid;       // [N] unit -> best candidate / new unit id
  int* partner;   // [N]
  int* list;      // [N] compacted unmatched units
};

constexpr int GROUP_ROUNDS = 4;
constexpr int GROUP_THREADS = 1024;

// One CTA per head.
__global__ void __launch_bounds__(GROUP_THREADS) k_group_tiles(Geo g, int G, const uint32_t* __restrict__ bits0,
                                                               TileScratch sc, int* __restrict__ tile_blk) {
  __shared__ int s_warp[32], s_total;
  const int bh = blockIdx.x, N = g.N, NW = (N + 31) >> 5;
  const size_t hb = static_cast<size_t>(bh);
  const uint32_t* b0 = bits0 + hb * N * NW;
  uint32_t* ub[2] = {sc.ubA + hb * N * NW, sc.ubB + hb * N * NW};
  int* mem[2] = {sc.memA + hb * (N + G), sc.memB + hb * (N + G)};
  int* owner = sc.owner + hb * N;
  int* nid = sc.nid + hb * N;
  int* partner = sc.partner + hb * N;
  int* list = sc.list + hb * N;
  const int ntiles = (N + G - 1) / G;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    owner[i] = i;
    mem[0][i] = i;
  }
  __syncthreads();
  int n = N, size = 1, cur = 0;
  const uint32_t* ubc = b0;  // bitmaps of the current level's units
  while (size < G) {
    for (int u = threadIdx.x; u < n; u += blockDim.x) partner[u] = -1;
    __syncthreads();
    for (int round = 0; round < GROUP_ROUNDS; ++round) {
      for (int u = threadIdx.x; u < n; u += blockDim.x) {
        int bv = -1;
        if (partner[u] < 0) {
          float bs = -1.f;
          for (int k = 0; k < size; ++k) {
            const int m = mem[cur][u * size + k];
            if (m < 0) continue;
            const int bt = m / (g.Nh * g.Nw), bhh = (m / g.Nw) % g.Nh, bw = m % g.Nw;
            for (int dt = -1; dt <= 1; ++dt)
              for (int dh = -1; dh <= 1; ++dh)
                for (int dw = -1; dw <= 1; ++dw) {
                  const int t = bt + dt, h = bhh + dh, w = bw + dw;
                  if (t < 0 || t >= g.Nt || h < 0 || h >= g.Nh || w < 0 || w >= g.Nw) continue;
                  const int v = owner[(t * g.Nh + h) * g.Nw + w];
                  if (v == u || partner[v] >= 0) continue;
                  const float s = jaccard(ubc + static_cast<size_t>(u) * NW, ubc + static_cast<size_t>(v) * NW, NW);
                  if (s > bs || (s == bs && v < bv)) { bs = s; bv = v; }
                }
          }
        }
        nid[u] = bv;
      }
      __syncthreads();
      for (int u = threadIdx.x; u < n; u += blockDim.x) {
        const int v = nid[u];
        if (partner[u] < 0 && v >= 0 && nid[v] == u) partner[u] = v;
      }
      __syncthreads();
    }
    // leftovers: pair in ascending unit id; an odd last one stays single (partner -2)
    int cnt = 0;
    for (int base = 0; base < n; base += blockDim.x) {
      const int u = base + threadIdx.x;
      const int f = (u < n && partner[u] < 0) ? 1 : 0;
      const int r = cta_excl_scan(f, s_warp, &s_total);
      if (f) list[cnt + r] = u;
      cnt += s_total;
      __syncthreads();
    }
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
      const int u = list[q];
      partner[u] = (q ^ 1) < cnt ? list[q ^ 1] : -2;
    }
    __syncthreads();
    // new units: one per leader (lower id of a pair, or a single), numbered in ascending leader id
    int nn = 0;
    for (int base = 0; base < n; base += blockDim.x) {
      const int u = base + threadIdx.x;
      const int f = (u < n && (partner[u] == -2 || u < partner[u])) ? 1 : 0;
      const int r = cta_excl_scan(f, s_warp, &s_total);
      if (f) {
        nid[u] = nn + r;
        if (partner[u] >= 0) nid[partner[u]] = nn + r;
      }
      nn += s_total;
      __syncthreads();
    }
    const int nxt = cur ^ 1, size2 = 2 * size;
    uint32_t* ubn = ub[nxt];
    for (int u = threadIdx.x; u < n; u += blockDim.x) {
      const int v = partner[u];
      if (!(v == -2 || u < v)) continue;
      const int t = nid[u];
      for (int k = 0; k < size; ++k) {
        mem[nxt][t * size2 + k] = mem[cur][u * size + k];
        mem[nxt][t * size2 + size + k] = v >= 0 ? mem[cur][v * size + k] : -1;
      }
      for (int w = 0; w < NW; ++w)
        ubn[static_cast<size_t>(t) * NW + w] =
            ubc[static_cast<size_t>(u) * NW + w] | (v >= 0 ? ubc[static_cast<size_t>(v) * NW + w] : 0u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) owner[i] = nid[owner[i]];
    __syncthreads();
    n = nn;
    size = size2;
    cur = nxt;
    ubc = ubn;
  }
  // tiles: unit t -> its (up to G) blocks
  int* out = tile_blk + hb * ntiles * G;
  for (int e = threadIdx.x; e < ntiles * G; e += blockDim.x) {
    const int t = e / G, k = e % G;
    out[e] = (t < n && k < size) ? mem[cur][t * size + k] : -1;
  }
}

size_t tile_scratch_bytes(int N, int G, size_t BH) {
  const size_t NW = (N + 31) / 32, ntiles = (N + G - 1) / G;
  auto a = [](size_t x) { return (x + 255) & ~size_t(255); };
  return a(BH * N * NW * 4) * 3 + a(BH * (N + G) * 4) * 2 + a(BH * N * 4) * 4 + a(BH * ntiles * G * 4);
}

cudaError_t launch_group_tiles(const Geo& g, int BH, int G, const int* q2k_num, const int* q2k_idx, void* scratch,
                               int* tile_blk_out[1], cudaStream_t st) {
  const size_t NW = (g.N + 31) / 32, ntiles = (g.N + G - 1) / G, N = g.N;
  auto a = [](size_t x) { return (x + 255) & ~size_t(255); };
  uint8_t* p = static_cast<uint8_t*>(scratch);
  uint32_t* bits = reinterpret_cast<uint32_t*>(p);
  p += a(BH * N * NW * 4);
  TileScratch sc;
  sc.ubA = reinterpret_cast<uint32_t*>(p);
  p += a(BH * N * NW * 4);
  sc.ubB = reinterpret_cast<uint32_t*>(p);
  p += a(BH * N * NW * 4);
  sc.memA = reinterpret_cast<int*>(p);
  p += a(BH * (N + G) * 4);
  sc.memB = reinterpret_cast<int*>(p);
  p += a(BH * (N + G) * 4);
  sc.owner = reinterpret_cast<int*>(p);
  p += a(BH * N * 4);
  sc.nid = reinterpret_cast<int*>(p);
  p += a(BH * N * 4);
  sc.partner = reinterpret_cast<int*>(p);
  p += a(BH * N * 4);
  sc.list = reinterpret_cast<int*>(p);
  p += a(BH * N * 4);
  int* tile_blk = reinterpret_cast<int*>(p);
  (void)ntiles;
  const int rows = g.N * BH;
  k_q2k_bits<<<(rows + 7) / 8, 256, 0, st>>>(g.N, rows, q2k_num, q2k_idx, bits);
  k_group_tiles<<<BH, GROUP_THREADS, 0, st>>>(g, G, bits, sc, tile_blk);
  tile_blk_out[0] = tile_blk;
  return cudaGetLastError();
}

}  // namespace bsa
