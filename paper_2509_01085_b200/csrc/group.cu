// group.cu — which query blocks share a forward tile (DESIGN.md §5 "Forward tiles").
//
// The forward packs G = 128 / SR query blocks into one 128-row MMA tile and walks the UNION of their admitted
// KV blocks (P:210 lists); rows whose block did not admit a step's KV block are masked, so the tensor work of
// a tile is |union| steps. Consecutive blocks overlap little (union / admitted ~ 2.8 at 32k), so the tiles
// are built from blocks with similar lists instead: a hierarchical mutual-best matching on the Jaccard
// similarity of the admission sets (level 1 pairs blocks, level 2 pairs the pairs, ... up to G members),
// ~21% fewer union steps at 32k. It is a pure scheduling choice: every row still attends exactly its own
// block's list, so the result is the same up to fp32 summation order.
//
//   k_group_bits   admission bitmap of every (b,h, query block) from its q2k list
//   k_group_cand   per block: its 16 most similar blocks (approximate top-16 of the Jaccard index)
//   k_group_match  per head, one CTA: level-wise mutual-best matching over the candidates, then the tile
//                  order perm[bh][0..N) (tile t = perm[t G .. t G + G))
#include "kernels.h"

namespace bsa {

constexpr int GRP_CAND = 8;     // candidates per block (level 1)
constexpr int GRP_ROUNDS = 4;   // mutual-best rounds per level

// one warp per row: bits[row][w] (NW words) of the admitted KV blocks
__global__ void __launch_bounds__(256) k_group_bits(int N, int rows, const int* __restrict__ q2k_num,
                                                    const int* __restrict__ q2k_idx, uint32_t* __restrict__ bits) {
  __shared__ uint32_t sb[8][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= rows) return;
  const int NW = (N + 31) >> 5;
  for (int w = lane; w < NW; w += 32) sb[warp][w] = 0u;
  __syncwarp();
  const int num = q2k_num[row];
  const int* idx = q2k_idx + static_cast<size_t>(row) * N;
  for (int t = lane; t < num; t += 32) {
    const int j = idx[t];
    atomicOr(&sb[warp][j >> 5], 1u << (j & 31));
  }
  __syncwarp();
  const int NWP = ((NW + 3) >> 2) << 2;  // rows padded to whole 16-byte vectors
  for (int w = lane; w < NWP; w += 32) bits[static_cast<size_t>(row) * NWP + w] = w < NW ? sb[warp][w] : 0u;
}

__device__ __forceinline__ bool cand_better(float ja, int a, float jb, int b) { return ja > jb || (ja == jb && a < b); }

// Candidates of every block i of a head: the GRP_CAND blocks j != i with the largest Jaccard index
// |A_i & A_j| / |A_i | A_j| (approximate: each lane keeps its best 2, the warp the best GRP_CAND of those 64).
// Warp per row, lanes over j; bitmaps read as 16-byte vectors through L1 (rows are NW4 = ceil(NW / 4) vectors,
// the bitmap array padded accordingly).
__global__ void __launch_bounds__(256) k_group_cand(int N, int BH, int NW4, const uint4* __restrict__ bits,
                                                    int* __restrict__ cand_j, float* __restrict__ cand_s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;  // bh * N + i
  if (row >= BH * N) return;
  const int bh = row / N, i = row - bh * N;
  const uint4* hb = bits + static_cast<size_t>(bh) * N * NW4;
  const uint4* ri = hb + static_cast<size_t>(i) * NW4;
  int ci = 0;
  for (int w = 0; w < NW4; ++w) {
    const uint4 a = __ldg(ri + w);
    ci += __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w);
  }
  float b0 = -1.f, b1 = -1.f;
  int j0 = INT_MAX, j1 = INT_MAX;
  for (int j = lane; j < N; j += 32) {
    if (j == i) continue;
    const uint4* rj = hb + static_cast<size_t>(j) * NW4;
    int inter = 0, cj = 0;
    for (int w = 0; w < NW4; ++w) {
      const uint4 a = __ldg(ri + w), b = __ldg(rj + w);
      inter += __popc(a.x & b.x) + __popc(a.y & b.y) + __popc(a.z & b.z) + __popc(a.w & b.w);
      cj += __popc(b.x) + __popc(b.y) + __popc(b.z) + __popc(b.w);
    }
    const int uni = ci + cj - inter;
    const float jac = uni > 0 ? static_cast<float>(inter) / static_cast<float>(uni) : 0.f;
    if (cand_better(jac, j, b1, j1)) {
      if (cand_better(jac, j, b0, j0)) { b1 = b0; j1 = j0; b0 = jac; j0 = j; }
      else { b1 = jac; j1 = j; }
    }
  }
  int head = 0;
  for (int r = 0; r < GRP_CAND; ++r) {
    float best = head == 0 ? b0 : (head == 1 ? b1 : -2.f);
    int bestj = head == 0 ? j0 : (head == 1 ? j1 : INT_MAX);
    const int mine = bestj;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bestj, o);
      if (cand_better(ob, oj, best, bestj)) { best = ob; bestj = oj; }
    }
    if (mine == bestj && bestj != INT_MAX) ++head;  // the lane that owned it advances
    if (lane == 0) {
      cand_j[static_cast<size_t>(row) * GRP_CAND + r] = (best >= 0.f && bestj != INT_MAX) ? bestj : -1;
      cand_s[static_cast<size_t>(row) * GRP_CAND + r] = best;
    }
  }
}

// Per head, one CTA of 1024 threads. Level l groups up to 2^l blocks; a level pairs the current groups by
// rounds of mutual best match (each alive group proposes its most Jaccard-similar alive candidate group; mutual
// proposals pair up), and the leftovers are paired in index order. The candidate groups of a group are the
// groups of its members' candidate blocks (level 0: k_group_cand's list); at levels >= 1 their similarity is
// the Jaccard index of the groups' union bitmaps (scratch `ubits`), computed once per level.
constexpr int GRP_LCAND = 2 * GRP_CAND;  // candidate groups per group (levels >= 1)

// Exclusive prefix sum of flags over i in [0, n) for a 1024-thread CTA (thread t owns i = 4t .. 4t+3);
// returns the total. `wsum` is 32 ints of shared scratch.
__device__ __forceinline__ int cta_excl_scan4(const int* flag, int* pos, int n, int* wsum) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int v[4], s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = 4 * t + k;
    v[k] = i < n ? flag[i] : 0;
    s += v[k];
  }
  int incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = wsum[lane], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    wsum[lane] = wi - w;  // exclusive warp offsets
  }
  __syncthreads();
  int run = wsum[warp] + incl - s;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = 4 * t + k;
    if (i < n) pos[i] = run;
    run += v[k];
  }
  __syncthreads();
  const int total = wsum[31] + __shfl_sync(0xffffffffu, incl, 31);  // (valid in warp 31)
  __shared__ int s_total;
  if (t == 1023) s_total = total;
  __syncthreads();
  return s_total;
}

__global__ void __launch_bounds__(1024) k_group_match(int N, int G, int ntiles, int lists_in_smem,
                                                      const uint32_t* __restrict__ bits,
                                                      const int* __restrict__ cand_j,
                                                      const float* __restrict__ cand_s, uint32_t* __restrict__ ubits,
                                                      int* __restrict__ perm, int* __restrict__ lcand,
                                                      float* __restrict__ lscore) {
  extern __shared__ int gsm[];
  const int bh = blockIdx.x, tid = threadIdx.x;
  const int NW = (((N + 31) >> 5) + 3) & ~3;  // padded row length (k_group_bits)
  int* grp = gsm;            // representative of each block's group (the group's smallest block)
  int* nxt = gsm + N;        // next member in the group's list (-1 = end)
  int* alive = gsm + 2 * N;  // 1 while the group (by representative) is unmatched at this level
  int* prop = gsm + 3 * N;   // this round's proposal of each group; reused as scan output
  int* tail = gsm + 4 * N;   // last member of each group's list
  int* byrank = gsm + 5 * N; // leftover group of each rank
  __shared__ int wsum[32];
  __shared__ int s_changed;
  // [N][GRP_LCAND] candidate groups of each group (-1 = none) and their similarity: shared memory if they fit
  int* lj = lists_in_smem ? gsm + 6 * N : lcand + static_cast<size_t>(bh) * GRP_LCAND * N;
  float* ls = lists_in_smem ? reinterpret_cast<float*>(gsm + 6 * N + GRP_LCAND * N)
                            : lscore + static_cast<size_t>(bh) * GRP_LCAND * N;
  // bitmaps of the blocks (hb) and of the groups (ub): shared memory when the lists are there too
  uint32_t* hbs = reinterpret_cast<uint32_t*>(gsm + 6 * N + 2 * GRP_LCAND * N);
  const uint32_t* hb = lists_in_smem ? hbs : bits + static_cast<size_t>(bh) * N * NW;
  uint32_t* ub = lists_in_smem ? hbs + static_cast<size_t>(N) * NW : ubits + static_cast<size_t>(bh) * N * NW;
  if (lists_in_smem)
    for (int v = tid; v < N * NW; v += blockDim.x) hbs[v] = __ldg(bits + static_cast<size_t>(bh) * N * NW + v);
  const int* cj = cand_j + static_cast<size_t>(bh) * N * GRP_CAND;
  const float* cs = cand_s + static_cast<size_t>(bh) * N * GRP_CAND;
  for (int i = tid; i < N; i += blockDim.x) {
    grp[i] = i;
    nxt[i] = -1;
    tail[i] = i;
  }
  __syncthreads();
  // merge group j into group r (r < j): r's list continues with j's
  auto absorb = [&](int r, int j) {
    nxt[tail[r]] = j;
    tail[r] = tail[j];
    for (int m = j; m >= 0; m = nxt[m]) grp[m] = r;
  };
  for (int size = 1; size < G; size <<= 1) {
    // (1) union bitmaps of the current groups (size 1: the blocks' own bitmaps are used directly)
    for (int r = tid; r < N; r += blockDim.x) {
      alive[r] = (grp[r] == r) ? 1 : 0;
      if (grp[r] != r || size == 1) continue;
      for (int w = 0; w < NW; ++w) {
        uint32_t u = 0u;
        for (int m = r; m >= 0; m = nxt[m]) u |= hb[static_cast<size_t>(m) * NW + w];
        ub[static_cast<size_t>(r) * NW + w] = u;
      }
    }
    __syncthreads();
    // (2) candidate groups and their similarity, once per level
    const uint32_t* gb = size == 1 ? hb : ub;
    for (int r = tid; r < N; r += blockDim.x) {
      if (grp[r] != r) continue;
      int n = 0;
      if (size == 1) {
        for (int k = 0; k < GRP_CAND; ++k) {
          lj[static_cast<size_t>(r) * GRP_LCAND + k] = cj[static_cast<size_t>(r) * GRP_CAND + k];
          ls[static_cast<size_t>(r) * GRP_LCAND + k] = cs[static_cast<size_t>(r) * GRP_CAND + k];
        }
        n = GRP_CAND;
      } else {
        int cu = 0;
        for (int w = 0; w < NW; ++w) cu += __popc(gb[static_cast<size_t>(r) * NW + w]);
        int seen[GRP_LCAND];
        for (int m = r; m >= 0 && n < GRP_LCAND; m = nxt[m])
          for (int k = 0; k < GRP_CAND && n < GRP_LCAND; ++k) {
            const int jb = cj[static_cast<size_t>(m) * GRP_CAND + k];
            if (jb < 0) continue;
            const int j = grp[jb];
            if (j == r) continue;
            bool dup = false;
            for (int q = 0; q < n; ++q) dup |= seen[q] == j;
            if (dup) continue;
            int inter = 0, cjn = 0;
            for (int w = 0; w < NW; ++w) {
              const uint32_t a = gb[static_cast<size_t>(r) * NW + w], b = gb[static_cast<size_t>(j) * NW + w];
              inter += __popc(a & b);
              cjn += __popc(b);
            }
            const int uni = cu + cjn - inter;
            seen[n] = j;
            lj[static_cast<size_t>(r) * GRP_LCAND + n] = j;
            ls[static_cast<size_t>(r) * GRP_LCAND + n] = uni > 0 ? static_cast<float>(inter) / uni : 0.f;
            ++n;
          }
      }
      for (int q = n; q < GRP_LCAND; ++q) lj[static_cast<size_t>(r) * GRP_LCAND + q] = -1;
    }
    __syncthreads();
    // (3) rounds of mutual best match
    for (int round = 0; round < GRP_ROUNDS; ++round) {
      if (tid == 0) s_changed = 0;
      for (int r = tid; r < N; r += blockDim.x) {
        prop[r] = -1;
        if (!alive[r]) continue;
        float best = -1.f;
        int bj = INT_MAX;
        for (int k = 0; k < GRP_LCAND; ++k) {
          const int j = lj[static_cast<size_t>(r) * GRP_LCAND + k];
          if (j < 0) break;
          if (!alive[j]) continue;
          const float sv = ls[static_cast<size_t>(r) * GRP_LCAND + k];
          if (cand_better(sv, j, best, bj)) { best = sv; bj = j; }
        }
        prop[r] = bj == INT_MAX ? -1 : bj;
      }
      __syncthreads();
      for (int r = tid; r < N; r += blockDim.x) {
        const int j = prop[r];
        if (alive[r] && j > r && prop[j] == r) {  // mutual: r (the smaller) absorbs j
          absorb(r, j);
          alive[r] = 0;
          alive[j] = 0;
          s_changed = 1;
        }
      }
      __syncthreads();
      const int changed = s_changed;
      __syncthreads();
      if (!changed) break;
    }
    // (4) leftovers: the still-unmatched groups, in index order, are paired consecutively
    const int nleft = cta_excl_scan4(alive, prop, N, wsum);
    for (int r = tid; r < N; r += blockDim.x)
      if (alive[r]) byrank[prop[r]] = r;
    __syncthreads();
    // the leftovers of ranks 2k and 2k+1 pair up
    for (int q = tid; 2 * q + 1 < nleft; q += blockDim.x) absorb(byrank[2 * q], byrank[2 * q + 1]);
    __syncthreads();
  }
  // tiles: one group per tile in representative order (G slots; -1 pads short groups and unused tiles)
  for (int i = tid; i < N; i += blockDim.x) alive[i] = (grp[i] == i) ? 1 : 0;
  __syncthreads();
  const int ngroups = cta_excl_scan4(alive, prop, N, wsum);
  int* ph = perm + static_cast<size_t>(bh) * ntiles * G;
  for (int r = tid; r < N; r += blockDim.x) {
    if (!alive[r]) continue;
    const int t = prop[r];
    if (t >= ntiles) continue;
    int k = 0;
    for (int m = r; m >= 0 && k < G; m = nxt[m]) ph[t * G + k++] = m;
    for (; k < G; ++k) ph[t * G + k] = -1;
  }
  for (int t = ngroups + tid; t < ntiles; t += blockDim.x)
    for (int k = 0; k < G; ++k) ph[t * G + k] = -1;
}

// tiles per head of the grouped forward: ceil(N / G) full groups plus at most one short group per level
int group_ntiles(int N, int G) {
  int levels = 0;
  while ((1 << levels) < G) ++levels;
  return (N + G - 1) / G + levels;
}

size_t group_ws_bytes(int N, int BH) {
  const size_t NW = ((N + 31) / 32 + 3) & ~size_t(3), rows = static_cast<size_t>(N) * BH;
  return rows * NW * 4 * 2 + rows * GRP_CAND * 8 + rows * GRP_LCAND * 8 + 4 * 256;
}

cudaError_t launch_group(int N, int BH, int G, const int* q2k_num, const int* q2k_idx, void* ws, int* perm,
                         cudaStream_t st) {
  const size_t NW = ((N + 31) / 32 + 3) & ~size_t(3), rows = static_cast<size_t>(N) * BH;
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint32_t* bits = reinterpret_cast<uint32_t*>(base);
  uint32_t* ubits = bits + rows * NW;
  int* cj = reinterpret_cast<int*>(ubits + rows * NW);
  float* cs = reinterpret_cast<float*>(cj + rows * GRP_CAND);
  int* lcand = reinterpret_cast<int*>(cs + rows * GRP_CAND);
  float* lscore = reinterpret_cast<float*>(lcand + rows * GRP_LCAND);
  const unsigned nb = static_cast<unsigned>((rows + 7) / 8);
  k_group_bits<<<nb, 256, 0, st>>>(N, static_cast<int>(rows), q2k_num, q2k_idx, bits);
  k_group_cand<<<nb, 256, 0, st>>>(N, BH, static_cast<int>(NW / 4), reinterpret_cast<const uint4*>(bits), cj, cs);
  const int sm_lists = 6 * N * 4 + 2 * GRP_LCAND * N * 4 + 2 * N * static_cast<int>(NW) * 4;
  const int in_smem = sm_lists <= 200 * 1024 ? 1 : 0;
  const int sm = in_smem ? sm_lists : 6 * N * 4;
  cudaError_t e = cudaFuncSetAttribute(k_group_match, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e != cudaSuccess) return e;
  k_group_match<<<BH, 1024, sm, st>>>(N, G, group_ntiles(N, G), in_smem, bits, cj, cs, ubits, perm, lcand, lscore);
  return cudaGetLastError();
}

}  // namespace bsa
