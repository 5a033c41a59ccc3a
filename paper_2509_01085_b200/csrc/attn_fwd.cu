// attn_fwd.cu — a7: block-sparse attention forward over kept queries x admitted KV blocks
// (Eq.5; kernel design P:204-210: "each Q block records its attended KV blocks
// with q2k_num and q2k_index"), followed by the fill that restores length L.
//
// B200 design:
//  * Query tiles of 128 rows of the packed Q^s (kept queries, block-major): each query block in a slot of its
//    kept count rounded up to a power of two (>= 16 rows), blocks of one slot size per tile (k_fwd_union
//    derives the tiling; persistent CTAs claim tiles). The softmax threads copy their Q^s row straight from
//    global memory into TMEM (packed bf16 pairs): Q is the A operand of every S MMA and is never
//    re-read from shared memory.
//  * The CTA walks the UNION of its blocks' KV lists (rotated start). KV block j arrives as ONE bulk
//    copy of its pre-swizzled K|V image (k_kv_image) into a 6-deep stage ring.
//  * S = Q^s K_j^T (M=128, N=BT) and O += P V_j (M=128, N=d) are tcgen05.mma kind::f16 with the A
//    operand in TMEM (Q, then P) and fp32 accumulators in TMEM; only K and V are read from shared
//    memory (the SS form with N = 64 is shared-memory-bandwidth bound on B200: tools/microbench/mma_rate.cu).
//    S and P are double-buffered in TMEM so QK(j+1) overlaps the softmax of j. Rows whose block did
//    not admit j write P = 0 (their MMA work is the union waste).
//  * Softmax: 128 threads, thread == TMEM lane == query row; online softmax in fp32 (log2 domain),
//    O rescaled in TMEM only when the running max grows by more than 2^8 (exact: same final ratio).
//  * Warp roles: w0-7 two softmax/epilogue groups, w8 TMEM allocator, w9 bulk-copy producer, w10 PV
//    issuer, w11 QK issuer (control roles on the highest warp ids: the warp arbiter favours them).
#include <cmath>
#include "kernels.h"
#include "ptx.cuh"

namespace bsa {

// Debug-only timeline of one CTA (set through bsa_debug_trace_fwd; null in production).
__device__ unsigned long long* g_fwd_trace = nullptr;
__device__ int g_fwd_trace_cta = 0;
#ifdef BSA_TRACE
__device__ __forceinline__ unsigned long long trace_clock() {
#ifdef BSA_TRACE_GLOBALTIMER
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
#else
  return clock64();
#endif
}
#define FWD_TRACE(slot, u)                           \
  do {                                               \
    if (trace_buf != nullptr && (u) < 1024)          \
      trace_buf[(slot) * 1024 + (u)] = trace_clock(); \
  } while (0)
#else
#define FWD_TRACE(slot, u) \
  do {                     \
  } while (0)
#endif

struct FwdParams {
  const bf16* Qs;         // packed kept queries [BH*Lq, d] (block-major)
  const uint8_t* kv_img;  // block-major K|V images (k_kv_image): one contiguous 2*BT*d*2-byte request per block
  Geo g;
  int Lq, SR, G;
  const int* kept_off;
  const int* kept_tok;
  const int* q2k_num;
  const int* q2k_idx;
  const int* perm;   // [BH][ntiles][G] query block of each tile slot (-1 = empty, slot g = rows [g SR, (g+1) SR)), or
                     // NULL: the packed tiles of k_fwd_union (tab / tcount)
  int ntiles;
  const int* tab;    // [tiles][MAX_G] packed tile entries, query block | row offset << 16 (-1 = none)
  const int* tcount; // number of packed tiles per head (device; written by k_fwd_union)
  int BH;
  int pack_min;      // smallest slot rows (16 by default; SR = one slot per block, the unpacked tiling)
  const uint32_t* ulists;  // [BH][ntiles][N] union entries of each tile (k_fwd_union), ucount[BH][ntiles] of them
  const int* ucount;
  int* work_ctr;           // next unclaimed tile (zeroed before the launch; the CTAs are persistent)
  float scale_log2;  // scale * log2(e)
  Rows O;            // raster output, strided
  float* lse;
  unsigned long long clsmask[8];  // key-validity mask of each block-extent class (host-computed, C23): the
                                  // image holds a block's n actual tokens in its first n rows, so bits [0, n)
  int clsn16[8];                  // key columns computed per class: n rounded up to the MMA's N step of 16
};

constexpr int FWD_THREADS = 384;
constexpr int FWD_STAGES = 6;  // K|V ring depth (5 when the two union lists of a large N need the room)
constexpr int MAX_N = 4096;
constexpr int MAX_G = 16;
// rows a query block with nk kept queries takes in a packed tile: nk rounded up to a power of two >= 8 (<= SR)
__host__ __device__ __forceinline__ int fwd_slot_size(int nk, int SR, int min_sz) {
  int sz = min_sz;
  while (sz < nk && sz < SR) sz <<= 1;
  return sz;
}

template <int D, int BT, int FWD_STAGES = bsa::FWD_STAGES>
struct FwdSmem {
  static constexpr int KV_BYTES = BT * D * 2;  // one K or V tile
  static constexpr int NCB = D / 64;            // 64-channel (128-byte) column blocks
  static constexpr int OFF_K = 0;               // stage s: K tile at OFF_K + 2 s KV_BYTES, V right after
  static constexpr int OFF_ULIST = OFF_K + FWD_STAGES * 2 * KV_BYTES;  // union entries (uint32) of 2 tiles
  // dynamic shared memory for N KV blocks: the ring, two union lists of N entries, alignment slack
  static constexpr int bytes(int N) { return OFF_ULIST + 2 * N * 4 + 1024; }
  // TMEM columns: O of the even / odd steps [0, 2D), S double buffer, Q^s (packed bf16 pairs), P double
  // buffer (packed). Buffer b = step parity = softmax group.
  static constexpr int T_O = 0, T_S = 2 * D, T_Q = 2 * D + 2 * BT, T_P = T_Q + D / 2;
  static constexpr int TMEM_COLS = (T_P + BT) <= 256 ? 256 : 512;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for x <= 0 on the FMA/ALU pipes (relieves the MUFU, 16 ex2/clk/SM): j = round(x) by the 1.5*2^23
// trick (its low mantissa bits hold j), f = x - j in [-0.5, 0.5], 2^f by a degree-3 fit (max relative
// error 1.0e-4, far below the bf16 rounding of P), 2^j added to the exponent field. x is clamped at -125
// (2^-125 stands in for 0, e.g. for masked keys).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float j = t - 12582912.f;
  const float f = x - j;
  const float p = fmaf(fmaf(fmaf(0.05500895f, f, 0.24221101f), f, 0.6932829f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Persistent: one CTA per SM claims tiles (b,h, tile) from an atomic counter. Warp 8 (after the TMEM
// allocation) prepares the NEXT tile -- slot query blocks, kept counts, its union list copied from k_fwd_union's
// output -- into the other half of a double-buffered metadata area while the current tile runs, so a tile
// costs its union steps plus the hand-over (Q^s of the next tile into TMEM, the epilogue of the last one),
// not a CTA launch and prologue (round 2: 11.8 us of fixed cost per tile in the one-CTA-per-tile kernel).
// Every role walks the same tile sequence with all barrier phases counted across tiles.
template <int D, int BT, int FWD_STAGES>
__global__ void __launch_bounds__(FWD_THREADS, 1) k_attn_fwd(const __grid_constant__ FwdParams p) {
  using SM = FwdSmem<D, BT, FWD_STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm + SM::OFF_K;
  uint32_t* ulist0 = reinterpret_cast<uint32_t*>(sm + SM::OFF_ULIST);

  __shared__ __align__(8) uint64_t bar_qt, bar_kv_full[FWD_STAGES], bar_kv_empty[FWD_STAGES], bar_s_full[2],
      bar_s_free[2], bar_p_full[2], bar_p_free[2], bar_o_final, bar_o_free, bar_meta_full[2], bar_meta_free[2];
  __shared__ float s_ml[2][2][128];  // epilogue exchange: [group][m, l][row]
  __shared__ uint32_t s_tmem;
  // per metadata buffer: claimed item (-1: no work left), slot query blocks / kept counts / kept offsets, U
  __shared__ int s_item[2], s_U[2], s_qb[2][MAX_G], s_nk[2][MAX_G], s_koff[2][MAX_G], s_roff[2][MAX_G];
  __shared__ uint8_t s_rowent[2][128];  // tile row -> its entry (0xFF: no query block)
  __shared__ int s_clsn16[8];
  // Key-validity mask of each block-extent class (bit t/h/w set = the block is the ragged last one along
  // that axis, C23): 8 classes, one 64-bit row mask each, so the per-step masking is a bit test instead of
  // per-column index arithmetic (which, unrolled, bloated the softmax loop past the instruction cache).
  __shared__ uint64_t s_clsmask[8];

  const Geo& g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef BSA_TRACE
  // per-CTA start / end stamps (debug builds; bsa_debug_trace_fwd(buf, -1)): tools/profiling/fwd_tail.py
  auto cta_stamp = [&](int k) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (g_fwd_trace != nullptr && g_fwd_trace_cta == -1) g_fwd_trace[2 * blockIdx.x + k] = t;
  };
  if (tid == 0) cta_stamp(0);
#endif
  const int G = p.G, SR = p.SR;
  const int NT = p.perm ? p.ntiles : *p.tcount;  // tiles per head
  const int total_tiles = NT * p.BH;
  constexpr int W_ALLOC = 8, W_PROD = 9, W_PV = 10, W_QK = 11;
  constexpr int META_READERS = 11;  // producer, PV issuer, QK issuer, 8 softmax warps

  if (tid == 0) {
    mbar_init(&bar_qt, 128);
    for (int s = 0; s < FWD_STAGES; ++s) { mbar_init(&bar_kv_full[s], 1); mbar_init(&bar_kv_empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_p_free[b], 1);
      mbar_init(&bar_s_full[b], 1);
      mbar_init(&bar_s_free[b], 128);
      mbar_init(&bar_p_full[b], 128);
      mbar_init(&bar_meta_full[b], 1);
      mbar_init(&bar_meta_free[b], META_READERS);
    }
    mbar_init(&bar_o_final, 1);
    mbar_init(&bar_o_free, 256);
    fence_mbar_init();
  }
  if (warp == W_ALLOC) tmem_alloc(&s_tmem, SM::TMEM_COLS);
  if (tid < 8) {
    s_clsmask[tid] = p.clsmask[tid];
    s_clsn16[tid] = p.clsn16[tid];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = s_tmem;
  constexpr uint32_t KV_BYTES = SM::KV_BYTES;
  // tile `it` of this CTA: its metadata buffer, the claimed item (-1 = done) and its rotation of the union
  // walk (concurrent CTAs start at different KV blocks instead of all streaming block 0, 1, 2, ... from the same
  // L2 slices at once; order does not change the result beyond fp32 summation order)
  auto wait_meta = [&](int it) {
    mbar_wait(&bar_meta_full[it & 1], (it >> 1) & 1);
    return s_item[it & 1];
  };
  auto release_meta = [&](int it) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&bar_meta_free[it & 1]);
  };
  auto rot_of = [&](int item, int U) {
    const int bh = item / NT, tile = item - bh * NT;
    return U > 0 ? static_cast<int>((static_cast<unsigned>(tile) * 2654435761u + bh * 40503u) % U) : 0;
  };

  if (warp == W_ALLOC) {
    // ============================ tile claimer / metadata preparation (one tile ahead)
    for (int it = 0;; ++it) {
      const int b = it & 1;
      if (it >= 2) mbar_wait(&bar_meta_free[b], ((it >> 1) - 1) & 1);  // every role is done with tile it - 2
      int item = 0;
      if (lane == 0) item = atomicAdd(p.work_ctr, 1);
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= total_tiles) item = -1;
      if (item >= 0) {
        const int tile = item % NT;
        int qb = -1, roff = 0;
        if (p.perm) {
          if (lane < G) { qb = p.perm[static_cast<size_t>(item) * G + lane]; roff = lane * SR; }
        } else if (lane < MAX_G) {
          const int e = p.tab[tile * MAX_G + lane];
          if (e >= 0) { qb = e & 0xFFFF; roff = e >> 16; }
        }
        const int nk = qb >= 0 ? p.kept_off[qb + 1] - p.kept_off[qb] : 0;
        if (lane < MAX_G) {
          s_qb[b][lane] = qb;
          s_nk[b][lane] = nk;
          s_koff[b][lane] = qb >= 0 ? p.kept_off[qb] : 0;
          s_roff[b][lane] = roff;
        }
        for (int r = lane; r < 128; r += 32) s_rowent[b][r] = 0xFF;
        __syncwarp();
        if (qb >= 0) {
          const int sz = p.perm ? SR : fwd_slot_size(nk, SR, p.pack_min);
          for (int r = roff; r < roff + sz; ++r) s_rowent[b][r] = static_cast<uint8_t>(lane);
        }
        const int U = p.ucount[item];
        const uint32_t* src = p.ulists + static_cast<size_t>(item) * g.N;
        uint32_t* dst = ulist0 + b * g.N;
        for (int u = lane; u < U; u += 32) dst[u] = __ldg(src + u);
        if (lane == 0) s_U[b] = U;
      }
      if (lane == 0) s_item[b] = item;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_meta_full[b]);  // (release: the warp's smem writes above)
      if (item < 0) break;
    }
  } else if (warp == W_PROD) {
    // ============================ bulk-copy producer
    int gs = 0;  // K|V steps over all tiles (ring position and phase)
    for (int it = 0;; ++it) {
      const int item = wait_meta(it);
      if (item < 0) break;
      const int b = it & 1, U = s_U[b], rot = rot_of(item, U), bh = item / NT;
      const uint32_t* ul = ulist0 + b * g.N;
      if (lane == 0) {
        for (int u = 0; u < U; ++u, ++gs) {
          const int s = gs % FWD_STAGES;
          const int x = u + rot;
          const uint32_t ent = ul[x >= U ? x - U : x];
          // only the first n16 rows (the block's tokens, padded to the MMA's N step) of each of the image's
          // 2 NCB column tiles are read: one request for a whole block, one per column tile for a ragged one
          const int n16 = s_clsn16[(ent >> 12) & 7];
          mbar_wait(&bar_kv_empty[s], ((gs / FWD_STAGES) & 1) ^ 1);
          mbar_expect_tx(&bar_kv_full[s], static_cast<uint32_t>(n16) * (4 * D));
          const int j = ent & 0xFFF;
          const uint8_t* src = p.kv_img + (static_cast<size_t>(bh) * g.N + j) * (2 * KV_BYTES);
          if (n16 == BT) {
            bulk_load(sK + s * 2 * KV_BYTES, src, 2 * KV_BYTES, &bar_kv_full[s]);
          } else {
#pragma unroll
            for (int t = 0; t < 2 * SM::NCB; ++t)
              bulk_load(sK + s * 2 * KV_BYTES + t * BT * 128, src + t * BT * 128, static_cast<uint32_t>(n16) * 128,
                        &bar_kv_full[s]);
          }
        }
      }
      gs = __shfl_sync(0xffffffffu, gs, 0);
      release_meta(it);
    }
  } else if (warp == W_QK || warp == W_PV) {
    // ============================ MMA issuers. One tensor pipe, two issuing warps with plain blocking
    // (suspending) waits: W_QK issues S(v) = Q^s K_v^T as soon as its K tile landed and its S buffer is
    // free (v & 1 = softmax group), W_PV issues O_b += P(u) V_u as soon as P(u) is written. QK therefore
    // runs ahead of PV by itself, and neither queue waits behind the other's dependencies. Each warp walks its
    // schedule whole (uniform registers); one elected lane issues.
    const bool leader = elect_one();
    constexpr uint32_t idesc_pv = umma_idesc_bf16(128, D, 0, 1);
    const uint32_t tO = tbase + SM::T_O, tS = tbase + SM::T_S, tQ = tbase + SM::T_Q, tP = tbase + SM::T_P;
    // base descriptors; an operand at byte offset o from the base is base + (o >> 4)
    const uint64_t dK0 = umma_desc_sw128(smem_u32(sK), 16, 1024);
    const uint64_t dV0 = umma_desc_sw128(smem_u32(sK + KV_BYTES), BT * 128, 1024);
    int gs = 0;               // steps over all tiles (K|V ring position)
    int nb[2] = {0, 0};       // uses of S buffer / P buffer b over all tiles
    for (int it = 0;; ++it) {
      const int item = wait_meta(it);
      if (item < 0) break;
      const int b = it & 1, U = s_U[b], rot = rot_of(item, U);
      const uint32_t* ul = ulist0 + b * g.N;
      auto entry_at = [&](int u) { int x = u + rot; return ul[x >= U ? x - U : x]; };
      if (warp == W_QK) {
        mbar_wait(&bar_qt, it & 1);  // Q^s of this tile is in TMEM
        for (int v = 0; v < U; ++v, ++gs) {
          const int s = gs % FWD_STAGES, sb = v & 1;
          const uint32_t idesc_qk = umma_idesc_bf16(128, s_clsn16[(entry_at(v) >> 12) & 7], 0, 0);  // N = n16
          mbar_wait(&bar_kv_full[s], (gs / FWD_STAGES) & 1);
          if (nb[sb] > 0) mbar_wait(&bar_s_free[sb], (nb[sb] - 1) & 1);
          tc_fence_after();
          const uint64_t kst = dK0 + ((s * 2 * KV_BYTES) >> 4);
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const int cb = kk >> 2, ko = (kk & 3) * 32;
              umma_ts(tS + sb * BT, tQ + kk * 8, kst + ((cb * BT * 128 + ko) >> 4), idesc_qk, kk > 0);
            }
            umma_commit(&bar_s_full[sb]);
          }
          __syncwarp();
          ++nb[sb];
        }
      } else {
        for (int u = 0; u < U; ++u, ++gs) {
          const int pb = u & 1, s = gs % FWD_STAGES;
          const int nkk = s_clsn16[(entry_at(u) >> 12) & 7] / 16;  // K = n16 keys
          const uint32_t tPu = tP + pb * (BT / 2);
          mbar_wait(&bar_p_full[pb], nb[pb] & 1);
          // the tile's first PV of each group overwrites O_b: the last tile's epilogue must have read it
          if (u < 2 && it > 0) mbar_wait(&bar_o_free, (it - 1) & 1);
          tc_fence_after();
          const uint64_t vst = dV0 + ((s * 2 * KV_BYTES) >> 4);
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < BT / 16; ++kk) {
              if (kk >= nkk) break;
              umma_ts(tO + pb * D, tPu + kk * 8, vst + ((kk * 2048) >> 4), idesc_pv, (u > 1 || kk > 0) ? 1u : 0u);
            }
            // QK(u) (the other issuer) completed before P(u) could exist, so this commit covers every
            // read of the stage
            umma_commit(&bar_kv_empty[s]);
            umma_commit(&bar_p_free[pb]);
          }
          __syncwarp();
          ++nb[pb];
        }
        if (leader) umma_commit(&bar_o_final);  // completes once every PV of the tile has landed in TMEM
        __syncwarp();
      }
      release_meta(it);
    }
  } else if (warp < 8) {
    // ============================ softmax + epilogue: two groups of four warps. Group b = warp / 4 runs
    // the steps u = b, b+2, ... with its own running max / sum and its own O accumulator (TMEM columns
    // [b D, (b+1) D)), so the two groups on one sub-partition (warps w and w+4 share TMEM lane quadrant
    // w % 4) fill each other's latency; the two partial results are merged in the epilogue (split-K).
    const int group = warp >> 2, q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t trow = tbase + (static_cast<uint32_t>(q4 * 32) << 16);
    const float sl2 = p.scale_log2;
    const uint32_t tS = trow + SM::T_S + group * BT, tP = trow + SM::T_P + group * (BT / 2);
    const uint32_t tO = trow + SM::T_O + group * D;
    int ns = 0;  // this group's steps over all tiles (phases of its S / P buffers)
    for (int it = 0;; ++it) {
      const int item = wait_meta(it);
      if (item < 0) break;
      const int b = it & 1, U = s_U[b], rot = rot_of(item, U), bh = item / NT;
      const uint32_t* ul = ulist0 + b * g.N;
      auto entry_at = [&](int u) { int x = u + rot; return ul[x >= U ? x - U : x]; };
      const int gi = s_rowent[b][row];  // this row's entry (its bit in an union entry's admitting mask)
      const int lr = gi != 0xFF ? row - s_roff[b][gi] : 0;
      const bool valid = gi != 0xFF && lr < s_nk[b][gi];
      const int mybit = 16 + (valid ? gi : 0);
      const size_t prow_idx = valid ? static_cast<size_t>(bh) * p.Lq + s_koff[b][gi] + lr : 0;
      if (group == 0) {
        // Q^s row -> TMEM (A operand of the S MMAs): bf16 pairs in memory order. The last tile's QKs are all
        // complete (its epilogue waited for every PV, each after its own S). (Loading the next tile's rows into
        // registers before the epilogue spilled the softmax role: 496 bytes.)
        uint4 qrow[D / 8];
        const uint4* src = reinterpret_cast<const uint4*>(p.Qs + prow_idx * D);
#pragma unroll
        for (int e = 0; e < D / 8; ++e) qrow[e] = valid ? src[e] : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c0 = 0; c0 < D / 2; c0 += 16) {
          float w[16];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint4 v = qrow[c0 / 4 + e];
            w[4 * e] = __uint_as_float(v.x);
            w[4 * e + 1] = __uint_as_float(v.y);
            w[4 * e + 2] = __uint_as_float(v.z);
            w[4 * e + 3] = __uint_as_float(v.w);
          }
          tmem_st16(trow + SM::T_Q + c0, w);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bar_qt);
      }
      float m_run = -INFINITY, l_run = 0.f;
      for (int u = group; u < U; u += 2, ++ns) {
        const int ph = ns & 1;  // phase of this group's buffers
        const uint32_t ent = entry_at(u);
        const int cls = (ent >> 12) & 7;
        // The softmax always covers all BT columns (columns past the block's n tokens are masked, so stale
        // TMEM values of a shorter S never leak): skipping the unused 16-column chunks of ragged blocks broke
        // the instruction scheduling of the exp loop (0.87 -> 0.99 ms); only the MMAs and copies use n16.
        const bool admit = valid && ((ent >> mybit) & 1u);
        mbar_wait(&bar_s_full[group], ph);
        tc_fence_after();
        float sv[BT];
#pragma unroll
        for (int c = 0; c < BT; c += 16) tmem_ld16(tS + c, sv + c);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bar_s_free[group]);
        float alpha = 1.f;
        bool need_rescale = false;
        if (admit) {
          // key validity (ragged edge blocks: only actual tokens, C23); raw scores, scale folded into ex2
          if (cls != 0) {
            const uint64_t km = s_clsmask[cls];
            const uint32_t k0 = static_cast<uint32_t>(km), k1 = static_cast<uint32_t>(km >> 32);
#pragma unroll
            for (int c = 0; c < BT; ++c)
              if (!(((c < 32 ? k0 : k1) >> (c & 31)) & 1u)) sv[c] = -INFINITY;
          }
          // row max and row sum with independent partial accumulators: a single serial chain of BT dependent
          // FMNMX/FADD would cost more than the MUFU work it waits on
          float mp[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < BT; ++c) mp[c & 3] = fmaxf(mp[c & 3], sv[c]);
          float mx = fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])) * sl2;
          if (mx > m_run + 8.f) {  // conditional rescale: keep the stale max unless it grew by > 2^8
            if (m_run != -INFINITY) { alpha = ex2(m_run - mx); need_rescale = true; }
            l_run *= alpha;
            m_run = mx;
          }
          // paired fp32 arithmetic (FFMA2 / FADD2): two columns per instruction for the scale-and-shift and
          // the row sum (1.003 -> 0.992 ms at 32k)
          float2 sp2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                           make_float2(0.f, 0.f)};
          const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m_run, -m_run);
#pragma unroll
          for (int c = 0; c < BT; c += 2) {  // one column in four on the FMA pipe, the rest on the MUFU
            const float2 x = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nm);
            sv[c] = ex2(x.x);
            sv[c + 1] = ((c + 1) & 3) == 3 ? ex2_poly(x.y) : ex2(x.y);
            sp2[(c >> 1) & 3] = __fadd2_rn(sp2[(c >> 1) & 3], make_float2(sv[c], sv[c + 1]));
          }
          l_run += ((sp2[0].x + sp2[0].y) + (sp2[1].x + sp2[1].y)) + ((sp2[2].x + sp2[2].y) + (sp2[3].x + sp2[3].y));
        } else {
#pragma unroll
          for (int c = 0; c < BT; ++c) sv[c] = 0.f;
        }
        // P buffer and O accumulator of this group are free once its previous PV completed
        if (ns > 0) mbar_wait(&bar_p_free[group], ph ^ 1);
        // O rescale in TMEM; warp-collective access
        if (__any_sync(0xffffffffu, need_rescale)) {
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D; c += 16) {
            float ov[16];
            tmem_ld16(tO + c, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) ov[e] *= alpha;
            tmem_st16(tO + c, ov);
          }
        }
        // P row -> TMEM (bf16 pairs, the A operand of PV)
#pragma unroll
        for (int c0 = 0; c0 < BT / 2; c0 += 16) {
          float w[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) w[e] = __uint_as_float(pack_bf16(sv[2 * (c0 + e)], sv[2 * (c0 + e) + 1]));
          tmem_st16(tP + c0, w);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bar_p_full[group]);
      }
      // group 0 issues the next tile's Q^s row loads now, so their latency overlaps this epilogue (its
      // metadata was prepared during this tile)
      // epilogue: merge the two groups' (m, l, O), O^s = O / l scattered to the kept token's raster row,
      // LSE in natural log. Group b writes output columns [b D/2, (b+1) D/2).
      s_ml[group][0][row] = m_run;
      s_ml[group][1][row] = l_run;
      mbar_wait(&bar_o_final, it & 1);
      tc_fence_after();
      named_bar_sync(1, 256);
      const float m0 = s_ml[0][0][row], l0 = s_ml[0][1][row], m1 = s_ml[1][0][row], l1 = s_ml[1][1][row];
      const bool has1 = U > 1;  // the odd group ran at least one step (its O columns were written)
      const float m = has1 ? fmaxf(m0, m1) : m0;
      const float a0 = valid ? ex2(m0 - m) : 0.f, a1 = (valid && has1) ? ex2(m1 - m) : 0.f;
      const float l = l0 * a0 + l1 * a1;
      const float inv = valid ? 1.f / l : 0.f;
      bf16* orow = nullptr;
      if (valid) {
        const int tok = p.kept_tok[prow_idx];
        orow = p.O.row(bh, tok);
        if (group == 0) p.lse[prow_idx] = (m + log2f(l)) * 0.6931471805599453f;
      }
      const float s0 = a0 * inv, s1 = a1 * inv;
#pragma unroll 1
      for (int c = group * (D / 2); c < (group + 1) * (D / 2); c += 16) {
        float o0[16], o1[16];
        tmem_ld16(trow + SM::T_O + c, o0);
        if (has1) tmem_ld16(trow + SM::T_O + D + c, o1);
        tmem_wait_ld();
        if (valid) {
          uint32_t w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float x0 = has1 ? o0[2 * e] * s0 + o1[2 * e] * s1 : o0[2 * e] * s0;
            const float x1 = has1 ? o0[2 * e + 1] * s0 + o1[2 * e + 1] * s1 : o0[2 * e + 1] * s0;
            w[e] = pack_bf16(x0, x1);
          }
          *reinterpret_cast<uint4*>(orow + c) = make_uint4(w[0], w[1], w[2], w[3]);
          *reinterpret_cast<uint4*>(orow + c + 8) = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      tc_fence_before();
      mbar_arrive(&bar_o_free);  // O read: the next tile's first PVs may overwrite it
      named_bar_sync(1, 256);    // (s_ml is rewritten by the next tile's epilogue)
      release_meta(it);
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef BSA_TRACE
  if (tid == 0) cta_stamp(1);
#endif
  if (warp == W_ALLOC) tmem_dealloc(tbase, SM::TMEM_COLS);
}

// Union pre-pass (one CTA per (tile, b,h)): the ascending union of the tile slots' admitted KV blocks (P:210
// q2k lists), entry = j | extent class << 12 (bit 2/1/0: ragged last block along t/h/w, C23) | mask << 16 of the
// slots that admitted j. Built here, in parallel for all tiles, so the attention CTA's prologue is one list copy.
//
// Packed tiles (perm == NULL): the tiles of build_fwd_tiling (tab / tcount).
template <int MAXG>
__global__ void __launch_bounds__(256) k_fwd_union(Geo g, int G, int ntiles, const int* __restrict__ perm,
                                                   const int* __restrict__ q2k_num, const int* __restrict__ q2k_idx,
                                                   uint32_t* __restrict__ ulists, int* __restrict__ ucount,
                                                   const int* __restrict__ tab, const int* __restrict__ tcount) {
  extern __shared__ uint32_t ubits[];  // [G][NW] slot bitmaps
  __shared__ int s_qb[MAXG];
  __shared__ int s_upre[MAX_N / 32];
  __shared__ int s_tot;
  const int tile = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NW = (g.N + 31) >> 5;
  int NT = ntiles;
  if (perm) {
    if (tid < G) s_qb[tid] = perm[(static_cast<size_t>(bh) * ntiles + tile) * G + tid];
  } else {  // packed tiles (k_kv_image's tiling CTA wrote tab / tcount)
    G = MAXG;
    NT = *tcount;
    if (tile >= NT) return;  // (uniform)
    if (tid < MAXG) {
      const int e = tab[tile * MAXG + tid];
      s_qb[tid] = e >= 0 ? e & 0xFFFF : -1;
    }
  }
  for (int w = tid; w < G * NW; w += 256) ubits[w] = 0u;
  __syncthreads();
  for (int gi = 0; gi < G; ++gi) {
    const int qb = s_qb[gi];
    if (qb < 0) continue;
    const size_t row = static_cast<size_t>(bh) * g.N + qb;
    const int num = q2k_num[row];
    const int* idx = q2k_idx + row * g.N;
    for (int a = tid; a < num; a += 256) {
      const int j = idx[a];
      atomicOr(&ubits[gi * NW + (j >> 5)], 1u << (j & 31));
    }
  }
  __syncthreads();
  if (warp == 0) {  // word popcount prefix of the union
    int carry = 0;
    for (int w0 = 0; w0 < NW; w0 += 32) {
      const int w = w0 + lane;
      uint32_t v = 0u;
      if (w < NW)
        for (int gi = 0; gi < G; ++gi) v |= ubits[gi * NW + w];
      const int c = __popc(v);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += a;
      }
      if (w < NW) s_upre[w] = carry + incl - c;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_tot = carry;
  }
  __syncthreads();
  const size_t tix = static_cast<size_t>(bh) * NT + tile;
  uint32_t* out = ulists + tix * g.N;
  for (int w = warp; w < NW; w += 8) {
    uint32_t v = 0u, mask = 0u;
    for (int gi = 0; gi < G; ++gi) {
      const uint32_t b = ubits[gi * NW + w];
      v |= b;
      mask |= ((b >> lane) & 1u) << gi;
    }
    if ((v >> lane) & 1u) {
      const int jj = w * 32 + lane;
      const int bt = jj / (g.Nh * g.Nw), bhh = (jj / g.Nw) % g.Nh, bw = jj % g.Nw;
      const uint32_t cls = (bt == g.Nt - 1 && g.T % g.ct ? 4u : 0u) | (bhh == g.Nh - 1 && g.H % g.ch ? 2u : 0u) |
                           (bw == g.Nw - 1 && g.W % g.cw ? 1u : 0u);
      out[s_upre[w] + __popc(v & ((1u << lane) - 1u))] = static_cast<uint32_t>(jj) | (cls << 12) | (mask << 16);
    }
  }
  if (tid == 0) ucount[tix] = s_tot;
}

int fwd_max_tiles(int N, int SR) { return (N + 128 / SR - 1) / (128 / SR) + 4; }

cudaError_t launch_fwd_union(const FwdArgs& a, uint32_t* ulists, int* ucount, cudaStream_t st) {
  const int G = a.perm ? 128 / a.SR : MAX_G;
  const int ntiles = a.perm ? a.ntiles : fwd_max_tiles(a.g.N, a.SR);  // packed: an upper bound (CTAs past it exit)
  const int NW = (a.g.N + 31) / 32;
  k_fwd_union<MAX_G><<<dim3(ntiles, a.BH), 256, G * NW * 4, st>>>(a.g, G, ntiles, a.perm, a.q2k_num, a.q2k_idx, ulists, ucount, a.tab,
                                                                 a.tcount);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 2D row map over a packed [rows, d] bf16 matrix, box {64, box_rows}, 128B swizzle.
bool make_map_2d(CUtensorMap* m, const void* base, int d, size_t rows, int box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
  cuuint64_t str[1] = {static_cast<cuuint64_t>(d) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2D row map over a packed [rows, d] fp32 matrix, box {32, box_rows} (128-byte rows), 128B swizzle.
bool make_map_rows_f32(CUtensorMap* m, const void* base, int d, size_t rows, int box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
  cuuint64_t str[1] = {static_cast<cuuint64_t>(d) * 4};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 5D block map over `heads` raster heads of a bf16 tensor, [heads][T][H][W][d] with token stride sl and head
// stride sh (elements; d contiguous), box {64, cw, ch, ct, 1}, 128B swizzle. base = token 0 of head 0.
bool make_map_5d(CUtensorMap* m, const void* base, const Geo& g, int d, int heads, long long sl, long long sh) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[5] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(g.W), static_cast<cuuint64_t>(g.H),
                        static_cast<cuuint64_t>(g.T), static_cast<cuuint64_t>(heads)};
  cuuint64_t rs = static_cast<cuuint64_t>(sl) * 2;
  cuuint64_t str[4] = {rs, rs * g.W, rs * g.W * g.H, static_cast<cuuint64_t>(sh) * 2};
  cuuint32_t box[5] = {64, static_cast<cuuint32_t>(g.cw), static_cast<cuuint32_t>(g.ch),
                       static_cast<cuuint32_t>(g.ct), 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, int BT, int ST>
static cudaError_t run_fwd_st(const FwdParams& p, int ntiles, int BH, cudaStream_t st) {
  const int smem = FwdSmem<D, BT, ST>::bytes(p.g.N);
  cudaError_t e = cudaFuncSetAttribute(k_attn_fwd<D, BT, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p.work_ctr, 0, sizeof(int), st)) != cudaSuccess) return e;
  const int total = ntiles * BH;
  k_attn_fwd<D, BT, ST><<<dim3(static_cast<unsigned>(total < sms ? total : sms)), FWD_THREADS, smem, st>>>(p);  // persistent
  return cudaGetLastError();
}
// six K|V stages when they fit next to the two union lists (N <= ~4000 at d = 128), else five
template <int D, int BT>
static cudaError_t run_fwd(const FwdParams& p, int ntiles, int BH, cudaStream_t st) {
  constexpr int kStatic = 4096;  // static shared memory of the kernel (< 3 KB) with margin
  if (FwdSmem<D, BT, 6>::bytes(p.g.N) + kStatic <= 227 * 1024) return run_fwd_st<D, BT, 6>(p, ntiles, BH, st);
  return run_fwd_st<D, BT, 5>(p, ntiles, BH, st);
}

cudaError_t launch_attn_fwd(const FwdArgs& a, cudaStream_t st) {
  FwdParams p;
  memset(&p, 0, sizeof(p));
  p.g = a.g;
  p.Lq = a.Lq;
  p.SR = a.SR;
  p.G = 128 / a.SR;
  p.kept_off = a.kept_off;
  p.kept_tok = a.kept_tok;
  p.q2k_num = a.q2k_num;
  p.q2k_idx = a.q2k_idx;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.O = a.O;
  p.lse = a.lse;
  p.kv_img = a.kv_img;
  p.Qs = a.Qs;
  p.perm = a.perm;
  p.ntiles = a.perm ? a.ntiles : fwd_max_tiles(a.g.N, a.SR);
  p.tab = a.tab;
  p.tcount = a.tcount;
  p.BH = a.BH;
  p.pack_min = a.pack_min;
  p.ulists = a.ulists;
  p.ucount = a.ucount;
  p.work_ctr = a.work_ctr;
  for (int cls = 0; cls < 8; ++cls) {  // key-validity mask per block-extent class (ragged last block per axis)
    const Geo& g = a.g;
    const int et = (cls & 4) ? g.T - (g.Nt - 1) * g.ct : g.ct;
    const int eh = (cls & 2) ? g.H - (g.Nh - 1) * g.ch : g.ch;
    const int ew = (cls & 1) ? g.W - (g.Nw - 1) * g.cw : g.cw;
    const int n = et * eh * ew;  // the image holds the block's n tokens in rows [0, n)
    p.clsmask[cls] = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
#ifndef BSA_FWD_FULLN
    p.clsn16[cls] = (n + 15) / 16 * 16;
#else
    p.clsn16[cls] = g.BT;
#endif
  }
  const int ntiles = p.ntiles;  // (an upper bound for the packed tiles: surplus CTAs find no work)
  if (a.d == 128 && a.g.BT == 64) return run_fwd<128, 64>(p, ntiles, a.BH, st);
  if (a.d == 128 && a.g.BT == 32) return run_fwd<128, 32>(p, ntiles, a.BH, st);
  if (a.d == 64 && a.g.BT == 64) return run_fwd<64, 64>(p, ntiles, a.BH, st);
  if (a.d == 64 && a.g.BT == 32) return run_fwd<64, 32>(p, ntiles, a.BH, st);
  return cudaErrorInvalidValue;
}

// K|V block images: for every (bh, KV block j) the exact shared-memory image the forward MMAs read, ONE
// contiguous bulk copy per KV step (small TMA boxes cost ~500 cycles each). Rows = keys: the block's n actual
// tokens in ascending raster order first (compacted: a ragged edge block's rows are a prefix, C23), zero rows
// up to n16 = n rounded up to 16 (the MMA's N step), nothing beyond (never read). Layout [K: d-half 0 as BT
// rows x 128 B, d-half 1 ...][V: same], 128-byte swizzled (8-row groups 1 KB apart: an image of 8-row groups
// 4 KB apart, which makes the first n16 keys one prefix, slowed the MMAs' operand reads, 0.87 -> 1.07 ms).
//
// Packed forward tiles, built by one extra CTA of this launch (so they cost no launch of their own): a query
// block takes fwd_slot_size(nk) rows (its kept count rounded up to a power of two >= pack_min, at most SR), and
// the blocks of one slot size fill tiles of 128 / size of them in block order (a ragged edge block's 8 or 16
// kept queries no longer pad a 32- or 64-row slot); the classes' tiles follow each other, smallest slots first
// by default. tab[tile][e] = query block | row offset << 16 (-1: empty), *tcount = tiles per head.
__device__ void build_fwd_tiling(const Geo& g, const FwdTiling& tl) {
  __shared__ int s_cnt[4], s_first[4], s_carry[4], s_w[8][4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < tl.max_tiles * MAX_G; i += 256) tl.tab[i] = -1;
  if (tid < 4) { s_cnt[tid] = 0; s_carry[tid] = 0; }
  __syncthreads();
  auto cls_of = [&](int j) {  // log2(slot size / 8), -1 for a block without kept queries
    const int nk = tl.kept_off[j + 1] - tl.kept_off[j];
    return nk > 0 ? 31 - __clz(fwd_slot_size(nk, tl.SR, tl.pack_min) >> 3) : -1;
  };
  for (int j = tid; j < g.N; j += 256) {
    const int c = cls_of(j);
    if (c >= 0) atomicAdd(&s_cnt[c], 1);
  }
  __syncthreads();
  if (tid == 0) {
    int t0 = 0;
    for (int ci = 0; ci < 4; ++ci) {
      const int c = tl.small_first ? ci : 3 - ci;
      s_first[c] = t0;
      t0 += (s_cnt[c] + (16 >> c) - 1) / (16 >> c);
    }
    *tl.tcount = t0;
  }
  __syncthreads();
  for (int j0 = 0; j0 < g.N; j0 += 256) {  // stable rank of each block within its class
    const int j = j0 + tid;
    const int c = j < g.N ? cls_of(j) : -1;
    unsigned bal[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bal[k] = __ballot_sync(0xffffffffu, c == k);
      if (lane == 0) s_w[warp][k] = __popc(bal[k]);
    }
    __syncthreads();
    if (c >= 0) {
      int rank = s_carry[c] + __popc(bal[c] & ((1u << lane) - 1u));
      for (int w = 0; w < warp; ++w) rank += s_w[w][c];
      const int per = 16 >> c, tile = s_first[c] + rank / per, slot = rank % per;
      tl.tab[tile * MAX_G + slot] = j | ((slot * (8 << c)) << 16);
    }
    __syncthreads();
    if (tid < 4)
      for (int w = 0; w < 8; ++w) s_carry[tid] += s_w[w][tid];
    __syncthreads();
  }
}

template <int D, int BT>
__global__ void __launch_bounds__(256) k_kv_image(Geo g, const Rows K, const Rows V, uint8_t* __restrict__ img,
                                                  const FwdTiling tl) {
  if (blockIdx.x == g.N) {  // the extra CTA of head 0 builds the forward tiling
    if (blockIdx.y == 0) build_fwd_tiling(g, tl);
    return;
  }
  constexpr int CPR = D / 8;        // 16-byte chunks per row
  constexpr int CHUNKS = BT * CPR;  // per tensor
  constexpr int PER = 2 * CHUNKS / 256;  // chunks per thread (K and V)
  const int j = blockIdx.x, bh = blockIdx.y;
  const Box x = block_box(g, j);
  const int n = x.e[0] * x.e[1] * x.e[2], n16 = (n + 15) & ~15;
  uint8_t* dst = img + (static_cast<size_t>(bh) * g.N + j) * (2 * BT * D * 2);
  const bf16* kh = K.head(bh);
  const bf16* vh = V.head(bh);
  // every load of the thread is issued before the first store (memory-level parallelism)
  uint4 val[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int v = threadIdx.x + 256 * k;
    const int t = v / CHUNKS, w = v % CHUNKS;
    const int r = w / CPR, c = w % CPR;
    val[k] = make_uint4(0, 0, 0, 0);
    if (r < n) {
      const int lw = r % x.e[2], lh = (r / x.e[2]) % x.e[1], lt = r / (x.e[2] * x.e[1]);
      const long long tok = (static_cast<long long>(x.o[0] + lt) * g.H + (x.o[1] + lh)) * g.W + (x.o[2] + lw);
      val[k] = __ldg(reinterpret_cast<const uint4*>((t ? vh + tok * V.sl : kh + tok * K.sl) + c * 8));
    }
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int v = threadIdx.x + 256 * k;
    const int t = v / CHUNKS, w = v % CHUNKS;
    const int r = w / CPR, c = w % CPR;
    if (r < n16)
      *reinterpret_cast<uint4*>(dst + t * (BT * D * 2) + (c >> 3) * (BT * 128) + sw128_off(r, c & 7)) = val[k];
  }
}

cudaError_t launch_kv_image(const Geo& g, int BH, int d, Rows K, Rows V, uint8_t* img, const FwdTiling& tl,
                            cudaStream_t st) {
  dim3 grid(g.N + 1, BH);  // + the tiling CTA
  if (d == 128 && g.BT == 64) k_kv_image<128, 64><<<grid, 256, 0, st>>>(g, K, V, img, tl);
  else if (d == 128 && g.BT == 32) k_kv_image<128, 32><<<grid, 256, 0, st>>>(g, K, V, img, tl);
  else if (d == 64 && g.BT == 64) k_kv_image<64, 64><<<grid, 256, 0, st>>>(g, K, V, img, tl);
  else if (d == 64 && g.BT == 32) k_kv_image<64, 32><<<grid, 256, 0, st>>>(g, K, V, img, tl);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// Fill (reading C9): O[t] = O^s[donor(t)] for pruned t. One warp per 32 tokens: the lanes read the 32
// donors (coalesced), a ballot gives the pruned ones, and groups of d/8 lanes copy one pruned row each, U rows
// per group in flight (all loads before the stores) -- the one-chunk-per-thread version was latency-bound at
// ~1.4 TB/s (two dependent loads per 16 bytes, half the threads idle on kept rows).
template <int CPR>
__global__ void __launch_bounds__(256) k_fill(int BH, int L, const int* __restrict__ donor, const Rows O) {
  constexpr int RPI = 32 / CPR, U = 4;  // rows per pass of the warp, passes in flight
  const int lane = threadIdx.x & 31;
  const size_t wid = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int wpr = (L + 31) >> 5;  // warps per head
  if (wid >= static_cast<size_t>(BH) * wpr) return;
  const int bh = static_cast<int>(wid / wpr), t0 = static_cast<int>(wid % wpr) * 32;
  const int t = t0 + lane;
  const int dn = t < L ? donor[static_cast<size_t>(bh) * L + t] : t;
  const unsigned mask = __ballot_sync(0xffffffffu, dn != t);
  const int n = __popc(mask), sub = lane / CPR, c = (lane % CPR) * 8;
  bf16* oh = O.head(bh);
  for (int base = 0; base < n; base += RPI * U) {
    uint4 v[U];
    int dst[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int idx = base + k * RPI + sub;
      const int pos = idx < n ? static_cast<int>(__fns(mask, 0, idx + 1)) : 0;
      const int src = __shfl_sync(0xffffffffu, dn, pos);
      dst[k] = idx < n ? t0 + pos : -1;
      if (dst[k] >= 0) v[k] = *reinterpret_cast<const uint4*>(oh + static_cast<size_t>(src) * O.sl + c);
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (dst[k] >= 0) *reinterpret_cast<uint4*>(oh + static_cast<size_t>(dst[k]) * O.sl + c) = v[k];
  }
}

// debug: record the per-step timeline of CTA `cta` into dev_buf ([6][1024] u64), or disable (NULL)
cudaError_t debug_trace_fwd(void* dev_buf, int cta) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_buf);
  cudaError_t e = cudaMemcpyToSymbol(g_fwd_trace, &p, sizeof(p));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_fwd_trace_cta, &cta, sizeof(int));
  return e;
}

cudaError_t launch_fill(int BH, int L, int d, const int* donor, Rows O, cudaStream_t st) {
  const size_t warps = static_cast<size_t>(BH) * ((L + 31) / 32);
  const unsigned grid = static_cast<unsigned>((warps + 7) / 8);
  if (d == 128) k_fill<16><<<grid, 256, 0, st>>>(BH, L, donor, O);
  else if (d == 64) k_fill<8><<<grid, 256, 0, st>>>(BH, L, donor, O);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace bsa
