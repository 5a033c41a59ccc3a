// attn_bwd.cu — a8: backward of the BSA sparse attention with the selection held fixed
// (reading C10; the paper only states that separate backward kernels exist).
//
//   prep    : dO^s[q] = dO[q] + sum of dO over pruned tokens whose donor is q (gradient of the fill,
//             P:155); D[q] = rowsum(dO^s * O^s); dQacc = 0.
//   main    : KV-stationary tcgen05 kernel, one CTA per (b,h, KV block j). It walks k2q[j] (query blocks
//             that admitted j) G blocks at a time: every row of the 128-row M tile belongs to a block
//             that admitted j, so no MMA work is wasted on masking. Per chunk:
//               S  = Q^s K_j^T, dP = dO^s V_j^T            (M=128 queries, N=BT keys)
//               P  = exp(scale S - LSE), dS = P (dP - D)    (thread == query row)
//               dV_j^T += dO^s^T P, dK_j^T += Q^s^T dS      (M=d=128, N=BT, K=128 queries; TMEM-resident)
//               dQ_part = dS K_j                            (M=128, N=d) -> L2 bulk reduce-add
//   finalize: dQ[kept] = scale * dQacc (bf16), dQ[pruned] = 0.
//
// Warp roles of the main kernel (384 threads): w0-3 gradient softmax (thread == query
// row == TMEM lane), w4-7 dQ drain (TMEM -> smem slices -> cp.reduce.async.bulk.tensor into the packed
// fp32 dQacc), w8 TMEM allocator, w9 gradient-MMA issuer (dV, dK, dQ), w10 bulk-copy producer (per query
// block: its QdO image and its LSE/D row statistics), w11 S/dP-MMA issuer. The control roles sit on the
// highest warp ids (the warp arbiter favours them) and suspend on mbarriers rather than spin; two MMA
// issuers with plain blocking waits let S/dP(c+1) run ahead of the gradient MMAs of chunk c by itself.
#include <cmath>
#include "kernels.h"

#ifdef BSA_HANG_DEBUG
namespace bsa {
__device__ unsigned* g_hang_rec = nullptr;
}
// a wait that spun ~forever records (barrier smem address, parity, warp, lane, cta) for the host to read
#define BSA_HANG_RECORD(addr, par)                                                                           \
  do {                                                                                                        \
    unsigned* _r = bsa::g_hang_rec;                                                                           \
    if (_r) {                                                                                                 \
      const unsigned _i = atomicAdd(_r, 1u);                                                                  \
      if (_i < 500u) {                                                                                        \
        unsigned* _e = _r + 8 + 8 * _i;                                                                       \
        _e[0] = (addr); _e[1] = (par); _e[2] = threadIdx.x >> 5; _e[3] = threadIdx.x & 31;                  \
        _e[4] = blockIdx.x; _e[5] = blockIdx.y;                                                               \
        __threadfence_system();                                                                               \
      }                                                                                                       \
    }                                                                                                         \
  } while (0)
#endif
#include "ptx.cuh"

namespace bsa {

bool make_map_2d(CUtensorMap* m, const void* base, int d, size_t rows, int box_rows);

// The backward's waits poll (ptx.cuh mbar_wait_spin) unless built with BSA_BWD_SUSPEND.
__device__ __forceinline__ void bwait(uint64_t* bar, uint32_t parity) {
#ifdef BSA_BWD_SUSPEND
  mbar_wait(bar, parity);
#else
  mbar_wait_spin(bar, parity);
#endif
}
bool make_map_5d(CUtensorMap* m, const void* base, const Geo& g, int d, int heads, long long sl, long long sh);
bool make_map_rows_f32(CUtensorMap* m, const void* base, int d, size_t rows, int box_rows);

__device__ __forceinline__ float ex2b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------------------------------------------ prep
// QdO image of a query block (what one chunk slot of the main kernel reads with ONE bulk copy):
// SR/8 groups of 8 rows; group q holds [Q^s d-half 0][Q^s d-half 1][dO^s d-half 0][dO^s d-half 1], each
// 8 rows x 128 B with the 128-byte swizzle. Consecutive groups (also across the blocks stacked in a
// chunk) are 2*NCB KB apart, so every UMMA operand over the chunk's 128 rows has a uniform stride.
// Next to it, the block's row statistics lsed[(b,h,block)] = [row][LSE*log2(e), D] for its SR rows
// (one more bulk copy per block). Rows beyond the block's kept count are zero with LSE = +inf, D = 0, so
// they contribute P = dS = 0.
//
// One CTA per (b,h, block): the block's tokens, their donors and their dO rows are staged in shared
// memory once (coalesced 16-byte loads), then one warp per kept row folds the dO of the pruned tokens
// whose donor it is (the gradient of the fill), forms D = rowsum(dO^s O^s) and writes its image
// row, row statistics and the zeroed dQ accumulator row.
// Claim order of the persistent main kernel: index order (neighbouring KV blocks of one head run together and
// share their query blocks' images in L2), except that the shortest ~5% of the items (by k2q length, i.e.
// chunk count) are moved to the end, in index order, so the kernel's tail is made of short items. (With items
// claimed in index order the CTAs finished over a 55 us spread at 32k, 2.4% of the SMs' time idle; a full
// longest-first order removed the tail but lost the L2 locality: attn_bwd 1.35 -> 1.51 ms at 32k, 22.4 -> 30.3
// ms at 75k; tools/profiling/bwd_tail.py.) One CTA: a length histogram gives the 5% threshold, then a stable
// partition by chunked ballot scans.
__device__ void build_item_order(const Geo& g, int heads, int b, const int* __restrict__ k2q_num,
                                 int* __restrict__ order, int* hist, int hist_cap /* shared ints */, int short_pct) {
  __shared__ int s_thr, s_nlong, s_w[8][2], s_carry[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, n_items = heads * g.N;
  const int top = g.N < hist_cap ? g.N : hist_cap - 1;  // (lengths >= top share the top bucket)
  const size_t base = static_cast<size_t>(b) * n_items;
  auto bucket = [&](int i) { const int v = k2q_num[base + i]; return v < top ? v : top; };
  for (int v = tid; v <= top; v += blockDim.x) hist[v] = 0;
  if (tid < 2) s_carry[tid] = 0;
  __syncthreads();
  for (int i = tid; i < n_items; i += blockDim.x) atomicAdd(&hist[bucket(i)], 1);
  __syncthreads();
  if (tid == 0) {  // threshold: the smallest length v with at least short_pct % of the items at or below it
    int run = 0, v = 0;
    for (; v < top; ++v) {
      run += hist[v];
      if (run * 100 >= short_pct * n_items) break;
    }
    s_thr = v;
    s_nlong = 0;
  }
  __syncthreads();
  const int thr = s_thr;
  for (int i = tid; i < n_items; i += blockDim.x) atomicAdd(&s_nlong, bucket(i) > thr ? 1 : 0);
  __syncthreads();
  const int nlong = s_nlong;
  for (int i0 = 0; i0 < n_items; i0 += blockDim.x) {  // stable partition: long items first, then short ones
    const int i = i0 + tid;
    const bool valid = i < n_items, is_long = valid && bucket(i) > thr;
    const unsigned bl = __ballot_sync(0xffffffffu, is_long), bs = __ballot_sync(0xffffffffu, valid && !is_long);
    if (lane == 0) { s_w[warp][0] = __popc(bl); s_w[warp][1] = __popc(bs); }
    __syncthreads();
    if (valid) {
      const int k = is_long ? 0 : 1;
      int pos = s_carry[k] + __popc((is_long ? bl : bs) & ((1u << lane) - 1u));
      for (int w = 0; w < warp; ++w) pos += s_w[w][k];
      order[base + (is_long ? pos : nlong + pos)] = i;
    }
    __syncthreads();
    if (tid < 2)
      for (int w = 0; w < 8; ++w) s_carry[tid] += s_w[w][tid];
    __syncthreads();
  }
}

template <int D>
__global__ void __launch_bounds__(256) k_bwd_prep(Geo g, int BH, int Lq, int SR, const int* __restrict__ kept_off,
                                                  const int* __restrict__ kept_tok, const int* __restrict__ donor,
                                                  const bf16* __restrict__ Qs, const Rows dO, const Rows O,
                                                  const float* __restrict__ lse,
                                                  uint8_t* __restrict__ qdo_img, float* __restrict__ lsed,
                                                  float* __restrict__ dQacc, const int* __restrict__ pair_total,
                                                  long long ds_cap, const Rows dQ, const int* __restrict__ k2q_num,
                                                  int* __restrict__ item_order, int launch_heads, int short_pct) {
  constexpr int PER = D / 32;  // channels per lane (4 or 2)
  constexpr int NCB = D / 64;
  constexpr int MAXT = 128;    // tokens per block (checked by the API)
  __shared__ __align__(16) bf16 s_do[MAXT * D];
  __shared__ int s_tok[MAXT], s_don[MAXT];
  const int blk = blockIdx.x, bh = blockIdx.y;
  if (blk == g.N) {  // the extra CTAs: the main kernel's claim order of launch bh (if there is one)
    if (bh < BH / launch_heads)
      build_item_order(g, launch_heads, bh, k2q_num, item_order, reinterpret_cast<int*>(s_do), MAXT * D / 2,
                       short_pct);
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t bi = static_cast<size_t>(bh) * g.N + blk;
  const size_t head = static_cast<size_t>(bh) * g.L;
  const bf16* doh = dO.head(bh);
  const bf16* oh = O.head(bh);
  const Box x = block_box(g, blk);
  const int n = box_size(x);
  const int ko = kept_off[blk], nk = kept_off[blk + 1] - ko;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int t = box_token(g, x, i);
    s_tok[i] = t;
    s_don[i] = donor[head + t];
  }
  __syncthreads();
  // dS path (pair_total == NULL: reduce path chosen on the host): no fp32 dQ accumulator to clear, and the
  // pruned rows of dQ are zeroed here (on the reduce path k_bwd_finalize writes every row)
  const bool ds = pair_total != nullptr && *pair_total <= ds_cap;
  bf16* dqh = dQ.head(bh);
  for (int v = threadIdx.x; v < n * (D / 8); v += blockDim.x) {
    const int i = v / (D / 8), c = (v % (D / 8)) * 8;
    *reinterpret_cast<uint4*>(s_do + i * D + c) = *reinterpret_cast<const uint4*>(doh + s_tok[i] * dO.sl + c);
    if (ds && s_don[i] != s_tok[i])  // dQ of a pruned token is 0 (reading C10)
      *reinterpret_cast<uint4*>(dqh + s_tok[i] * dQ.sl + c) = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const int ch0 = lane * PER;
  for (int lr = warp; lr < SR; lr += 8) {
    uint8_t* gbase = qdo_img + bi * static_cast<size_t>(SR) * D * 4 + (lr >> 3) * (2 * NCB * 1024);
    const uint32_t inrow = sw128_off(lr & 7, (ch0 & 63) >> 3) + (ch0 & 7) * 2;
    uint8_t* qdst = gbase + (ch0 >> 6) * 1024 + inrow;
    uint8_t* ddst = gbase + (NCB + (ch0 >> 6)) * 1024 + inrow;
    float* ld = lsed + bi * 2 * SR + 2 * lr;  // [row][LSE * log2 e, D]: a block prefix is one contiguous copy
    if (lr >= nk) {
      if (lane == 0) {
        ld[0] = INFINITY;
        ld[1] = 0.f;
      }
      if (PER == 4) {
        *reinterpret_cast<uint2*>(qdst) = make_uint2(0, 0);
        *reinterpret_cast<uint2*>(ddst) = make_uint2(0, 0);
      } else {
        *reinterpret_cast<uint32_t*>(qdst) = 0u;
        *reinterpret_cast<uint32_t*>(ddst) = 0u;
      }
      continue;
    }
    const size_t prow = static_cast<size_t>(bh) * Lq + ko + lr;
    const int tok = kept_tok[prow];
    if (PER == 4) *reinterpret_cast<uint2*>(qdst) = *reinterpret_cast<const uint2*>(Qs + prow * D + ch0);
    else *reinterpret_cast<uint32_t*>(qdst) = *reinterpret_cast<const uint32_t*>(Qs + prow * D + ch0);
    // dO^s = dO[tok] + sum of dO over the block's pruned tokens whose donor is tok (ascending token order)
    float acc[PER];
    int self = -1;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const bool is_self = i < n && s_tok[i] == tok;
      const unsigned ms = __ballot_sync(0xffffffffu, is_self);
      if (ms) self = i0 + __ffs(ms) - 1;
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = __bfloat162float(s_do[self * D + ch0 + e]);
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      const bool match = i < n && s_tok[i] != tok && s_don[i] == tok;
      unsigned m = __ballot_sync(0xffffffffu, match);
      while (m) {
        const int src = i0 + __ffs(m) - 1;
        m &= m - 1;
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[e] += __bfloat162float(s_do[src * D + ch0 + e]);
      }
    }
    float dsum = 0.f;
    const bf16* orow = oh + tok * O.sl + ch0;
    bf16 hv[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      hv[e] = __float2bfloat16_rn(acc[e]);
      dsum += __bfloat162float(hv[e]) * __bfloat162float(orow[e]);
    }
    if (PER == 4) *reinterpret_cast<uint2*>(ddst) = *reinterpret_cast<const uint2*>(hv);
    else *reinterpret_cast<uint32_t*>(ddst) = *reinterpret_cast<const uint32_t*>(hv);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
    if (lane == 0) {
      ld[0] = lse[prow] * 1.4426950408889634f;
      ld[1] = dsum;
    }
    if (!ds) {
      float* dq = dQacc + prow * D + ch0;
      if (PER == 4) *reinterpret_cast<float4*>(dq) = make_float4(0.f, 0.f, 0.f, 0.f);
      else *reinterpret_cast<float2*>(dq) = make_float2(0.f, 0.f);
    }
  }
}

// ------------------------------------------------------------------------------------ main
// Debug-only timeline of one CTA (bsa_debug_trace_bwd; null in production).
__device__ unsigned long long* g_bwd_trace = nullptr;
__device__ int g_bwd_trace_cta = 0;
#ifdef BSA_TRACE
#define BWD_TRACE(slot, u)                                                                              \
  do {                                                                                                  \
    unsigned long long* _t = g_bwd_trace;                                                               \
    if (_t != nullptr && (int)(blockIdx.y * gridDim.x + blockIdx.x) == g_bwd_trace_cta && (u) < 1024) \
      _t[(slot) * 1024 + (u)] = clock64();                                                              \
  } while (0)
#define CTA_STAMP(k)                                                                                   \
  do {                                                                                                 \
    if (g_bwd_trace != nullptr && g_bwd_trace_cta == -1) {                                             \
      unsigned long long _g;                                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g));                                          \
      g_bwd_trace[16 * static_cast<size_t>(blockIdx.y * gridDim.x + blockIdx.x) + (k)] = _g;           \
    }                                                                                                  \
  } while (0)
#else
#define BWD_TRACE(slot, u) \
  do {                     \
  } while (0)
#define CTA_STAMP(k) \
  do {               \
  } while (0)
#endif

// Debug-only progress counters (BSA_PROGRESS builds): per CTA 16 words in host-mapped memory, written with
// volatile stores so the host can read where every role stands while the kernel runs (hang diagnosis).
__device__ unsigned* g_bwd_prog = nullptr;
#ifdef BSA_PROGRESS
#define PROG(slot, v)                                                                                      \
  do {                                                                                                     \
    unsigned* _p = g_bwd_prog;                                                                             \
    if (_p) *reinterpret_cast<volatile unsigned*>(_p + 16 * (blockIdx.y * gridDim.x + blockIdx.x) + (slot)) = (v); \
  } while (0)
#else
#define PROG(slot, v) \
  do {                \
  } while (0)
#endif

struct BwdParams {
  const uint8_t* qdo_img;  // per query block Q^s|dO^s images (k_bwd_prep), SR*d*4 bytes each
  CUtensorMap mK;    // 5D block map
  CUtensorMap mV;
  CUtensorMap mDQ;     // dQacc [BH*Lq, d] fp32, box {32 columns, 32 rows}, 128B swizzle (bulk reduce-add target)
  CUtensorMap mDQh;    // the same with 16 and 8 rows per box (pieces of blocks that keep fewer rows)
  CUtensorMap mDQq;
  CUtensorMap mdK;     // 5D block maps over the dK / dV outputs (TMA store of the finished block)
  CUtensorMap mdV;
  Geo g;
  const float* lsed;   // per query block [SR rows][LSE*log2e, D] (k_bwd_prep)
  int Lq, SR, G;
  const int* kept_off;
  const int* k2q_num;
  const int* k2q_idx;
  float* dQacc;
  int bh0;             // first (b,h) of this launch: hc + bh0 indexes the internal buffers, hc (item / N) is the
                       // head coordinate of the K/V/dK/dV tensor maps
  int items;           // work items of this launch: heads x N KV blocks, item = hc * N + j
  int* work_ctr;       // next unclaimed item (zeroed before the launch)
  const int* item_order;  // [launch][items] claim order (build_item_order), or NULL: index order
  float scale_log2;
  float scale;
  // dS path (DESIGN.md §5 "Backward"): when the selection's admitted (query block, KV block) pairs fit the
  // workspace (*pair_total <= ds_cap), the main kernel stores each pair's bf16 dS tile (SR rows x 128 B, the
  // swizzled shared-memory image) at ds_buf + k2q_slot[..] * SR * 128 and k_bwd_dq forms dQ from them; else the
  // main kernel reduces fp32 dQ partials into dQacc (reduce path) and k_bwd_finalize converts them.
  const int* pair_total;
  long long ds_cap;
  const int* k2q_slot;  // [BH][N][N]: pair slot of k2q entry (j, p) (k_pair_slot)
  uint8_t* ds_buf;
};

// dQ staging: 2 slots of 32 rows per drain warp (one 4 KB reduce box per 32-column slice when SR >= 32): half the
// reduce operations of 16-row boxes for the same bytes, attn_bwd 1.70 -> 1.47 ms at 32k
#ifndef BSA_DQ_SLOT_ROWS
#define BSA_DQ_SLOT_ROWS 32
#endif
#ifndef BSA_DQ_SLOTS
#define BSA_DQ_SLOTS 2
#endif
constexpr int BWD_THREADS = 384;
constexpr int BWD_MAX_G = 16;

template <int D, int BT, bool DS = false>
struct BwdSmem {
  static constexpr int NCB = D / 64;
  static constexpr int KV_BYTES = BT * D * 2;
  static constexpr int TILE_BYTES = 128 * D * 2;            // Q^s or dO^s rows of one chunk
  static constexpr int PG = 2 * NCB * 1024;                 // stride of 8-row groups in a QdO image
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES + 1024;  // QdO images of the chunk's blocks + their lsed
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KV_BYTES;
  static constexpr int OFF_ST = OFF_V + KV_BYTES;           // 2 stages
  static constexpr int OFF_P = OFF_ST + 2 * STAGE_BYTES;    // [128][64] bf16
  static constexpr int OFF_DS = OFF_P + 16384;
  static constexpr int OFF_ZERO = OFF_DS + 16384;           // d=64 only: zero MN chunk for M=128 padding
  // dQ staging per drain warp: DQ_SLOTS slots of DQ_SROWS rows x 32 fp32 (128B-swizzled, the reduce map's box)
  static constexpr int DQ_SROWS = BSA_DQ_SLOT_ROWS;
  static constexpr int DQ_SLOTS = BSA_DQ_SLOTS;
  static constexpr int DQ_SLOT_BYTES = DQ_SROWS * 128;
  static constexpr int OFF_DQS = OFF_ZERO + (D == 64 ? 16384 : 0);
  // the dynamic region is declared 1024-byte aligned (checked at run time), so no alignment slack is added
  // dS path: no dQ staging; the chunk ring's pair slots sit there instead
  static constexpr int OFF_SLOT = OFF_DQS;
  static constexpr int TOTAL = OFF_DQS + (DS ? 4 * 16 * 4 : 4 * DQ_SLOTS * DQ_SLOT_BYTES);
  static constexpr int TMEM_COLS = (4 * BT + 2 * D) <= 256 ? 256 : 512;
};

// Persistent CTAs (one per SM): the producer warp claims KV blocks (items over all heads of the launch) with
// an atomic counter and publishes them through a ring in shared memory; every role walks the same item
// sequence with all barrier phases counted across items (chunk counter c runs over all of the CTA's chunks).
// So the dQ drain of a block's last chunks, its dK/dV epilogue and the next block's K/V load overlap the next
// block's first chunks, the CTA prologue (barrier init, TMEM allocation, stage zeroing) is paid once per SM,
// and dynamic claiming bounds the tail by one block (fixed runs of 2 / 4 / 8 / 16 consecutive blocks per CTA
// measured 1.71 / 1.72 / 1.82 / 1.97 ms at 32k: tail imbalance of static assignment).
constexpr int ITEM_RING = 8;
// readers of the item ring: S/dP issuer, gradient issuer, 4 softmax warps (+ 4 dQ drain warps on the reduce path)
template <bool DS>
__host__ __device__ constexpr int item_readers() { return DS ? 6 : 10; }
// rows a query block with nk kept queries takes in a chunk: nk rounded up to a power of two >= 8 (<= SR)
__device__ __forceinline__ int slot_size(int nk, int SR) {
  int sz = 8;
  while (sz < nk && sz < SR) sz <<= 1;
  return sz;
}

template <int D, int BT, bool DS>
__global__ void __launch_bounds__(BWD_THREADS, 1) k_attn_bwd(const __grid_constant__ BwdParams p) {
  using SM = BwdSmem<D, BT, DS>;
  // one of the two instantiations runs: the dS path when the pairs fit, else the reduce path (uniform exit)
  if (DS != (p.pair_total != nullptr && *p.pair_total <= p.ds_cap)) return;
  constexpr int NCB = SM::NCB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  if (threadIdx.x == 0 && (smem_u32(smem_raw) & 1023u) != 0u) __trap();  // SW128 tiles need 1024-byte alignment
  uint8_t* sK = sm + SM::OFF_K;
  uint8_t* sV = sm + SM::OFF_V;
  uint8_t* sP = sm + SM::OFF_P;
  uint8_t* sdS = sm + SM::OFF_DS;
  auto stage_q = [&](int s) { return sm + SM::OFF_ST + s * SM::STAGE_BYTES; };  // Q^s d-half 0 of group 0
  auto stage_do = [&](int s) { return sm + SM::OFF_ST + s * SM::STAGE_BYTES + NCB * 1024; };
  auto stage_ld = [&](int s) {  // [LSE*log2e, D] of the chunk's 128 rows (row r at 2 r)
    return reinterpret_cast<float*>(sm + SM::OFF_ST + s * SM::STAGE_BYTES + 2 * SM::TILE_BYTES);
  };

  __shared__ __align__(8) uint64_t bar_kv, bar_c_full[2], bar_c_empty[2], bar_sd_full, bar_sd_free, bar_ps_full,
      bar_ps_free, bar_dq_full[2], bar_dq_free[2], bar_acc, bar_acc_free, bar_item_full[ITEM_RING],
      bar_item_empty[ITEM_RING];
  __shared__ int s_item[ITEM_RING];
  __shared__ uint32_t s_tmem;
  // Chunk metadata ring (first packed row, kept count, block id of each slot; row -1 = empty slot), written
  // by the producer for chunk c into entry c & 3. Four deep: the producer rewrites an entry only after
  // the MMAs of chunk c-2 completed, by which time the softmax and drain warps are done with chunk c-4.
  // Chunk composition ring (entry c & 3 for chunk c, written by the producer): per query block e of the chunk its
  // first packed row (dQacc row) s_row0 and kept count | chunk row offset << 8 in s_nk; s_cinfo = number of
  // blocks | (last chunk of its KV block) << 8. Blocks are packed into the 128 rows by slot size (SR rounded
  // down to what they keep: 32 / 16 / 8 rows at r = 0.5), first fit on 8-row-group boundaries.
  __shared__ int s_row0[4][BWD_MAX_G], s_nk[4][BWD_MAX_G], s_cinfo[4];

  const Geo& g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = p.G, SR = p.SR;
  // per KV block (hc, j): admitting query blocks, rotation of the chunk order (concurrent CTAs start on
  // different query blocks: no L2 hot spot)
  auto nq_of = [&](int bh, int j) { return p.k2q_num[static_cast<size_t>(bh) * g.N + j]; };
  auto rot_of = [&](int bh, int j, int nch) {
    return nch > 0 ? static_cast<int>((static_cast<unsigned>(j) * 2654435761u + bh * 40503u) % nch) : 0;
  };
  // item `it` of this CTA (-1: no work left); every reader hands its ring slot back after reading it
  auto read_item = [&](int it) {
    const int s = it % ITEM_RING;
    bwait(&bar_item_full[s], (it / ITEM_RING) & 1);
    const int v = s_item[s];
    __syncwarp();
    if (lane == 0) mbar_arrive(&bar_item_empty[s]);
    return v;
  };

#ifdef BSA_TRACE
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
#ifdef BSA_HANG_DEBUG
  if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0 && g_hang_rec) {
    unsigned* m = g_hang_rec + 8 + 8 * 500;
    m[0] = smem_u32(&bar_kv); m[1] = smem_u32(&bar_c_full[0]); m[2] = smem_u32(&bar_c_full[1]);
    m[3] = smem_u32(&bar_c_empty[0]); m[4] = smem_u32(&bar_c_empty[1]); m[5] = smem_u32(&bar_sd_full);
    m[6] = smem_u32(&bar_sd_free); m[7] = smem_u32(&bar_ps_full); m[8] = smem_u32(&bar_ps_free);
    m[9] = smem_u32(&bar_dq_full[0]); m[10] = smem_u32(&bar_dq_full[1]); m[11] = smem_u32(&bar_dq_free[0]);
    m[12] = smem_u32(&bar_dq_free[1]); m[13] = smem_u32(&bar_acc); m[14] = smem_u32(&bar_acc_free);
  }
#endif
  if (tid == 0) {
    mbar_init(&bar_kv, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_c_full[s], 1);
      mbar_init(&bar_c_empty[s], 1);
      mbar_init(&bar_dq_full[s], 1);
      mbar_init(&bar_dq_free[s], 128);
    }
    mbar_init(&bar_sd_full, 1);
    mbar_init(&bar_sd_free, 128);
    mbar_init(&bar_ps_full, 128);
    mbar_init(&bar_ps_free, 1);
    mbar_init(&bar_acc, 1);
    mbar_init(&bar_acc_free, 128);
    for (int s = 0; s < ITEM_RING; ++s) {
      mbar_init(&bar_item_full[s], 1);
      mbar_init(&bar_item_empty[s], item_readers<DS>());
    }
    fence_mbar_init();
  }
  // Warp roles (the warp arbiter favours higher ids, so the single-thread producer and MMA roles get the
  // highest ones and are not starved by the math warps sharing their sub-partition):
  // w0-3 gradient softmax + dK/dV epilogue (TMEM quadrant = warp), w4-7 dQ drain (quadrant = warp - 4),
  // w8 TMEM allocator, w9 gradient-MMA issuer, w10 producer, w11 S/dP-MMA issuer.
  constexpr int W_ALLOC = 8, W_B = 9, W_PROD = 10, W_SD = 11;
  if (warp == W_ALLOC) tmem_alloc(&s_tmem, SM::TMEM_COLS);
  // zero both stages once (rows of unused slots must be finite: they meet P = dS = 0 in the MMAs; after a
  // stage's first fill its stale rows stay finite)
  for (int o = tid * 16; o < 2 * SM::STAGE_BYTES; o += BWD_THREADS * 16)
    *reinterpret_cast<uint4*>(sm + SM::OFF_ST + o) = make_uint4(0, 0, 0, 0);
  if (D == 64)
    for (int o = tid * 16; o < 16384; o += BWD_THREADS * 16)
      *reinterpret_cast<uint4*>(sm + SM::OFF_ZERO + o) = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = s_tmem;
  // TMEM columns: S, dP, dV^T, dK^T, dQ of chunk parity 0, dQ of parity 1
  const uint32_t tS = tbase, tdP = tbase + BT, tdV = tbase + 2 * BT, tdK = tbase + 3 * BT, tdQ = tbase + 4 * BT;
  if (tid == 0) CTA_STAMP(4);

  if (warp == W_PROD) {
    // ============================ producer (lane 0 claims items and issues TMA; all lanes fetch metadata)
    int c = 0;  // global chunk counter
    for (int it = 0;; ++it) {
      if (lane == 0) {  // claim the next item and publish it once every reader released the slot's last use
        const int rs = it % ITEM_RING;
        if (it >= ITEM_RING) bwait(&bar_item_empty[rs], ((it / ITEM_RING) - 1) & 1);
        const int v = atomicAdd(p.work_ctr, 1);
        s_item[rs] = v >= p.items ? -1 : (p.item_order ? p.item_order[static_cast<size_t>(p.bh0) * g.N + v] : v);
        mbar_arrive(&bar_item_full[rs]);
      }
      __syncwarp();
      const int item = s_item[it % ITEM_RING];
      if (item < 0) break;
      const int hc = item / g.N, j = item - hc * g.N, bh = p.bh0 + hc;
      const int nq = nq_of(bh, j);
      if (nq == 0) continue;
      const int* qlist = p.k2q_idx + (static_cast<size_t>(bh) * g.N + j) * g.N;
      const uint32_t blk_bytes = static_cast<uint32_t>(SR * D * 4);
      // k2q[j] is consumed in order: lane l of the fetched window holds entry w0 + l (block, kept offset, count)
      int t = 0, w0 = -64, wqb = 0, wko = 0, wnk = 0;
      for (bool last = false; !last; ++c) {
        const int s = c & 1, ring = c & 3;
        // compose chunk c first (lane e holds its entry e), then wait for the stage and publish: the list reads
        // overlap the wait
        uint32_t used = 0u;  // 8-row groups of the chunk already taken
        int ne = 0, e_qb = -1, e_roff = 0, e_sz = 0, e_t = 0, e_row0 = 0, e_nk = 0;
        while (t < nq && ne < BWD_MAX_G) {
          if (t >= w0 + 32) {  // next window of 32 list entries, fetched in parallel
            w0 = t;
            const int pos = t + lane;
            if (pos < nq) {
              wqb = qlist[pos];
              wko = p.kept_off[wqb];
              wnk = p.kept_off[wqb + 1] - wko;
            }
          }
          const int l = t - w0;
          const int nk = __shfl_sync(0xffffffffu, wnk, l);
          const int sz = slot_size(nk, SR), ng = sz >> 3;
          const uint32_t pat = (1u << ng) - 1u;
          int o = 0;
          while (o + ng <= 16 && (used & (pat << o))) o += ng;
          if (o + ng > 16) break;  // no aligned room left: the chunk is full
          used |= pat << o;
          const int qb = __shfl_sync(0xffffffffu, wqb, l), ko = __shfl_sync(0xffffffffu, wko, l);
          if (lane == ne) {
            e_qb = qb;
            e_roff = 8 * o;
            e_sz = sz;
            e_t = t;
            e_row0 = bh * p.Lq + ko;
            e_nk = nk;
          }
          ++ne;
          ++t;
        }
        last = t >= nq;
        int e_slot = -1;
        if (DS && e_qb >= 0) e_slot = p.k2q_slot[(static_cast<size_t>(bh) * g.N + j) * g.N + e_t];
        if (lane == 0) PROG(0, c * 4 + 0);
        bwait(&bar_c_empty[s], ((c >> 1) & 1) ^ 1);
        if (lane == 0) PROG(0, c * 4 + 1);
        if (lane < ne) {
          s_row0[ring][lane] = e_row0;
          s_nk[ring][lane] = e_nk | (e_roff << 8);
          if (DS) reinterpret_cast<int*>(sm + SM::OFF_SLOT)[ring * 16 + lane] = e_slot;
        }
        if (lane == 0) s_cinfo[ring] = ne | (last ? 256 : 0);
        // per block: its first sz rows of the QdO image (8-row groups) and of the [LSE, D] row statistics
        uint32_t bytes = e_qb >= 0 ? static_cast<uint32_t>(e_sz / 8) * SM::PG + 8u * e_sz : 0u;
#pragma unroll
        for (int x = 16; x > 0; x >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, x);
        __syncwarp();
        if (lane == 0) {
          mbar_expect_tx(&bar_c_full[s], bytes);
          BWD_TRACE(0, c);
          if (c == 0) CTA_STAMP(11);
        }
        __syncwarp();
        if (e_qb >= 0) {
          const size_t qimg = static_cast<size_t>(bh) * g.N + e_qb;
          bulk_load(stage_q(s) + (e_roff >> 3) * SM::PG, p.qdo_img + qimg * blk_bytes,
                    static_cast<uint32_t>(e_sz / 8) * SM::PG, &bar_c_full[s]);
          bulk_load(stage_ld(s) + 2 * e_roff, p.lsed + qimg * 2 * SR, 8u * e_sz, &bar_c_full[s]);
        }
        __syncwarp();
      }
    }
  } else if (warp == W_SD || warp == W_B) {
    // ============================ MMA issuer: whole warp walks the schedule (uniform registers), one
    // elected lane issues. Descriptors are precomputed bases advanced by (byte offset >> 4).
    const bool leader = elect_one();
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, BT, 0, 0);  // Q K^T / dO V^T
    constexpr uint32_t idesc_t = umma_idesc_bf16(128, BT, 1, 1);  // dO^T P / Q^T dS (M = d padded to 128)
    constexpr uint32_t idesc_q = umma_idesc_bf16(128, D, 0, 1);   // dS K
    const uint32_t zero = smem_u32(sm + SM::OFF_ZERO);
    // K-major A over the chunk's 128 rows: 8-row groups SM::PG apart (QdO image layout)
    const uint64_t dQa = umma_desc_sw128(smem_u32(stage_q(0)), 16, SM::PG);
    const uint64_t dDa = umma_desc_sw128(smem_u32(stage_do(0)), 16, SM::PG);
    // MN-major A over d (K = query rows, 16 per step = two 8-row groups, SBO = SM::PG); the second
    // 64-channel chunk sits LBO = 1 KB after the first (d = 128)
    const uint64_t dQt = umma_desc_sw128(smem_u32(stage_q(0)), 1024, SM::PG);
    const uint64_t dDt = umma_desc_sw128(smem_u32(stage_do(0)), 1024, SM::PG);
    const uint64_t dK = umma_desc_sw128(smem_u32(sK), 16, 1024), dV = umma_desc_sw128(smem_u32(sV), 16, 1024);
    const uint64_t dKt = umma_desc_sw128(smem_u32(sK), BT * 128, 1024);
    const uint64_t dP = umma_desc_sw128(smem_u32(sP), 8192, 1024), dS = umma_desc_sw128(smem_u32(sdS), 8192, 1024);
    const uint64_t dSa = umma_desc_sw128(smem_u32(sdS), 16, 1024);
    int c = 0, nacc = 0;
    for (int it = 0;; ++it) {
      const int item = read_item(it);
      if (item < 0) break;
      const int hc = item / g.N, j = item - hc * g.N, bh = p.bh0 + hc;
      if (nq_of(bh, j) == 0) continue;
      if (warp == W_SD) {
        // K/V tiles of the block: the previous block's are read until its last MMA (bar_acc)
        if (leader) {
          if (nacc > 0) bwait(&bar_acc, (nacc - 1) & 1);
          const int bt = j / (g.Nh * g.Nw), bhh = (j / g.Nw) % g.Nh, bw = j % g.Nw;
          mbar_expect_tx(&bar_kv, 2 * SM::KV_BYTES);
          for (int cb = 0; cb < NCB; ++cb) {
            tma_load_5d(sK + cb * BT * 128, &p.mK, &bar_kv, cb * 64, bw * g.cw, bhh * g.ch, bt * g.ct, hc);
            tma_load_5d(sV + cb * BT * 128, &p.mV, &bar_kv, cb * 64, bw * g.cw, bhh * g.ch, bt * g.ct, hc);
          }
        }
        __syncwarp();
        if (lane == 0) PROG(9, 1000 + nacc);
        bwait(&bar_kv, nacc & 1);
        if (lane == 0) PROG(9, 2000 + nacc);
        // S/dP(v) = Q^s K^T, dO^s V^T of chunk v, issued as soon as its stage landed and the softmax
        // warps hold S/dP(v-1) in registers (single TMEM buffer)
        for (bool last = false; !last; ++c) {
          const int sv = c & 1;
          const uint32_t sov = (sv * SM::STAGE_BYTES) >> 4;  // stage offset in descriptor units
          if (lane == 0) PROG(1, c * 4 + 0);
          bwait(&bar_c_full[sv], (c >> 1) & 1);
          last = (s_cinfo[c & 3] >> 8) & 1;
          BWD_TRACE(11, c);
          if (lane == 0) PROG(1, c * 4 + 1);
          if (c >= 1) bwait(&bar_sd_free, (c - 1) & 1);
          if (lane == 0) PROG(1, c * 4 + 2);
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const int cb = kk >> 2, ko = (kk & 3) * 32;
#ifndef BSA_ABLATE_BWD_MMA
              umma_ss(tS, dQa + sov + ((cb * 1024 + ko) >> 4), dK + ((cb * BT * 128 + ko) >> 4), idesc_s, kk > 0);
              umma_ss(tdP, dDa + sov + ((cb * 1024 + ko) >> 4), dV + ((cb * BT * 128 + ko) >> 4), idesc_s, kk > 0);
#endif
            }
            umma_commit(&bar_sd_full);
          }
          __syncwarp();
          BWD_TRACE(1, c);
        }
      } else {
        // gradient MMAs of chunk c once P/dS(c) is in smem and the drain emptied dQ buffer c & 1. S/dP(c)
        // (the other issuer) completed before P/dS(c) could exist, so the c_empty commit below covers
        // every read of the stage. The first chunk of a block overwrites dV/dK: the epilogue of the
        // previous block must have read them (bar_acc_free).
        if (lane == 0) PROG(10, 1000 + nacc);
        if (nacc > 0) bwait(&bar_acc_free, (nacc - 1) & 1);
        if (lane == 0) PROG(10, 2000 + nacc);
        int cl = 0;  // chunk of this KV block (its first gradient MMAs overwrite dV / dK)
        for (bool last = false; !last; ++c, ++cl) {
          const int s = c & 1, qbuf = c & 1;
          const uint32_t so = (s * SM::STAGE_BYTES) >> 4;
          if (lane == 0) PROG(2, c * 4 + 0);
          bwait(&bar_ps_full, c & 1);
          last = (s_cinfo[c & 3] >> 8) & 1;
          if (lane == 0) PROG(2, c * 4 + 1);
          if (!DS && c >= 2) bwait(&bar_dq_free[qbuf], ((c - 2) >> 1) & 1);  // drain has read dQ(c-2) from TMEM
          if (lane == 0) PROG(2, c * 4 + 2);
          tc_fence_after();
          BWD_TRACE(2, c);
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {  // K = 128 query rows
              const uint32_t ko = (kk * 2 * SM::PG) >> 4;
              uint64_t aq, ad;
              if (D == 128) {
                aq = dQt + so + ko;
                ad = dDt + so + ko;
              } else {  // d = 64: the missing second d-chunk reads the zero block
                const uint32_t qk = smem_u32(stage_q(s)) + kk * 2 * SM::PG, dk = smem_u32(stage_do(s)) + kk * 2 * SM::PG;
                aq = umma_desc_sw128(qk, zero - qk, SM::PG);
                ad = umma_desc_sw128(dk, zero - dk, SM::PG);
              }
#ifndef BSA_ABLATE_BWD_MMA
              umma_ss(tdV, ad, dP + ((kk * 2048) >> 4), idesc_t, (cl > 0 || kk > 0) ? 1u : 0u);
              umma_ss(tdK, aq, dS + ((kk * 2048) >> 4), idesc_t, (cl > 0 || kk > 0) ? 1u : 0u);
#endif
            }
            umma_commit(&bar_c_empty[s]);  // the stage is free once dV/dK have read it
            if (!DS) {
#pragma unroll
              for (int kk = 0; kk < BT / 16; ++kk) {
#ifndef BSA_ABLATE_BWD_MMA
                umma_ss(tdQ + qbuf * D, dSa + ((kk * 32) >> 4), dKt + ((kk * 2048) >> 4), idesc_q, kk > 0);
#endif
              }
              umma_commit(&bar_dq_full[qbuf]);
            }
            umma_commit(&bar_ps_free);
          }
          __syncwarp();
          BWD_TRACE(3, c);
        }
        if (leader) umma_commit(&bar_acc);  // after the block's last gradient MMA: all its MMAs are done
        __syncwarp();
      }
      ++nacc;
    }
  } else if (warp < 4) {
    // ============================ gradient softmax (thread == query row == TMEM lane) + dK/dV epilogue
    const int q4 = warp;
    const int row = q4 * 32 + lane;
    const uint32_t trow = tbase + (static_cast<uint32_t>(q4 * 32) << 16);
    // Key columns of a ragged block past its extent need no mask here: their K/V rows arrive as zeros
    // (TMA out-of-grid fill), so they add nothing to dQ = dS K, and their dK/dV columns are never stored.
    const float sl2 = p.scale_log2;
    const uint32_t sP_u = smem_u32(sP) + row * 128, sdS_u = smem_u32(sdS) + row * 128;
    int c = 0, nacc = 0;
    bool store_pending = false;  // a dK/dV TMA store still reading sP/sdS (issued by row 0)
    for (int it = 0;; ++it) {
      const int item = read_item(it);
      if (item < 0) break;
      // only `item` stays live across the chunk loop (the block coordinates are re-derived for the store)
      const bool any_chunk = p.k2q_num[static_cast<size_t>(p.bh0) * g.N + item] > 0;
      for (bool last = !any_chunk; any_chunk;) {
        const int s = c & 1;
        if (row == 0) PROG(3, c * 8 + 0);
        bwait(&bar_c_full[s], (c >> 1) & 1);
        if (row == 0) PROG(3, c * 8 + 1);
        if (row == 0 && c == 0) CTA_STAMP(8);
        const int cinfo = s_cinfo[c & 3], ne = cinfo & 255;
        last = (cinfo >> 8) & 1;
        bool valid = false;  // this row belongs to a block of the chunk and is one of its kept rows
        for (int e = 0; e < ne; ++e) {
          const int v = s_nk[c & 3][e], roff = v >> 8, nk = v & 255;
          if (row >= roff && row < roff + nk) valid = true;
        }
        const float nl = valid ? -stage_ld(s)[2 * row] : -INFINITY;  // invalid rows: P = dS = 0
        const float Dq = valid ? stage_ld(s)[2 * row + 1] : 0.f;
        bwait(&bar_sd_full, c & 1);
        if (row == 0) PROG(3, c * 8 + 2);
        tc_fence_after();
        if (row == 0) BWD_TRACE(4, c);
        if (row == 0 && c == 0) CTA_STAMP(9);
        // the whole S/dP row goes to registers first, so the TMEM buffer is handed back to the MMA warp
        // (S/dP of the next chunk) before any math
        float sv[BT], dp[BT];
#pragma unroll
        for (int c16 = 0; c16 < BT; c16 += 16) {
          tmem_ld16(trow + c16, sv + c16);
          tmem_ld16(trow + BT + c16, dp + c16);
        }
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bar_sd_free);
        if (row == 0) BWD_TRACE(8, c);
#pragma unroll
        for (int cc = 0; cc < BT; ++cc) {
          const float pr = ex2b(fmaf(sv[cc], sl2, nl));
          sv[cc] = pr;
          dp[cc] = pr * (dp[cc] - Dq);
        }
        if (row == 0) BWD_TRACE(9, c);
        if (row == 0) PROG(3, c * 8 + 3);
        if (c >= 1) bwait(&bar_ps_free, (c - 1) & 1);  // MMAs of chunk c-1 done with sP/sdS
        if (DS) {  // this warp's dS store of chunk c-1 has read its sdS rows
          if (lane == 0) bulk_wait_group_read<0>();
          __syncwarp();
        }
        if (row == 0) PROG(3, c * 8 + 4);
        if (store_pending) {  // the previous block's dK/dV store must have read sP/sdS
          if (row == 0) bulk_wait_group_read<0>();
          named_bar_sync(1, 128);
          store_pending = false;
        }
        if (row == 0) PROG(3, c * 8 + 5);
        if (row == 0) BWD_TRACE(10, c);
#pragma unroll
        for (int c8 = 0; c8 < BT / 8; ++c8) {
          const uint32_t off = ((static_cast<uint32_t>(c8) ^ (row & 7)) << 4);
          const float* a = sv + c8 * 8;
          const float* b = dp + c8 * 8;
          sts128(sP_u + off, pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
          sts128(sdS_u + off, pack_bf16(b[0], b[1]), pack_bf16(b[2], b[3]), pack_bf16(b[4], b[5]), pack_bf16(b[6], b[7]));
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bar_ps_full);
        if (DS) {
          // this warp's 32 dS rows -> the pair slots of the query blocks they belong to (bulk copies of the
          // swizzled rows; k_bwd_dq loads them back as MMA operands). Rows past a block's kept count are 0.
          __syncwarp();
          if (lane == 0) {
            const int* slots = reinterpret_cast<const int*>(sm + SM::OFF_SLOT) + (c & 3) * 16;
            const int w0 = q4 * 32;
            for (int e = 0; e < ne; ++e) {
              const int v = s_nk[c & 3][e], roff = v >> 8, nk = v & 255, sz = slot_size(nk, SR);
              const int sl = slots[e];
              const int r0 = max_i(roff, w0), r1 = min_i(roff + sz, w0 + 32);
              if (sl < 0 || r0 >= r1 || r0 - roff >= nk) continue;
              bulk_store(p.ds_buf + (static_cast<size_t>(sl) * SR + (r0 - roff)) * 128, sdS + r0 * 128,
                         static_cast<uint32_t>(r1 - r0) * 128);
            }
            bulk_commit_group();
          }
        }
        if (row == 0) BWD_TRACE(5, c);
        ++c;
        if (last) break;
      }
      if (row == 0) CTA_STAMP(5);
      // dK_j, dV_j: TMEM lane == channel (row of dK^T / dV^T), columns == keys of block j. Transposed into
      // the block's [key][64-channel] SW128 tiles in sP (dK) and sdS (dV) -- free once the block's last
      // gradient MMA completed -- and written with the same 5D block box the K/V tiles came in with, so
      // keys past a ragged block's extent are clipped by TMA. bar_acc_free hands dV/dK back to the next
      // block's first gradient MMAs as soon as they are in registers.
      const int ch_ = row;
      const uint32_t tdk = smem_u32(sP), tdv = smem_u32(sdS);
      if (row == 0) PROG(11, 1000 + nacc);
      if (any_chunk) {
        bwait(&bar_acc, nacc & 1);
        tc_fence_after();
      }
      if (row == 0) PROG(11, 2000 + nacc);
      if (store_pending || DS) {  // (a block with no chunks right after another block's store; dS stores)
        if (DS ? lane == 0 : row == 0) bulk_wait_group_read<0>();
        named_bar_sync(1, 128);
        store_pending = false;
      }
#pragma unroll 1
      for (int cc0 = 0; cc0 < BT; cc0 += 16) {
        float kv[16], vv[16];
        if (any_chunk) {
          tmem_ld16(trow + 3 * BT + cc0, kv);
          tmem_ld16(trow + 2 * BT + cc0, vv);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) kv[e] = vv[e] = 0.f;
        }
        if (ch_ < D) {
          const uint32_t cofs = (ch_ >> 6) * BT * 128 + (ch_ & 7) * 2;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint32_t o = cofs + sw128_off(cc0 + e, (ch_ & 63) >> 3);
            sts16(tdk + o, __bfloat16_as_ushort(__float2bfloat16_rn(kv[e] * p.scale)));
            sts16(tdv + o, __bfloat16_as_ushort(__float2bfloat16_rn(vv[e])));
          }
        }
      }
      if (any_chunk) {
        tc_fence_before();
        mbar_arrive(&bar_acc_free);
        ++nacc;
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (row == 0) {
        const int hc = item / g.N, j = item - hc * g.N;
        const int bt = j / (g.Nh * g.Nw), bhh = (j / g.Nw) % g.Nh, bw = j % g.Nw;
        for (int cb = 0; cb < NCB; ++cb) {
          tma_store_5d(&p.mdK, sP + cb * BT * 128, cb * 64, bw * g.cw, bhh * g.ch, bt * g.ct, hc);
          tma_store_5d(&p.mdV, sdS + cb * BT * 128, cb * 64, bw * g.cw, bhh * g.ch, bt * g.ct, hc);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      store_pending = true;
      if (row == 0) CTA_STAMP(6);
    }
    if (row == 0) bulk_wait_group<0>();  // the last stores are complete before the CTA exits
  } else if (warp < 8 && !DS) {
    // ============================ dQ drain: TMEM dQ partial -> smem slices -> TMA bulk reduce-add
    // Each warp owns TMEM lane quadrant q4 (chunk rows 32 q4 .. +32), split into 32/R sub-boxes of R =
    // min(SR, 16) rows that each belong to one query block and map to R consecutive packed dQacc rows.
    // Per 32-column slice: tcgen05.ld -> two 16-row x 128 B slots (128B swizzle, the map's layout) ->
    // one cp.reduce.async.bulk.tensor add per sub-box; the L2 does the fp32 adds (no per-thread atomics;
    // 128-byte row segments reach ~6 TB/s of reduce traffic on B200, tools/microbench/red_rate.cu). Rows past a
    // block's kept count hold exact zeros (P = dS = 0 there), so a sub-box may overlap the next block's
    // rows harmlessly. Slots form a per-warp ring; each 16-row half is one bulk group.
    const int q4 = warp - 4;
    const int row = q4 * 32 + lane;
    constexpr int SROWS = SM::DQ_SROWS, NSL = SM::DQ_SLOTS, SPS = 32 / SROWS;  // slots per 32-column slice
    static_assert(SROWS == 32, "a drain slot holds the warp's 32 rows of one 32-column slice");
    uint8_t* slots = sm + SM::OFF_DQS + q4 * NSL * SM::DQ_SLOT_BYTES;
    int slot_i = 0;
    int c = 0;
    for (int it = 0;; ++it) {
      const int item = read_item(it);
      if (item < 0) break;
      const int hc = item / g.N, j = item - hc * g.N, bh = p.bh0 + hc;
      const bool any_chunk = nq_of(bh, j) > 0;
      for (bool last = !any_chunk; any_chunk;) {
        const int qbuf = c & 1;
        if (lane == 0) PROG(4 + q4, c * 8 + 0);
        bwait(&bar_dq_full[qbuf], (c >> 1) & 1);
        if (lane == 0) PROG(4 + q4, c * 8 + 1);
        tc_fence_after();
        if (row == 0) BWD_TRACE(6, c);
        const int ring = c & 3;
        // this quadrant's pieces of the chunk's blocks (a block's rows inside [32 q4, 32 q4 + 32), 8 / 16 / 32 of
        // them, at most four), read into registers now: the ring entry may be rewritten once dQ(c) is released
        const int cinfo = s_cinfo[ring], ne = cinfo & 255;
        last = (cinfo >> 8) & 1;
        int pdst = -1, poff = 0, prows = 0;
        if (lane < ne) {
          const int v = s_nk[ring][lane], roff = v >> 8, nk = v & 255, sz = slot_size(nk, SR);
          const int r0 = max_i(roff, q4 * 32), r1 = min_i(roff + sz, q4 * 32 + 32);
          if (r0 < r1 && r0 - roff < nk) {
            pdst = s_row0[ring][lane] + (r0 - roff);
            poff = r0 - q4 * 32;
            prows = r1 - r0;
          }
        }
        unsigned pm = __ballot_sync(0xffffffffu, pdst >= 0);
        const bool any = pm != 0u;
        int dk[4], dof[4], drw[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int e = pm ? __ffs(pm) - 1 : 0;
          dk[k] = __shfl_sync(0xffffffffu, pdst, e);
          dof[k] = __shfl_sync(0xffffffffu, poff, e);
          drw[k] = __shfl_sync(0xffffffffu, prows, e);
          if (!pm) dk[k] = -1;
          pm &= pm - 1u;
        }
#pragma unroll 1
        for (int cs = 0; cs < D; cs += 32) {
          float v[32];
          const uint32_t tq = tdQ + qbuf * D + (static_cast<uint32_t>(q4 * 32) << 16) + cs;
          tmem_ld16(tq, v);
          tmem_ld16(tq + 16, v + 16);
          tmem_wait_ld();
          if (cs + 32 == D) {  // the whole partial is out of TMEM: dQ buffer free for chunk c+2
            tc_fence_before();
            mbar_arrive(&bar_dq_free[qbuf]);
          }
          if (any) {
            const int s_first = slot_i;
            slot_i = (slot_i + SPS) % NSL;
            // the slots' previous reduces (issued >= NSL - SPS groups ago) must have read them
            if (lane == 0) PROG(4 + q4, c * 8 + 2 + cs / 32);
            if (lane == 0) bulk_wait_group_read<NSL - SPS>();
            __syncwarp();
            const int my = lane / SROWS, rr = lane % SROWS;
            const uint32_t srow = smem_u32(slots + ((s_first + my) % NSL) * SM::DQ_SLOT_BYTES) + rr * 128;
#pragma unroll
            for (int k = 0; k < 8; ++k)
              sts128(srow + ((k ^ (rr & 7)) << 4), __float_as_uint(v[4 * k]), __float_as_uint(v[4 * k + 1]),
                     __float_as_uint(v[4 * k + 2]), __float_as_uint(v[4 * k + 3]));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              uint8_t* slot = slots + s_first * SM::DQ_SLOT_BYTES;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if (dk[k] < 0) continue;
                // the box covering the piece's rows (8 / 16 / 32; its rows are a prefix-aligned part of the slot)
                const CUtensorMap* m = drw[k] == 32 ? &p.mDQ : drw[k] == 16 ? &p.mDQh : &p.mDQq;
                tma_reduce_add_2d(m, slot + dof[k] * 128, cs, dk[k]);
              }
              bulk_commit_group();
            }
          }
        }
        if (row == 0) BWD_TRACE(7, c);
        ++c;
        if (last) break;
      }
    }
    if (lane == 0) PROG(4 + q4, 999999);
    if (lane == 0) bulk_wait_group<0>();
    if (lane == 0) PROG(4 + q4, 1999999);
    if (row == 0) CTA_STAMP(7);
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_ALLOC) tmem_dealloc(tbase, SM::TMEM_COLS);
#ifdef BSA_TRACE
  // trace mode cta == -1: per-CTA [start, end, smid, nchunks] (globaltimer ns)
  if (g_bwd_trace != nullptr && g_bwd_trace_cta == -1 && tid == 0) {
    unsigned long long* e = g_bwd_trace + 16 * static_cast<size_t>(blockIdx.y * gridDim.x + blockIdx.x);
    unsigned long long t1;
    unsigned sm_id;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_id));
    const int nch = 0;
    e[0] = t_start;
    e[1] = t1;
    e[2] = sm_id;
    e[3] = nch;
  }
#endif
}


// ------------------------------------------------------------------------------------ dS path: pair slots
// The dS tiles of query block i are stored contiguously in q2k order: pair (i, t-th admitted KV block) at slot
// base(bh) + q2k_off[bh][i] + t. k_pair_off: per head the exclusive scan of q2k_num and its total.
__global__ void __launch_bounds__(1024) k_pair_off(int N, const int* __restrict__ q2k_num, int* __restrict__ q2k_off,
                                                   int* __restrict__ tot) {
  __shared__ int s_w[32];
  __shared__ int s_chunk;
  const int bh = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int* num = q2k_num + static_cast<size_t>(bh) * N;
  int carry = 0;
  for (int b0 = 0; b0 < N; b0 += 1024) {
    const int i = b0 + tid;
    const int v = i < N ? num[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += a;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int w = s_w[lane];
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += a;
      }
      s_w[lane] = wi - w;  // exclusive prefix of the warp totals
      if (lane == 31) s_chunk = wi;
    }
    __syncthreads();
    if (i < N) q2k_off[static_cast<size_t>(bh) * N + i] = carry + s_w[warp] + incl - v;
    carry += s_chunk;
    __syncthreads();
  }
  if (tid == 0) tot[bh] = carry;
}

// k_pair_slot: slot of every k2q entry (KV block j, p-th admitting query block i) = base(bh) + q2k_off[i] + rank
// of j in q2k[i] (binary search in the ascending list; k2q is its exact transpose). One warp per KV block.
// The last head's first CTA also writes the total number of pairs (the path switch).
__global__ void __launch_bounds__(256) k_pair_slot(int N, int BH, const int* __restrict__ q2k_num,
                                                   const int* __restrict__ q2k_idx, const int* __restrict__ k2q_num,
                                                   const int* __restrict__ k2q_idx, const int* __restrict__ q2k_off,
                                                   const int* __restrict__ tot, int* __restrict__ k2q_slot,
                                                   int* __restrict__ pair_total) {
  __shared__ int s_part[8];
  const int bh = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int b = 0;
  for (int h = threadIdx.x; h < bh; h += 256) b += tot[h];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
  if (lane == 0) s_part[warp] = b;
  __syncthreads();
  const int base = s_part[0] + s_part[1] + s_part[2] + s_part[3] + s_part[4] + s_part[5] + s_part[6] + s_part[7];
  if (bh == BH - 1 && blockIdx.x == 0 && threadIdx.x == 0) *pair_total = base + tot[bh];
  const int j = blockIdx.x * 8 + warp;
  if (j >= N) return;
  const size_t hN = static_cast<size_t>(bh) * N;
  const int nq = k2q_num[hN + j];
  for (int pp = lane; pp < nq; pp += 32) {
    const int i = k2q_idx[(hN + j) * N + pp];
    const int* row = q2k_idx + (hN + i) * N;
    int lo = 0, hi = q2k_num[hN + i];  // first position with row[pos] >= j
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (row[mid] < j) lo = mid + 1;
      else hi = mid;
    }
    k2q_slot[(hN + j) * N + pp] = base + q2k_off[hN + i] + lo;
  }
}

// ------------------------------------------------------------------------------------ dS path: dQ
// dQ[kept rows of block i] = scale * sum over its admitted KV blocks j of dS_ij K_j, formed transposed so the
// tensor-core M is the channel dimension: dQ_i^T (d x SR) += K_j^T (d x BT, MN-major) dS_ij^T (BT x SR, K-major),
// one TMEM accumulator per query block of the CTA's tile (fp32, deterministic order: ascending j).
// Warps 0-3: epilogue (thread = channel = TMEM lane), warp 4: producer (K_j by the 5D block box, dS tile by one
// bulk copy), warp 5: TMEM allocator + MMA issuer.
constexpr int DQ_STAGES = 4;
constexpr int DQ_THREADS = 192;
template <int D, int BT>
struct DqSmem {
  static constexpr int NCB = D / 64;
  static constexpr int K_BYTES = BT * D * 2;
  static constexpr int DS_BYTES = 64 * 128;  // up to 64 rows of 128 B (SR <= 64; N >= 16 rows read)
  static constexpr int STAGE = K_BYTES + DS_BYTES;
  static constexpr int OFF_ZERO = DQ_STAGES * STAGE;  // d = 64: zero channels 64..127 of the M = 128 operand
  static constexpr int TOTAL = OFF_ZERO + (D == 64 ? BT * 128 : 0);
};

struct DqParams {
  CUtensorMap mK;
  Geo g;
  int Lq, SR, N16, Gq, bh0;
  const int* kept_off;
  const int* kept_tok;
  const int* q2k_num;
  const int* q2k_idx;
  const int* q2k_off;
  const int* tot;
  const int* pair_total;
  long long ds_cap;
  const uint8_t* ds_buf;
  float scale;
  Rows dQ;
};

template <int D, int BT>
__global__ void __launch_bounds__(DQ_THREADS) k_bwd_dq(const __grid_constant__ DqParams p) {
  using SM = DqSmem<D, BT>;
  if (!(*p.pair_total <= p.ds_cap)) return;  // reduce path
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  __shared__ __align__(8) uint64_t bar_full[DQ_STAGES], bar_empty[DQ_STAGES], bar_acc[16];
  __shared__ uint32_t s_tmem;
  __shared__ int s_base;
  const Geo& g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hc = blockIdx.y, bh = p.bh0 + hc;
  const int Gq = p.Gq, N16 = p.N16, SR = p.SR;
  const int i0 = blockIdx.x * Gq;
  const int nblk = min_i(Gq, g.N - i0);
  const size_t hN = static_cast<size_t>(bh) * g.N;
  if (tid == 0) {
    for (int s = 0; s < DQ_STAGES; ++s) { mbar_init(&bar_full[s], 1); mbar_init(&bar_empty[s], 1); }
    for (int k = 0; k < 16; ++k) mbar_init(&bar_acc[k], 1);
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(&s_tmem, Gq * N16 <= 32 ? 32 : Gq * N16 <= 64 ? 64 : Gq * N16 <= 128 ? 128 : 256);
  if (warp == 4) {  // pair base of this head
    int b = 0;
    for (int h = lane; h < bh; h += 32) b += p.tot[h];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if (lane == 0) s_base = b;
  }
  if (D == 64)
    for (int o = tid * 16; o < BT * 128; o += DQ_THREADS * 16)
      *reinterpret_cast<uint4*>(sm + SM::OFF_ZERO + o) = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tacc = s_tmem;
  const int base = s_base;

  if (warp == 4) {
    // ============================ producer: every admitted pair of the tile's blocks, block by block
    int n = 0;
    for (int gi = 0; gi < nblk; ++gi) {
      const int i = i0 + gi;
      const int num = p.q2k_num[hN + i];
      const size_t off = static_cast<size_t>(base) + p.q2k_off[hN + i];
      const int* list = p.q2k_idx + (hN + i) * g.N;
      for (int t0 = 0; t0 < num; t0 += 32) {
        const int jl = t0 + lane < num ? list[t0 + lane] : 0;  // 32 list entries fetched at once
        const int cnt = min_i(32, num - t0);
        for (int e = 0; e < cnt; ++e, ++n) {
          const int j = __shfl_sync(0xffffffffu, jl, e);
          const int s = n % DQ_STAGES;
          if (lane == 0) {
            mbar_wait(&bar_empty[s], ((n / DQ_STAGES) & 1) ^ 1);
            mbar_expect_tx(&bar_full[s], SM::K_BYTES + SR * 128);
            uint8_t* st = sm + s * SM::STAGE;
            const int bt = j / (g.Nh * g.Nw), bhh = (j / g.Nw) % g.Nh, bw = j % g.Nw;
            for (int cb = 0; cb < SM::NCB; ++cb)
              tma_load_5d(st + cb * BT * 128, &p.mK, &bar_full[s], cb * 64, bw * g.cw, bhh * g.ch, bt * g.ct, hc);
            bulk_load(st + SM::K_BYTES, p.ds_buf + (off + t0 + e) * static_cast<size_t>(SR) * 128, SR * 128,
                      &bar_full[s]);
          }
        }
      }
    }
  } else if (warp == 5) {
    // ============================ MMA issuer: dQ_i^T += K_j^T dS_ij^T (M = 128 channels, N = N16 rows, K = BT)
    const bool leader = elect_one();
    const uint32_t idesc = umma_idesc_bf16(128, N16, 1, 0);
    const uint32_t zero = smem_u32(sm + SM::OFF_ZERO);
    int n = 0;
    for (int gi = 0; gi < nblk; ++gi) {
      const int num = p.q2k_num[hN + i0 + gi];
      for (int t = 0; t < num; ++t, ++n) {
        const int s = n % DQ_STAGES;
        mbar_wait(&bar_full[s], (n / DQ_STAGES) & 1);
        tc_fence_after();
        if (leader) {
          const uint32_t ka = smem_u32(sm + s * SM::STAGE), da = ka + SM::K_BYTES;
#pragma unroll
          for (int kk = 0; kk < BT / 16; ++kk) {
            // A: K_j^T, MN-major over channels (64-channel chunks BT * 128 B apart; d = 64 reads the zero block)
            const uint64_t adesc = umma_desc_sw128(ka + kk * 2048, D == 128 ? BT * 128 : zero - ka, 1024);
            const uint64_t bdesc = umma_desc_sw128(da + kk * 32, 16, 1024);  // B: dS rows, K-major over keys
            umma_ss(tacc + gi * N16, adesc, bdesc, idesc, (t > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&bar_empty[s]);
          if (t == num - 1) umma_commit(&bar_acc[gi]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 4) {
    // ============================ epilogue: thread = channel (TMEM lane), columns = the block's rows
    const int ch = warp * 32 + lane;
    const uint32_t trow = tacc + (static_cast<uint32_t>(warp * 32) << 16);
    for (int gi = 0; gi < nblk; ++gi) {
      const int i = i0 + gi;
      const int num = p.q2k_num[hN + i];
      const int ko = p.kept_off[i], nk = p.kept_off[i + 1] - ko;
      if (num > 0) {
        mbar_wait(&bar_acc[gi], 0);
        tc_fence_after();
      }
      for (int c0 = 0; c0 < nk; c0 += 16) {
        float v[16];
        if (num > 0) {
          tmem_ld16(trow + gi * N16 + c0, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = 0.f;
        }
        if (ch < D) {
          const int* toks = p.kept_tok + static_cast<size_t>(bh) * p.Lq + ko;
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (c0 + e < nk) p.dQ.row(bh, toks[c0 + e])[ch] = __float2bfloat16_rn(v[e] * p.scale);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(tacc, Gq * N16 <= 32 ? 32 : Gq * N16 <= 64 ? 64 : Gq * N16 <= 128 ? 128 : 256);
}

// ------------------------------------------------------------------------------------ finalize
// dQ of one (b,h, block): kept tokens (ascending) take scale * dQacc of their packed row kept_off[b] + rank,
// pruned tokens get 0 (reading C10). One CTA per block: the block's donors decide kept / pruned, a ballot
// prefix gives the rank, and every row is written once with 16-byte stores.
template <int D>
__global__ void __launch_bounds__(256) k_bwd_finalize(Geo g, int Lq, float scale, const int* __restrict__ kept_off,
                                                      const int* __restrict__ donor, const float* __restrict__ dQacc,
                                                      const Rows dQ, const int* __restrict__ pair_total,
                                                      long long ds_cap) {
  if (pair_total != nullptr && *pair_total <= ds_cap) return;  // dS path: k_bwd_dq wrote dQ
  constexpr int MAXT = 128, VPR = D / 8;
  __shared__ int s_tok[MAXT], s_prow[MAXT], s_wk[8];
  const int blk = blockIdx.x, bh = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Box x = block_box(g, blk);
  const int n = box_size(x);
  const int t = threadIdx.x;
  bool kept = false;
  if (t < n) {
    const int tok = box_token(g, x, t);
    s_tok[t] = tok;
    kept = __ldg(donor + static_cast<size_t>(bh) * g.L + tok) == tok;
  }
  const unsigned kb = __ballot_sync(0xffffffffu, kept);
  if (lane == 0) s_wk[warp] = __popc(kb);
  __syncthreads();
  if (t < n) {
    int pos = __popc(kb & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) pos += s_wk[w];
    s_prow[t] = kept ? static_cast<int>(static_cast<size_t>(bh) * Lq + kept_off[blk] + pos) : -1;
  }
  __syncthreads();
  bf16* dqh = dQ.head(bh);
  for (int v = t; v < n * VPR; v += 256) {
    const int i = v / VPR, c = (v % VPR) * 8;
    const int prow = s_prow[i];
    uint4 o = make_uint4(0, 0, 0, 0);
    if (prow >= 0) {
      const float4* src = reinterpret_cast<const float4*>(dQacc + static_cast<size_t>(prow) * D + c);
      const float4 a = src[0], b = src[1];
      o.x = pack_bf16(a.x * scale, a.y * scale);
      o.y = pack_bf16(a.z * scale, a.w * scale);
      o.z = pack_bf16(b.x * scale, b.y * scale);
      o.w = pack_bf16(b.z * scale, b.w * scale);
    }
    *reinterpret_cast<uint4*>(dqh + s_tok[i] * dQ.sl + c) = o;
  }
}

// The K/V/dK/dV tensor maps index heads with one stride: one launch over all B*Hh heads when the batch stride
// continues the head stride (sb == Hh sh, e.g. contiguous [B, Hh, L, d], or B == 1), else one launch per batch.
static bool heads_uniform(const Rows& x, int B) { return B == 1 || x.sb == x.Hh * x.sh; }

template <int D, int BT, bool DS>
static cudaError_t run_bwd1(const BwdParams& p, int sms, cudaStream_t st) {
  constexpr int smem = BwdSmem<D, BT, DS>::TOTAL;
  cudaError_t e = cudaFuncSetAttribute(k_attn_bwd<D, BT, DS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_attn_bwd<D, BT, DS><<<dim3(static_cast<unsigned>(min_i(p.items, sms))), BWD_THREADS, smem, st>>>(p);  // persistent
  return cudaGetLastError();
}
// dS mode: both instantiations are launched and the one the device-side pair count does not select exits at once;
// reduce mode (pair_total == NULL): only the reduce instantiation
template <int D, int BT>
static cudaError_t run_bwd(const BwdParams& p, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess && p.pair_total != nullptr) e = run_bwd1<D, BT, true>(p, sms, st);
  if (e == cudaSuccess) e = run_bwd1<D, BT, false>(p, sms, st);
  return e;
}

// slot of every admitted pair for the dS path (k_pair_off, k_pair_slot) and the path switch *pair_total
cudaError_t launch_bwd_pairs(const BwdArgs& a, cudaStream_t st) {
  k_pair_off<<<a.BH, 1024, 0, st>>>(a.g.N, a.q2k_num, a.q2k_off, a.pair_tot);
  k_pair_slot<<<dim3((a.g.N + 7) / 8, a.BH), 256, 0, st>>>(a.g.N, a.BH, a.q2k_num, a.q2k_idx, a.k2q_num, a.k2q_idx,
                                                            a.q2k_off, a.pair_tot, a.k2q_slot, a.pair_total);
  return cudaGetLastError();
}

template <int D, int BT>
static cudaError_t run_dq(const DqParams& p, int heads, cudaStream_t st) {
  constexpr int smem = DqSmem<D, BT>::TOTAL;
  cudaError_t e = cudaFuncSetAttribute(k_bwd_dq<D, BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_bwd_dq<D, BT><<<dim3((p.g.N + p.Gq - 1) / p.Gq, heads), DQ_THREADS, smem, st>>>(p);
  return cudaGetLastError();
}

// dS path: dQ of the kept rows from the stored dS tiles (exits at once on the reduce path)
cudaError_t launch_bwd_dq(const BwdArgs& a, cudaStream_t st) {
  DqParams p;
  memset(&p, 0, sizeof(p));
  p.g = a.g;
  p.Lq = a.Lq;
  p.SR = a.SR;
  p.N16 = a.SR < 16 ? 16 : a.SR;
  p.Gq = 128 / p.N16;
  p.kept_off = a.kept_off;
  p.kept_tok = a.kept_tok;
  p.q2k_num = a.q2k_num;
  p.q2k_idx = a.q2k_idx;
  p.q2k_off = a.q2k_off;
  p.tot = a.pair_tot;
  p.pair_total = a.pair_total;
  p.ds_cap = a.ds_cap;
  p.ds_buf = a.ds_buf;
  p.scale = a.scale;
  p.dQ = a.dQ;
  const bool one = heads_uniform(a.K, a.B);
  const int launches = one ? 1 : a.B, heads = one ? a.BH : a.Hh;
  for (int b = 0; b < launches; ++b) {
    if (!make_map_5d(&p.mK, a.K.p + b * a.K.sb, a.g, a.d, heads, a.K.sl, a.K.sh)) return cudaErrorInvalidValue;
    p.bh0 = b * a.Hh;
    cudaError_t e = cudaErrorInvalidValue;
    if (a.d == 128 && a.g.BT == 64) e = run_dq<128, 64>(p, heads, st);
    else if (a.d == 128 && a.g.BT == 32) e = run_dq<128, 32>(p, heads, st);
    else if (a.d == 64 && a.g.BT == 64) e = run_dq<64, 64>(p, heads, st);
    else if (a.d == 64 && a.g.BT == 32) e = run_dq<64, 32>(p, heads, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}


// launches of the main kernel: one over all heads when the K/V/dK/dV head strides are uniform, else one per batch
static int bwd_launch_heads(const BwdArgs& a) {
  const bool one = heads_uniform(a.K, a.B) && heads_uniform(a.V, a.B) && heads_uniform(a.dK, a.B) &&
                   heads_uniform(a.dV, a.B);
  return one ? a.BH : a.Hh;
}

cudaError_t launch_bwd_prep(const BwdArgs& a, cudaStream_t st) {
  // one CTA per (b,h, query block), plus one per main-kernel launch for its claim order
  const dim3 prep_blocks(a.g.N + (a.item_order ? 1 : 0), a.BH);
  const int lh = bwd_launch_heads(a);
  if (a.d == 128)
    k_bwd_prep<128><<<prep_blocks, 256, 0, st>>>(a.g, a.BH, a.Lq, a.SR, a.kept_off, a.kept_tok, a.donor, a.Qs, a.dO,
                                                 a.O, a.lse, a.qdo_img, a.lsed, a.dQacc, a.pair_total, a.ds_cap, a.dQ,
                                                 a.k2q_num, a.item_order, lh, a.short_pct);
  else
    k_bwd_prep<64><<<prep_blocks, 256, 0, st>>>(a.g, a.BH, a.Lq, a.SR, a.kept_off, a.kept_tok, a.donor, a.Qs, a.dO,
                                                a.O, a.lse, a.qdo_img, a.lsed, a.dQacc, a.pair_total, a.ds_cap, a.dQ,
                                                a.k2q_num, a.item_order, lh, a.short_pct);
  return cudaGetLastError();
}

cudaError_t launch_bwd_main(const BwdArgs& a, cudaStream_t st) {
  BwdParams p;
  memset(&p, 0, sizeof(p));
  p.g = a.g;
  p.Lq = a.Lq;
  p.SR = a.SR;
  p.G = 128 / a.SR;
  p.kept_off = a.kept_off;
  p.k2q_num = a.k2q_num;
  p.k2q_idx = a.k2q_idx;
  p.dQacc = a.dQacc;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.scale = a.scale;
  p.qdo_img = a.qdo_img;
  p.lsed = a.lsed;
  p.pair_total = a.pair_total;
  p.ds_cap = a.ds_cap;
  p.k2q_slot = a.k2q_slot;
  p.ds_buf = a.ds_buf;
  const size_t dq_rows_total = static_cast<size_t>(a.BH) * a.Lq;
  if (!make_map_rows_f32(&p.mDQ, a.dQacc, a.d, dq_rows_total, 32) ||
      !make_map_rows_f32(&p.mDQh, a.dQacc, a.d, dq_rows_total, 16) ||
      !make_map_rows_f32(&p.mDQq, a.dQacc, a.d, dq_rows_total, 8))
    return cudaErrorInvalidValue;
  const int heads = bwd_launch_heads(a), launches = a.BH / heads;
  p.item_order = a.item_order;
  // one work counter per launch, zeroed on the stream (the persistent CTAs claim items from it)
  cudaError_t ez = cudaMemsetAsync(a.work_ctr, 0, sizeof(int) * launches, st);
  if (ez != cudaSuccess) return ez;
  p.items = heads * a.g.N;
  for (int b = 0; b < launches; ++b) {
    p.work_ctr = a.work_ctr + b;
    const Rows* ts[4] = {&a.K, &a.V, &a.dK, &a.dV};
    CUtensorMap* ms[4] = {&p.mK, &p.mV, &p.mdK, &p.mdV};
    for (int t = 0; t < 4; ++t)
      if (!make_map_5d(ms[t], ts[t]->p + b * ts[t]->sb, a.g, a.d, heads, ts[t]->sl, ts[t]->sh))
        return cudaErrorInvalidValue;
    p.bh0 = b * a.Hh;
    cudaError_t e = cudaErrorInvalidValue;
    if (a.d == 128 && a.g.BT == 64) e = run_bwd<128, 64>(p, st);
    else if (a.d == 128 && a.g.BT == 32) e = run_bwd<128, 32>(p, st);
    else if (a.d == 64 && a.g.BT == 64) e = run_bwd<64, 64>(p, st);
    else if (a.d == 64 && a.g.BT == 32) e = run_bwd<64, 32>(p, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_bwd_finalize(const BwdArgs& a, cudaStream_t st) {
  const dim3 grid(a.g.N, a.BH);
  if (a.d == 128)
    k_bwd_finalize<128><<<grid, 256, 0, st>>>(a.g, a.Lq, a.scale, a.kept_off, a.donor, a.dQacc, a.dQ, a.pair_total,
                                              a.ds_cap);
  else
    k_bwd_finalize<64><<<grid, 256, 0, st>>>(a.g, a.Lq, a.scale, a.kept_off, a.donor, a.dQacc, a.dQ, a.pair_total,
                                             a.ds_cap);
  return cudaGetLastError();
}

cudaError_t debug_progress_bwd(void* dev_ptr) {
  unsigned* p = static_cast<unsigned*>(dev_ptr);
#ifdef BSA_HANG_DEBUG
  return cudaMemcpyToSymbol(g_hang_rec, &p, sizeof(p));
#else
  return cudaMemcpyToSymbol(g_bwd_prog, &p, sizeof(p));
#endif
}

cudaError_t debug_trace_bwd(void* dev_buf, int cta) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_buf);
  cudaError_t e = cudaMemcpyToSymbol(g_bwd_trace, &p, sizeof(p));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_bwd_trace_cta, &cta, sizeof(int));
  return e;
}

}  // namespace bsa
