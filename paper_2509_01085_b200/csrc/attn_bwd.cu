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
//               dQ_part = dS K_j                            (M=128, N=d) -> fp32 vector reductions
//   finalize: dQ[kept] = scale * dQacc (bf16), dQ[pruned] = 0.
#include <cmath>
#include "kernels.h"
#include "ptx.cuh"

namespace bsa {

bool make_map_2d(CUtensorMap* m, const void* base, int d, size_t rows, int box_rows);
bool make_map_5d(CUtensorMap* m, const void* base, const Geo& g, int d, int BH);

__device__ __forceinline__ float ex2b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------------------------------------------ prep
// One warp per packed kept row.
template <int D>
__global__ void __launch_bounds__(256) k_bwd_prep(Geo g, int BH, int Lq, const int* __restrict__ kept_tok,
                                                  const int* __restrict__ donor, const bf16* __restrict__ dO,
                                                  const bf16* __restrict__ O, bf16* __restrict__ dOs,
                                                  float* __restrict__ Dvec, float* __restrict__ dQacc) {
  constexpr int PER = D / 32;  // channels per lane (4 or 2)
  const size_t wid = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= static_cast<size_t>(BH) * Lq) return;
  const size_t bh = wid / Lq;
  const int tok = kept_tok[wid];
  const size_t head = bh * g.L;
  float acc[PER];
  {
    const bf16* src = dO + (head + tok) * D + lane * PER;
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = __bfloat162float(src[e]);
  }
  // donees of tok live in tok's block
  int t = tok / (g.H * g.W), h = (tok / g.W) % g.H, w = tok % g.W;
  int b = ((t / g.ct) * g.Nh + h / g.ch) * g.Nw + w / g.cw;
  const Box x = block_box(g, b);
  const int n = box_size(x);
  for (int i0 = 0; i0 < n; i0 += 32) {
    int i = i0 + lane;
    int ti = i < n ? box_token(g, x, i) : -1;
    bool match = i < n && ti != tok && donor[head + ti] == tok;
    unsigned m = __ballot_sync(0xffffffffu, match);
    while (m) {
      int src_lane = __ffs(m) - 1;
      m &= m - 1;
      int tsrc = __shfl_sync(0xffffffffu, ti, src_lane);
      const bf16* src = dO + (head + tsrc) * D + lane * PER;
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[e] += __bfloat162float(src[e]);
    }
  }
  float dsum = 0.f;
  const bf16* orow = O + (head + tok) * D + lane * PER;
  bf16* out = dOs + wid * D + lane * PER;
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    bf16 hv = __float2bfloat16_rn(acc[e]);
    out[e] = hv;
    dsum += __bfloat162float(hv) * __bfloat162float(orow[e]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
  if (lane == 0) Dvec[wid] = dsum;
  float* dq = dQacc + wid * D + lane * PER;
#pragma unroll
  for (int e = 0; e < PER; ++e) dq[e] = 0.f;
}

// ------------------------------------------------------------------------------------ main
struct BwdParams {
  CUtensorMap mQs;   // 2D {d, BH*Lq}, box {64, SR}
  CUtensorMap mdOs;  // 2D, same geometry
  CUtensorMap mK;    // 5D block map
  CUtensorMap mV;
  Geo g;
  int Lq, SR, G;
  const int* kept_off;
  const int* k2q_num;
  const int* k2q_idx;
  const float* lse;
  const float* Dvec;
  float* dQacc;
  bf16* dK;
  bf16* dV;
  float scale_log2;
  float scale;
};

constexpr int BWD_THREADS = 256;

template <int D, int BT>
struct BwdSmem {
  static constexpr int NCB = D / 64;
  static constexpr int KV_BYTES = BT * D * 2;
  static constexpr int TILE_BYTES = 128 * D * 2;  // Q^s or dO^s chunk tile
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KV_BYTES;
  static constexpr int OFF_Q = OFF_V + KV_BYTES;          // 2 stages
  static constexpr int OFF_DO = OFF_Q + 2 * TILE_BYTES;   // 2 stages
  static constexpr int OFF_P = OFF_DO + 2 * TILE_BYTES;   // [128][64]
  static constexpr int OFF_DS = OFF_P + 16384;
  static constexpr int OFF_ZERO = OFF_DS + 16384;         // d=64 only: zero MN chunk for M=128 padding
  static constexpr int TOTAL = OFF_ZERO + (D == 64 ? 16384 : 0) + 1024;
  static constexpr int TMEM_COLS = (4 * BT + D) <= 256 ? 256 : 512;
};

template <int D, int BT>
__global__ void __launch_bounds__(BWD_THREADS, 1) k_attn_bwd(const __grid_constant__ BwdParams p) {
  using SM = BwdSmem<D, BT>;
  constexpr int NCB = SM::NCB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm + SM::OFF_K;
  uint8_t* sV = sm + SM::OFF_V;
  uint8_t* sQ = sm + SM::OFF_Q;
  uint8_t* sdO = sm + SM::OFF_DO;
  uint8_t* sP = sm + SM::OFF_P;
  uint8_t* sdS = sm + SM::OFF_DS;

  __shared__ __align__(8) uint64_t bar_kv, bar_c_full[2], bar_c_empty[2], bar_sd_full, bar_sd_free, bar_ps_full,
      bar_ps_free, bar_dq_full, bar_dq_free;
  __shared__ uint32_t s_tmem;

  const Geo& g = p.g;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j = blockIdx.x, bh = blockIdx.y;
  const int G = p.G, SR = p.SR;
  const size_t jrow = static_cast<size_t>(bh) * g.N + j;
  const int nq = p.k2q_num[jrow];
  const int* qlist = p.k2q_idx + jrow * g.N;
  const int nchunks = (nq + G - 1) / G;

  if (tid == 0) {
    mbar_init(&bar_kv, 1);
    for (int s = 0; s < 2; ++s) { mbar_init(&bar_c_full[s], 1); mbar_init(&bar_c_empty[s], 1); }
    mbar_init(&bar_sd_full, 1);
    mbar_init(&bar_sd_free, 128);
    mbar_init(&bar_ps_full, 128);
    mbar_init(&bar_ps_free, 1);
    mbar_init(&bar_dq_full, 1);
    mbar_init(&bar_dq_free, 128);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&s_tmem, SM::TMEM_COLS);
  // zero the Q/dO stages (rows of unused slots must be finite: they meet P = dS = 0 in the MMAs)
  for (int o = tid * 16; o < 4 * SM::TILE_BYTES; o += BWD_THREADS * 16)
    *reinterpret_cast<uint4*>(sQ + o) = make_uint4(0, 0, 0, 0);
  if (D == 64)
    for (int o = tid * 16; o < 16384; o += BWD_THREADS * 16)
      *reinterpret_cast<uint4*>(sm + SM::OFF_ZERO + o) = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = s_tmem;
  const uint32_t tS = tbase, tdP = tbase + BT, tdV = tbase + 2 * BT, tdK = tbase + 3 * BT, tdQ = tbase + 4 * BT;
  const Box xj = block_box(g, j);

  if (warp == 0) {
    if (lane == 0 && nchunks > 0) {
      tma_prefetch(&p.mQs);
      tma_prefetch(&p.mdOs);
      int bt = j / (g.Nh * g.Nw), bhh = (j / g.Nw) % g.Nh, bw = j % g.Nw;
      mbar_expect_tx(&bar_kv, 2 * SM::KV_BYTES);
      for (int cb = 0; cb < NCB; ++cb) {
        tma_load_5d(sK + cb * BT * 128, &p.mK, &bar_kv, cb * 64, bw * g.cw, bhh * g.ch, bt * g.ct, bh);
        tma_load_5d(sV + cb * BT * 128, &p.mV, &bar_kv, cb * 64, bw * g.cw, bhh * g.ch, bt * g.ct, bh);
      }
      for (int c = 0; c < nchunks; ++c) {
        int s = c & 1;
        mbar_wait(&bar_c_empty[s], ((c >> 1) & 1) ^ 1);
        int nb = min_i(G, nq - c * G);
        mbar_expect_tx(&bar_c_full[s], static_cast<uint32_t>(2 * nb * NCB * SR * 128));
        for (int gi = 0; gi < nb; ++gi) {
          int qb = qlist[c * G + gi];
          int row0 = bh * p.Lq + p.kept_off[qb];
          for (int cb = 0; cb < NCB; ++cb) {
            tma_load_2d(sQ + s * SM::TILE_BYTES + cb * 16384 + gi * SR * 128, &p.mQs, &bar_c_full[s], cb * 64, row0);
            tma_load_2d(sdO + s * SM::TILE_BYTES + cb * 16384 + gi * SR * 128, &p.mdOs, &bar_c_full[s], cb * 64,
                        row0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nchunks > 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, BT, 0, 0);   // Q K^T / dO V^T
      constexpr uint32_t idesc_t = umma_idesc_bf16(128, BT, 1, 1);   // dO^T P / Q^T dS (M = d padded to 128)
      constexpr uint32_t idesc_q = umma_idesc_bf16(128, D, 0, 1);    // dS K
      const uint32_t zero_lbo = (D == 64) ? 0u : 16384u;
      mbar_wait(&bar_kv, 0);
      for (int c = 0; c < nchunks; ++c) {
        int s = c & 1;
        mbar_wait(&bar_c_full[s], (c >> 1) & 1);
        if (c >= 1) mbar_wait(&bar_sd_free, (c - 1) & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(sQ + s * SM::TILE_BYTES), da = smem_u32(sdO + s * SM::TILE_BYTES);
        const uint32_t kb = smem_u32(sK), vb = smem_u32(sV);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          int cb = kk >> 2, ko = (kk & 3) * 32;
          umma_ss(tS, umma_desc_sw128(qa + cb * 16384 + ko, 16, 1024), umma_desc_sw128(kb + cb * BT * 128 + ko, 16, 1024),
                  idesc_s, kk > 0);
          umma_ss(tdP, umma_desc_sw128(da + cb * 16384 + ko, 16, 1024),
                  umma_desc_sw128(vb + cb * BT * 128 + ko, 16, 1024), idesc_s, kk > 0);
        }
        umma_commit(&bar_sd_full);
        mbar_wait(&bar_ps_full, c & 1);
        if (c >= 1) mbar_wait(&bar_dq_free, (c - 1) & 1);
        tc_fence_after();
        const uint32_t pa = smem_u32(sP), sa = smem_u32(sdS);
        // MN-major A over d: chunk 2 (d 64..127) sits LBO bytes after chunk 1; for d = 64 it is the zero block
        const uint32_t lbo_q = (D == 128) ? 16384u : (smem_u32(sm + SM::OFF_ZERO) - qa);
        const uint32_t lbo_d = (D == 128) ? 16384u : (smem_u32(sm + SM::OFF_ZERO) - da);
        (void)zero_lbo;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 128 query rows
          umma_ss(tdV, umma_desc_sw128(da + kk * 2048, lbo_d, 1024), umma_desc_sw128(pa + kk * 2048, 8192, 1024),
                  idesc_t, (c > 0 || kk > 0) ? 1u : 0u);
          umma_ss(tdK, umma_desc_sw128(qa + kk * 2048, lbo_q, 1024), umma_desc_sw128(sa + kk * 2048, 8192, 1024),
                  idesc_t, (c > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < BT / 16; ++kk)
          umma_ss(tdQ, umma_desc_sw128(sa + kk * 32, 16, 1024), umma_desc_sw128(kb + kk * 2048, BT * 128, 1024),
                  idesc_q, kk > 0);
        umma_commit(&bar_dq_full);
        umma_commit(&bar_c_empty[s]);
        umma_commit(&bar_ps_free);
      }
    }
  } else if (warp >= 4) {
    const int q4 = warp - 4;
    const int row = q4 * 32 + lane;
    const uint32_t trow = tbase + (static_cast<uint32_t>(q4 * 32) << 16);
    const int gi = row / SR, lr = row % SR;
    // key validity of block j (ragged edges, C23)
    uint64_t kmask = 0;
    for (int c = 0; c < BT; ++c) {
      int lw = c % g.cw, lh = (c / g.cw) % g.ch, lt = c / (g.cw * g.ch);
      if (lt < xj.e[0] && lh < xj.e[1] && lw < xj.e[2]) kmask |= 1ull << c;
    }
    for (int c = 0; c < nchunks; ++c) {
      int nb = min_i(G, nq - c * G);
      bool valid = false;
      size_t prow = 0;
      float lse2 = 0.f, Dq = 0.f;
      if (gi < nb) {
        int qb = qlist[c * G + gi];
        int nk = p.kept_off[qb + 1] - p.kept_off[qb];
        if (lr < nk) {
          valid = true;
          prow = static_cast<size_t>(bh) * p.Lq + p.kept_off[qb] + lr;
          lse2 = p.lse[prow] * 1.4426950408889634f;
          Dq = p.Dvec[prow];
        }
      }
      mbar_wait(&bar_sd_full, c & 1);
      tc_fence_after();
      float sv[BT], dp[BT];
#pragma unroll
      for (int cc = 0; cc < BT; cc += 16) {
        tmem_ld16(trow + cc, sv + cc);
        tmem_ld16(trow + BT + cc, dp + cc);
      }
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&bar_sd_free);
#pragma unroll
      for (int cc = 0; cc < BT; ++cc) {
        float pr = (valid && ((kmask >> cc) & 1ull)) ? ex2b(sv[cc] * p.scale_log2 - lse2) : 0.f;
        sv[cc] = pr;
        dp[cc] = pr * (dp[cc] - Dq);
      }
      if (c >= 1) mbar_wait(&bar_ps_free, (c - 1) & 1);
#pragma unroll
      for (int c16 = 0; c16 < BT / 8; ++c16) {
        uint32_t wp[4], wd[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 hp = __floats2bfloat162_rn(sv[c16 * 8 + 2 * e], sv[c16 * 8 + 2 * e + 1]);
          __nv_bfloat162 hd = __floats2bfloat162_rn(dp[c16 * 8 + 2 * e], dp[c16 * 8 + 2 * e + 1]);
          wp[e] = *reinterpret_cast<uint32_t*>(&hp);
          wd[e] = *reinterpret_cast<uint32_t*>(&hd);
        }
        *reinterpret_cast<uint4*>(sP + sw128_off(row, c16)) = make_uint4(wp[0], wp[1], wp[2], wp[3]);
        *reinterpret_cast<uint4*>(sdS + sw128_off(row, c16)) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bar_ps_full);
      // dQ partial of this chunk -> fp32 vector reductions into the packed accumulator
      mbar_wait(&bar_dq_full, c & 1);
      tc_fence_after();
      float* dst = p.dQacc + prow * D;
#pragma unroll 1
      for (int cc = 0; cc < D; cc += 16) {
        float v[16];
        tmem_ld16(trow + 4 * BT + cc, v);
        tmem_wait_ld();
        if (valid) {
#pragma unroll
          for (int e = 0; e < 16; e += 4)
            asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst + cc + e), "f"(v[e]), "f"(v[e + 1]),
                         "f"(v[e + 2]), "f"(v[e + 3])
                         : "memory");
        }
      }
      tc_fence_before();
      mbar_arrive(&bar_dq_free);
    }
    // dK_j, dV_j: TMEM lane == channel (row of dK^T / dV^T), columns == keys of block j
    const size_t head = static_cast<size_t>(bh) * g.L;
    const int ch_ = row;  // channel
    if (nchunks > 0) {
      // the last dq_full completion covers every MMA issued before it
      float kv[BT], vv[BT];
#pragma unroll
      for (int cc = 0; cc < BT; cc += 16) {
        tmem_ld16(trow + 3 * BT + cc, kv + cc);
        tmem_ld16(trow + 2 * BT + cc, vv + cc);
      }
      tmem_wait_ld();
      if (ch_ < D) {
#pragma unroll 4
        for (int cc = 0; cc < BT; ++cc) {
          if (!((kmask >> cc) & 1ull)) continue;
          int lw = cc % g.cw, lh = (cc / g.cw) % g.ch, lt = cc / (g.cw * g.ch);
          size_t tok = (static_cast<size_t>(xj.o[0] + lt) * g.H + (xj.o[1] + lh)) * g.W + (xj.o[2] + lw);
          p.dK[(head + tok) * D + ch_] = __float2bfloat16_rn(kv[cc] * p.scale);
          p.dV[(head + tok) * D + ch_] = __float2bfloat16_rn(vv[cc]);
        }
      }
    } else if (ch_ < D) {
      for (int cc = 0; cc < BT; ++cc) {
        if (!((kmask >> cc) & 1ull)) continue;
        int lw = cc % g.cw, lh = (cc / g.cw) % g.ch, lt = cc / (g.cw * g.ch);
        size_t tok = (static_cast<size_t>(xj.o[0] + lt) * g.H + (xj.o[1] + lh)) * g.W + (xj.o[2] + lw);
        p.dK[(head + tok) * D + ch_] = __float2bfloat16_rn(0.f);
        p.dV[(head + tok) * D + ch_] = __float2bfloat16_rn(0.f);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tbase, SM::TMEM_COLS);
}

// ------------------------------------------------------------------------------------ finalize
__global__ void k_bwd_zero_pruned(int BH, int L, int d, const int* __restrict__ donor, bf16* __restrict__ dQ) {
  size_t v = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int vpr = d / 8;
  if (v >= static_cast<size_t>(BH) * L * vpr) return;
  size_t rowi = v / vpr;
  int c = static_cast<int>(v % vpr) * 8;
  if (donor[rowi] != static_cast<int>(rowi % L))
    *reinterpret_cast<uint4*>(dQ + rowi * d + c) = make_uint4(0, 0, 0, 0);
}

__global__ void k_bwd_finalize(int BH, int L, int Lq, int d, float scale, const int* __restrict__ kept_tok,
                               const float* __restrict__ dQacc, bf16* __restrict__ dQ) {
  size_t v = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int vpr = d / 8;
  if (v >= static_cast<size_t>(BH) * Lq * vpr) return;
  size_t prow = v / vpr;
  int c = static_cast<int>(v % vpr) * 8;
  size_t bh = prow / Lq;
  int tok = kept_tok[prow];
  const float4* src = reinterpret_cast<const float4*>(dQacc + prow * d + c);
  float4 a = src[0], b = src[1];
  __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x * scale, a.y * scale), h1 = __floats2bfloat162_rn(a.z * scale, a.w * scale);
  __nv_bfloat162 h2 = __floats2bfloat162_rn(b.x * scale, b.y * scale), h3 = __floats2bfloat162_rn(b.z * scale, b.w * scale);
  uint4 o;
  o.x = *reinterpret_cast<uint32_t*>(&h0);
  o.y = *reinterpret_cast<uint32_t*>(&h1);
  o.z = *reinterpret_cast<uint32_t*>(&h2);
  o.w = *reinterpret_cast<uint32_t*>(&h3);
  *reinterpret_cast<uint4*>(dQ + (bh * L + tok) * d + c) = o;
}

template <int D, int BT>
static cudaError_t run_bwd(const BwdParams& p, int BH, cudaStream_t st) {
  constexpr int smem = BwdSmem<D, BT>::TOTAL;
  cudaError_t e = cudaFuncSetAttribute(k_attn_bwd<D, BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  k_attn_bwd<D, BT><<<dim3(p.g.N, BH), BWD_THREADS, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_bwd_prep(const BwdArgs& a, cudaStream_t st) {
  const size_t rows = static_cast<size_t>(a.BH) * a.Lq;
  const unsigned prep_blocks = static_cast<unsigned>((rows * 32 + 255) / 256);
  if (a.d == 128)
    k_bwd_prep<128><<<prep_blocks, 256, 0, st>>>(a.g, a.BH, a.Lq, a.kept_tok, a.donor, a.dO, a.O, a.dOs, a.Dvec,
                                                 a.dQacc);
  else
    k_bwd_prep<64><<<prep_blocks, 256, 0, st>>>(a.g, a.BH, a.Lq, a.kept_tok, a.donor, a.dO, a.O, a.dOs, a.Dvec,
                                                a.dQacc);
  return cudaGetLastError();
}

cudaError_t launch_bwd_main(const BwdArgs& a, cudaStream_t st) {
  const size_t rows = static_cast<size_t>(a.BH) * a.Lq;
  BwdParams p;
  memset(&p, 0, sizeof(p));
  p.g = a.g;
  p.Lq = a.Lq;
  p.SR = a.SR;
  p.G = 128 / a.SR;
  p.kept_off = a.kept_off;
  p.k2q_num = a.k2q_num;
  p.k2q_idx = a.k2q_idx;
  p.lse = a.lse;
  p.Dvec = a.Dvec;
  p.dQacc = a.dQacc;
  p.dK = a.dK;
  p.dV = a.dV;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.scale = a.scale;
  if (!make_map_2d(&p.mQs, a.Qs, a.d, rows, a.SR)) return cudaErrorInvalidValue;
  if (!make_map_2d(&p.mdOs, a.dOs, a.d, rows, a.SR)) return cudaErrorInvalidValue;
  if (!make_map_5d(&p.mK, a.K, a.g, a.d, a.BH)) return cudaErrorInvalidValue;
  if (!make_map_5d(&p.mV, a.V, a.g, a.d, a.BH)) return cudaErrorInvalidValue;
  if (a.d == 128 && a.g.BT == 64) return run_bwd<128, 64>(p, a.BH, st);
  if (a.d == 128 && a.g.BT == 32) return run_bwd<128, 32>(p, a.BH, st);
  if (a.d == 64 && a.g.BT == 64) return run_bwd<64, 64>(p, a.BH, st);
  if (a.d == 64 && a.g.BT == 32) return run_bwd<64, 32>(p, a.BH, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_bwd_finalize(const BwdArgs& a, cudaStream_t st) {
  const size_t rows = static_cast<size_t>(a.BH) * a.Lq;
  size_t tz = static_cast<size_t>(a.BH) * a.g.L * (a.d / 8);
  k_bwd_zero_pruned<<<static_cast<unsigned>((tz + 255) / 256), 256, 0, st>>>(a.BH, a.g.L, a.d, a.donor, a.dQ);
  size_t tf = rows * (a.d / 8);
  k_bwd_finalize<<<static_cast<unsigned>((tf + 255) / 256), 256, 0, st>>>(a.BH, a.g.L, a.Lq, a.d, a.scale, a.kept_tok,
                                                                          a.dQacc, a.dQ);
  return cudaGetLastError();
}

}  // namespace bsa
