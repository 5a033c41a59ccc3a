// kernels.h — internal launchers of libbsa (not part of the C ABI; see include/bsa.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "geom.cuh"

namespace bsa {

using bf16 = __nv_bfloat16;

// A [B, Hh, L, d] bf16 tensor given by element strides (include/bsa.h bsa_tensor; d contiguous): element
// (b, h, n, c) is p[b sb + h sh + n sl + c]. Kernels index heads by bh = b Hh + h.
struct Rows {
  bf16* p;
  long long sb, sh, sl;
  int Hh;
  __host__ __device__ __forceinline__ bf16* head(int bh) const {
    const int b = bh / Hh;
    return p + b * sb + static_cast<long long>(bh - b * Hh) * sh;
  }
  __host__ __device__ __forceinline__ bf16* row(int bh, long long n) const { return head(bh) + n * sl; }
};

// a1 partition
cudaError_t launch_partition(const Geo& g, double r, int* block_off, int* block_tok, int* block_ext, int* kept_off,
                             cudaStream_t st);
// a2+a3 query selection (one pass over Q)
cudaError_t launch_select_queries(const Geo& g, double r, int BH, int d, int Lq, Rows Q, const int* kept_off,
                                  int* kept_tok, int* donor, double* q_pooled, bf16* q_packed, cudaStream_t st);
// a2 block pooling in fp64
cudaError_t launch_pool(const Geo& g, int BH, int d, Rows X, double* Xc, cudaStream_t st);
// a4 pooled block scores S[bh][i][j] = Qc[i].Kc[j] / sqrt(d)
cudaError_t launch_scores(int N, int BH, int d, const double* Qc, const double* Kc, double* S, cudaStream_t st);
// a5+a6 threshold + admission per row; sets bit i of kvbits[bh][j] for every admitted (i, j)
cudaError_t launch_admit(int N, int BH, const double* S, int k, double z, double tau, int unified, int* q2k_num,
                         int* q2k_idx, double* thresh, uint32_t* qbits, int* ovf, cudaStream_t st);
// transpose of the admission: k2q lists (ascending query blocks per KV block)
cudaError_t launch_k2q(int N, int BH, const uint32_t* qbits, uint32_t* kvbits, int* k2q_num, int* k2q_idx,
                       cudaStream_t st);

// gather Q^s rows (kept queries) into packed [BH, Lq, d]
cudaError_t launch_gather_rows(int BH, int Lq, int d, Rows X, const int* kept_tok, bf16* out, cudaStream_t st);

// a7 forward: tcgen05 sparse attention over packed Q^s, then the donor fill
struct FwdArgs {
  Geo g;
  int BH, d, Lq, SR;  // SR = query rows per slot (power of two >= max kept per block)
  Rows K, V;         // raster, strided
  const bf16* Qs;     // packed [BH, Lq, d]
  const int* kept_off;
  const int* kept_tok;
  const int* donor;
  const int* q2k_num;
  const int* q2k_idx;
  float scale;
  Rows O;
  float* lse;
  const uint8_t* kv_img;  // workspace: K|V block images (launch_kv_image)
  const int* perm;        // [BH][ntiles][G] query blocks of each tile (launch_group), or NULL: packed tiles
  int ntiles;
  const int* tab;         // workspace: [fwd_max_tiles][16] packed tile entries (FwdTiling, launch_kv_image)
  const int* tcount;      // workspace: their count
  int pack_min;           // smallest packed slot (16 rows by default), or SR (one slot per block)
  uint32_t* ulists;       // workspace: [BH][ntiles][N] union entries per tile (launch_fwd_union)
  int* ucount;            // workspace: [BH][ntiles] their counts
  int* work_ctr;          // workspace: tile counter of the persistent forward
};
int fwd_max_tiles(int N, int SR);  // upper bound of the packed forward tiles per head
cudaError_t launch_fwd_union(const FwdArgs& a, uint32_t* ulists, int* ucount, cudaStream_t st);
// packed forward tiling (built by an extra CTA of the K|V image launch, attn_fwd.cu build_fwd_tiling)
struct FwdTiling {
  const int* kept_off;
  int SR, pack_min, small_first, max_tiles;
  int* tab;     // [max_tiles][16] query block | row offset << 16, -1 = empty
  int* tcount;  // tiles per head
};
cudaError_t launch_kv_image(const Geo& g, int BH, int d, Rows K, Rows V, uint8_t* img, const FwdTiling& tl,
                            cudaStream_t st);
cudaError_t launch_attn_fwd(const FwdArgs& a, cudaStream_t st);
cudaError_t debug_trace_fwd(void* dev_buf, int cta);
cudaError_t debug_trace_bwd(void* dev_buf, int cta);
cudaError_t debug_progress_bwd(void* dev_ptr);
cudaError_t launch_fill(int BH, int L, int d, const int* donor, Rows O, cudaStream_t st);

// forward tiles: query blocks with similar KV lists share a tile (group.cu)
size_t group_ws_bytes(int N, int BH);
int group_ntiles(int N, int G);
cudaError_t launch_group(int N, int BH, int G, const int* q2k_num, const int* q2k_idx, void* ws, int* perm,
                         cudaStream_t st);

// Ulysses sequence parallelism: row reorders around the all-to-all (sp.cu)
cudaError_t launch_sp_group(int mode, int Ls, int Hh, int d, int P, int hoff, int Hs, const void* src, void* dst,
                            cudaStream_t st);
cudaError_t launch_sp_relayout(int mode, int B, int Ls, int Hh, int d, int P, const void* src, void* dst,
                               cudaStream_t st);

// a8 backward
struct BwdArgs {
  Geo g;
  int B, Hh, BH, d, Lq, SR;
  Rows K, V, O, dO;    // raster, strided
  const bf16* Qs;      // packed
  const int* kept_off;
  const int* kept_tok;
  const int* donor;
  const int* k2q_num;
  const int* k2q_idx;
  const float* lse;
  float scale;
  Rows dQ, dK, dV;
  // workspace
  uint8_t* qdo_img;  // [BH, N] query-block images of Q^s|dO^s, SR*d*4 bytes each (k_bwd_prep)
  float* lsed;       // [BH, N, SR, 2]: per query block and row, LSE*log2(e) and D
  float* dQacc;  // [BH, Lq, d]
  int* work_ctr;  // [B] item counters of the persistent main kernel (one per launch)
  int* item_order;  // [BH * N] its claim order: the shortest short_pct % of the k2q lists last (launch_bwd_prep)
  int short_pct;
  // dS path (attn_bwd.cu): selection lists, pair slots, the path switch and the dS tile store
  const int* q2k_num;
  const int* q2k_idx;
  int* q2k_off;      // [BH, N] head-local exclusive scan of q2k_num
  int* pair_tot;     // [BH] pairs per head
  int* pair_total;   // [1] all pairs (dS path iff <= ds_cap)
  int* k2q_slot;     // [BH, N, N]
  uint8_t* ds_buf;   // ds_cap tiles of SR x 128 B
  long long ds_cap;
};
cudaError_t launch_bwd_pairs(const BwdArgs& a, cudaStream_t st);
cudaError_t launch_bwd_dq(const BwdArgs& a, cudaStream_t st);
cudaError_t launch_bwd_prep(const BwdArgs& a, cudaStream_t st);
cudaError_t launch_bwd_main(const BwdArgs& a, cudaStream_t st);
cudaError_t launch_bwd_finalize(const BwdArgs& a, cudaStream_t st);

// host helpers
double normal_quantile(double u);  // Phi^-1, Acklam initial guess + Halley refinement
int slot_rows(int max_block_kept);  // power of two >= max(8, max_block_kept)

}  // namespace bsa
