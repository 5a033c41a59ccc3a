/*
 * bsa.h — C ABI of libbsa.so, the B200 (sm_100a) implementation of the hot path of BSA,
 * "Bidirectional Sparse Attention" (arXiv 2509.01085, /root/reference/PAPER.md).
 *
 * The path has five calls, in the order a training step uses them:
 *   bsa_block_partition   3D block partition of the (T,H,W) token grid      (§3.2.1)
 *   bsa_select_queries    query pruning by cosine to the unit centre (Eq.2)  (§3.2.2)
 *   bsa_select_kv_blocks  statistical threshold (Eq.3) + cumulative admission (Eq.4) (§3.2.3)
 *   bsa_attn_fwd          block-sparse attention over kept queries x admitted KV blocks (Eq.5)
 *                         and the fill that restores length L
 *   bsa_attn_bwd          its gradient (semantics in DESIGN.md reading C10)
 *
 * Conventions (all calls):
 *  - Tensors Q, K, V, O, dO, dQ, dK, dV are bf16 [B, Hh, L, d] passed as a bsa_tensor: a device pointer and
 *    element strides (sb, sh, sl) of the batch, head and token dimensions; the d channels of a row are
 *    contiguous. The problem statement is per head, Q, K, V in R^{L x d}, so any layout whose
 *    rows of one head are evenly spaced works: contiguous [B, Hh, L, d] (sb = Hh L d, sh = L d, sl = d), a
 *    model's [B, L, Hh, d] (sb = L Hh d, sh = d, sl = Hh d), or Q/K/V views of a fused [B, L, 3, Hh, d]
 *    projection (sl = 3 Hh d). Tokens are in raster order n = t*H*W + h*W + w. d must be 64 or 128;
 *    pointers must be 16-byte aligned and strides positive multiples of 8 elements with sl >= d
 *    (BSA_ERR_INVALID_SHAPE otherwise). Output tensors must not overlap any input or each other.
 *    Index arrays are int32, device memory; q_pooled / q_packed / lse and all selection arrays are packed.
 *  - Ownership: the caller allocates every buffer (device unless stated) and passes a CUDA stream
 *    (cudaStream_t, passed as void*; NULL = legacy default stream). The library never allocates,
 *    frees or synchronises; every call only enqueues work on `stream` and returns. Calls are
 *    reentrant; the only global state is the thread-local last-error string and the opt-in
 *    instrumentation below (a launch counter and event timing).
 *  - Errors: every call returns BSA_OK (0) or an error code; argument validation happens before
 *    any launch, so nothing is written on a validation error. bsa_last_error() gives the message.
 *  - Geometry: grid (T,H,W), block (ct,ch,cw), query-selection unit (ut,uh,uw) (the paper's window
 *    (w_t,w_h,w_w)); ut=uh=uw=0 means unit = block (block-centre selection, the north_star
 *    default). Grids need not be divisible by the block: edge blocks are truncated (reading C1).
 *    Block ids are row-major over (ceil(T/ct), ceil(H/ch), ceil(W/cw)). KV selection and the attention
 *    kernels require N = number of blocks <= 4096 (BSA_ERR_INVALID_SHAPE otherwise); the attention kernels
 *    also require ct*ch*cw in {32, 64}.
 *  - r in (0,1] is the query keep ratio (Eq.2's retention ratio); a unit of n tokens keeps
 *    clamp(ceil(r*n - 1e-9), 1, n) queries (reading C6). k in [1,N] is Eq.3's key count (k = N turns
 *    the threshold off, reading C15); tau in (0,1] is Eq.4's cumulative-mass target (reading C17).
 */
#ifndef BSA_H_
#define BSA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum bsa_status {
  BSA_OK = 0,
  BSA_ERR_INVALID_SHAPE = 1,       /* zero extents, unsupported d or block size, misaligned pointer */
  BSA_ERR_CONFIG = 2,              /* r, k, tau, unit dims or scale out of range */
  BSA_ERR_SELECTION_MISMATCH = 3,  /* buffers/workspace sized for another geometry, or NULL */
  BSA_ERR_UNSUPPORTED_DEVICE = 4,  /* current device is not sm_100 */
  BSA_ERR_CUDA = 5                 /* a CUDA launch failed; message carries cudaGetErrorString */
};

/* A bf16 [B, Hh, L, d] tensor: element (b, h, n, c) at ((bf16*)ptr)[b*sb + h*sh + n*sl + c]. */
typedef struct bsa_tensor {
  void* ptr;
  int64_t sb, sh, sl;
} bsa_tensor;

typedef struct bsa_geom {
  int32_t T, H, W;    /* latent token grid */
  int32_t ct, ch, cw; /* cuboid block (C_t, C_h, C_w) */
  int32_t ut, uh, uw; /* selection unit (window); 0,0,0 = whole block */
} bsa_geom;

/* Workspace-using operations (bsa_workspace_bytes `op`). */
enum bsa_op { BSA_OP_SELECT_KV = 1, BSA_OP_ATTN_FWD = 2, BSA_OP_ATTN_BWD = 3 };

int bsa_version(void);
const char* bsa_strerror(int status);
/* Message of the last error raised on the calling thread ("" if none). */
const char* bsa_last_error(void);

/* Host-only: Eq.3's integer key count from a fraction, k = clamp(ceil(f*N - 1e-9), 1, N) (reading C6: plain fp
 * ceil is wrong, e.g. 0.07*100 = 7.000000000000001). f in (0,1], N >= 1; errors CONFIG / INVALID_SHAPE. */
int bsa_resolve_k(double f, int32_t N, int32_t* k);

/* Host-only: the z = U(1 - k/n) of Eq.3 that bsa_select_kv_blocks uses for (k, N): the standard
 * normal quantile (reading C14) of 1 - k/N clamped to [1/(2N), 1 - 1/(2N)] (Acklam's approximation refined by
 * two Halley steps on erfc). k in [1, N]; for k == N the threshold itself is bypassed (reading C15) but z is
 * still defined (it is what BSA_KV_UNIFIED_PROB uses). */
int bsa_kv_quantile(int32_t k, int32_t N, double* z);

/* Host-only sizes for allocation: N blocks, Lq kept queries per (b,h) (= sum over blocks of the
 * per-block kept counts, which depend only on geometry and r), and the largest per-block kept
 * count. Any output pointer may be NULL. */
int bsa_sizes(const bsa_geom* g, double r, int32_t* N, int32_t* Lq, int32_t* max_block_kept);

/* Bytes of device workspace `op` needs for this problem (0 is possible). */
int bsa_workspace_bytes(int op, const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, size_t* bytes);

/* a1 — 3D block partition. Writes, for the geometry and r:
 *   block_off[N+1]  prefix of block sizes (block b owns block_tok[block_off[b] .. block_off[b+1]))
 *   block_tok[L]    tokens of each block, ascending raster index inside a block
 *   block_ext[3N]   actual (truncated) extent (e_t, e_h, e_w) of each block
 *   kept_off[N+1]   prefix of per-block kept-query counts (packed-query row ranges)
 * Any output may be NULL (skipped). Deterministic; depends only on (g, r). */
int bsa_block_partition(const bsa_geom* g, double r, int32_t* block_off, int32_t* block_tok, int32_t* block_ext,
                        int32_t* kept_off, void* stream);

/* a2+a3 — query pruning (Eq.2) in one pass over Q.
 * For each unit: c_i = cos(q_centre, q_i) (centre = floor-midpoint of the unit's actual extent,
 * c_centre = 1, zero norm -> 0); tokens ordered by (c ascending, index ascending) and the first
 * clamp(ceil(r|u|-1e-9),1,|u|) are kept (rank of 1-cos descending, Eq.2 literal). Each pruned token
 * gets a donor: the kept token of its unit with the largest cosine to it (ties -> lowest index).
 * All decisions are taken in fp64 on the exact bf16 input values.
 *   kept_off   [N+1]          from bsa_block_partition (same g, r)
 *   kept_tok   [B,Hh,Lq] out  kept tokens, block-major, ascending inside each block
 *   donor      [B,Hh,L]  out  donor token of every token (itself if kept)
 *   q_pooled   [B,Hh,N,d] out fp64 block means of Q; may be NULL
 *   q_packed   [B,Hh,Lq,d] out bf16 rows of the kept queries in kept_tok order (Q^s); may be NULL */
int bsa_select_queries(const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q,
                       const int32_t* kept_off, int32_t* kept_tok, int32_t* donor, double* q_pooled, void* q_packed,
                       void* stream);

/* a2+a4+a5+a6 — KV-block selection (Eq.3, Eq.4) per (b,h, query block i):
 *   s_j = Qc[i].Kc[j]/sqrt(d) (fp64), mu/sigma population statistics over the N scores,
 *   k < N: p = mu + sigma * Phi^-1(clamp(1-k/N, 1/(2N), 1-1/(2N))), candidates C = {j: s_j >= p}
 *          (empty -> {argmax}); k == N: C = all blocks.
 *   Admit the shortest prefix of C ordered by (s desc, j asc) whose exp(s - max) mass reaches
 *   tau * total (tau >= 1: all of C).
 *   q_pooled  [B,Hh,N,d] fp64 from bsa_select_queries, or NULL (then Q is pooled here; else Q.ptr may be NULL)
 *   q2k_num   [B,Hh,N]   out |S_i|;   q2k_idx [B,Hh,N,N] out S_i ascending in row i's first q2k_num
 *                         entries (the rest is left unwritten)
 *   k2q_num   [B,Hh,N]   out number of query blocks admitting KV block j; k2q_idx [B,Hh,N,N] out
 *                         those query blocks ascending (the transpose, used by bsa_attn_bwd); both
 *                         may be NULL
 *   thresh    [B,Hh,N]   out p per row (-inf when k == N); may be NULL
 *   ws/ws_bytes          device workspace of at least bsa_workspace_bytes(BSA_OP_SELECT_KV, ...) */
int bsa_select_kv_blocks(const bsa_geom* g, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q, const double* q_pooled,
                         bsa_tensor K, int32_t k, double tau, int32_t* q2k_num, int32_t* q2k_idx, int32_t* k2q_num,
                         int32_t* k2q_idx, double* thresh, void* ws, size_t ws_bytes, void* stream);

/* Variant of bsa_select_kv_blocks with the reading of Eq.3/Eq.4 as a parameter (the north_star's
 * "selection variants" row; C17, C28):
 *   BSA_KV_TWO_STAGE     the library's reading (identical to bsa_select_kv_blocks): Eq.3's p thresholds the
 *                        raw scores into candidates, Eq.4 admits the shortest prefix of their softmax
 *                        reaching tau.
 *   BSA_KV_UNIFIED_PROB  SPEC's unified_prob: Eq.3 is taken over the softmax-normalised row,
 *                        p = mu + sigma Phi^-1(clamp(1 - k/N, 1/(2N), 1 - 1/(2N))) clamped to (0, 1] (no
 *                        k = N bypass), and Eq.4 admits the shortest prefix (s desc, j asc) of ALL blocks
 *                        whose probability mass reaches p; tau is ignored. thresh[row] = p.
 * The paper's "fixed threshold" KV variant (Table 2) is BSA_KV_TWO_STAGE with k = N. Other
 * arguments, ownership and errors as bsa_select_kv_blocks; an unknown mode is BSA_ERR_CONFIG. */
enum bsa_kv_mode { BSA_KV_TWO_STAGE = 0, BSA_KV_UNIFIED_PROB = 1 };
int bsa_select_kv_blocks_ex(const bsa_geom* g, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q,
                            const double* q_pooled, bsa_tensor K, int32_t k, double tau, int32_t mode,
                            int32_t* q2k_num, int32_t* q2k_idx, int32_t* k2q_num, int32_t* k2q_idx, double* thresh,
                            void* ws, size_t ws_bytes, void* stream);

/* a7 — sparse attention forward (Eq.5) + fill:
 *   for each kept query q of block i: O^s[q] = softmax(scale * q K_S^T) V_S over the tokens of the
 *   KV blocks admitted by i; O[kept] = O^s, O[pruned t] = O^s[donor(t)]; lse[q] = natural-log
 *   log-sum-exp of the scaled logits (packed order). bf16 tcgen05 MMAs, fp32 accumulation and
 *   online softmax.
 *   q_packed [B,Hh,Lq,d] Q^s from bsa_select_queries, or NULL (then gathered from Q into ws; Q.ptr may be NULL
 *            when q_packed is given)
 *   O        [B,Hh,L,d] out (strided);  lse [B,Hh,Lq] out fp32;  scale > 0 finite (1/sqrt(d)) */
int bsa_attn_fwd(const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q, bsa_tensor K,
                 bsa_tensor V, const void* q_packed, const int32_t* kept_off, const int32_t* kept_tok,
                 const int32_t* donor, const int32_t* q2k_num, const int32_t* q2k_idx, float scale, bsa_tensor O,
                 float* lse, void* ws, size_t ws_bytes, void* stream);

/* a8 — backward of bsa_attn_fwd with the selection held fixed (reading C10):
 *   dO^s[q] = dO[q] + sum of dO over the pruned tokens whose donor is q; D = rowsum(dO^s * O^s);
 *   dV, dK accumulate over admitting query blocks; dQ[kept] = scale * dS K, dQ[pruned] = 0;
 *   tokens of KV blocks no query block admitted get dK = dV = 0.
 *   O and lse are the outputs of bsa_attn_fwd; q2k_* and k2q_* from bsa_select_kv_blocks (both directions of
 *   the same selection: dK/dV walk k2q, dQ walks q2k).
 *   dQ, dK, dV [B,Hh,L,d] out bf16 (strided; Q.ptr may be NULL when q_packed is given).
 *   dQ is formed one of two ways, chosen on the device from the selection's number of admitted (query block,
 *   KV block) pairs against the workspace's capacity (a pair density of 1/8, at most 24 GiB):
 *     dS path (BSA_BWD_DS set and the pairs fit): the KV-stationary kernel stores every pair's bf16 dS tile and a query-stationary
 *       kernel forms dQ^T = sum_j K_j^T dS_ij^T in TMEM (fp32, ascending j: deterministic);
 *     reduce path (default; denser selections under BSA_BWD_DS): fp32 dQ partials, one per (query row block, admitted KV block), are
 *       reduced in L2 (cp.reduce.async.bulk.tensor) into an fp32 workspace: the summation order is not
 *       deterministic, so dQ may differ run to run in the last fp32 bits before the bf16 rounding. */
int bsa_attn_bwd(const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q, bsa_tensor K,
                 bsa_tensor V, bsa_tensor O, bsa_tensor dO, const void* q_packed, const int32_t* kept_off,
                 const int32_t* kept_tok, const int32_t* donor, const int32_t* q2k_num, const int32_t* q2k_idx,
                 const int32_t* k2q_num, const int32_t* k2q_idx, const float* lse, float scale, bsa_tensor dQ,
                 bsa_tensor dK, bsa_tensor dV, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- Ulysses sequence parallelism
 * (SURVEY.md §8(e) mode 2). A sequence-parallel model gives each of P ranks a contiguous
 * chunk of Ls = L/P raster tokens of all Hh heads, [B][Ls][Hh][d]. Selection needs every pooled block
 * of a head, so around BSA the caller runs one all-to-all (NCCL; equal contiguous
 * chunks of B*Hp*Ls*d elements, Hp = Hh/P) per tensor and this call reorders rows into and out of its
 * buffers (no arithmetic; bf16 rows of d channels, d % 8 == 0; src and dst must not overlap):
 *   BSA_SP_SEQ_TO_SEND    src [B][Ls][Hh][d]     -> dst [P][B][Hp][Ls][d]  (chunk p: head group p)
 *   BSA_SP_RECV_TO_HEADS  src [P][B][Hp][Ls][d]  -> dst [B][Hp][P*Ls][d]   (BSA layout, whole sequence)
 *   BSA_SP_HEADS_TO_SEND  src [B][Hp][P*Ls][d]   -> dst [P][B][Hp][Ls][d]  (chunk s: sequence chunk s)
 *   BSA_SP_RECV_TO_SEQ    src [P][B][Hp][Ls][d]  -> dst [B][Ls][Hh][d]     (back to the model layout)
 * Token-major variants (B = 1: the exchange then needs no reorder on the BSA side at all, because the received
 * [P][Ls][Hp][d] = [L][Hp][d] buffer is a strided [1, Hp, L, d] bsa_tensor (sh = d, sl = Hp d), and BSA's outputs
 * written in that layout are already the send buffer of the return exchange):
 *   BSA_SP_SEQ_TO_SEND_T  src [B][Ls][Hh][d]     -> dst [P][B][Ls][Hp][d]  (chunk p: head group p)
 *   BSA_SP_RECV_T_TO_SEQ  src [P][B][Ls][Hp][d]  -> dst [B][Ls][Hh][d]     (back to the model layout)
 * Errors: BSA_ERR_INVALID_SHAPE for non-positive sizes, d % 8 != 0 or misaligned pointers;
 * BSA_ERR_CONFIG for Hh % P != 0 or an unknown mode. */
enum bsa_sp_mode {
  BSA_SP_SEQ_TO_SEND = 0, BSA_SP_RECV_TO_HEADS = 1, BSA_SP_HEADS_TO_SEND = 2, BSA_SP_RECV_TO_SEQ = 3,
  BSA_SP_SEQ_TO_SEND_T = 4, BSA_SP_RECV_T_TO_SEQ = 5
};
int bsa_sp_relayout(int mode, int32_t B, int32_t Ls, int32_t Hh, int32_t d, int32_t P, const void* src, void* dst,
                    void* stream);
/* Head-group variant of the token-major exchange (B = 1), used to pipeline the exchange of head group g+1 with
 * the attention of group g: each rank's chunk carries heads [p Hp + hoff, p Hp + hoff + Hs) of its destination p
 * (Hp = Hh/P, 0 <= hoff, hoff + Hs <= Hp):
 *   BSA_SP_GROUP_SEND  src [Ls][Hh][d]                      -> dst [P][Ls][Hs][d]
 *   BSA_SP_GROUP_RECV  src [P][Ls][Hs][d]                   -> dst [Ls][Hh][d], only those heads written
 * Errors as bsa_sp_relayout; a group outside [0, Hp) is BSA_ERR_CONFIG. */
enum bsa_sp_group_mode { BSA_SP_GROUP_SEND = 0, BSA_SP_GROUP_RECV = 1 };
int bsa_sp_relayout_group(int mode, int32_t Ls, int32_t Hh, int32_t d, int32_t P, int32_t hoff, int32_t Hs,
                          const void* src, void* dst, void* stream);

/* ---------------------------------------------------------------- instrumentation (off the hot path)
 * Kernel ids reported by bsa_timing_read / counted by bsa_launch_count. */
enum bsa_kernel_id {
  BSA_K_PARTITION = 0, BSA_K_SELECT_Q, BSA_K_POOL, BSA_K_SCORES, BSA_K_ADMIT, BSA_K_K2Q, BSA_K_GATHER,
  BSA_K_ATTN_FWD, BSA_K_FILL, BSA_K_BWD_PREP, BSA_K_ATTN_BWD, BSA_K_BWD_FINAL, BSA_K_KV_IMAGE, BSA_K_SP_RELAYOUT,
  BSA_K_GROUP, BSA_K_BWD_PAIRS, BSA_K_BWD_DQ, BSA_K_FWD_UNION, BSA_K_COUNT
};
/* Backward dQ path (process-wide): BSA_BWD_REDUCE (default) always takes the reduce path; BSA_BWD_DS takes the
 * dS path whenever the selection's pairs fit (the device-side switch described at bsa_attn_bwd). The default is
 * the reduce path because it measured faster on the BASELINE workloads. Unknown mode:
 * BSA_ERR_CONFIG. */
enum bsa_bwd_path { BSA_BWD_REDUCE = 0, BSA_BWD_DS = 1 };
int bsa_set_bwd_path(int mode);
/* Forward query tiling (process-wide). A query block takes its kept count rounded up to a power of two rows, at
 * least min_slot_rows and at most SR (the largest kept count rounded up); blocks of one slot size fill 128-row
 * tiles in block order (PAPER.md P:204-210 leaves the tiling of the Q blocks to the kernel). min_slot_rows: 0 =
 * the default (16), 8, 16, 32, 64, or 128 (>= SR: one SR-row slot per block, i.e. 128/SR consecutive blocks per
 * tile). order: BSA_FWD_SMALL_FIRST (default: tiles of the smallest slots, which union the most KV lists, are
 * claimed first) or BSA_FWD_LARGE_FIRST. Results do not depend on either beyond fp32 summation order (each row's
 * softmax runs over its own admitted blocks). Other values: BSA_ERR_CONFIG. Overrides BSA_FWD_PACK /
 * BSA_FWD_ORDER from the environment. */
enum bsa_fwd_order { BSA_FWD_SMALL_FIRST = 0, BSA_FWD_LARGE_FIRST = 1 };
int bsa_set_fwd_tiling(int min_slot_rows, int order);
/* Capacity of the backward's dS path in admitted (query block, KV block) pairs for this geometry (-1 unless
 * BSA_BWD_DS is set): bsa_attn_bwd takes the dS path iff sum(q2k_num) <= *pairs. Errors as
 * bsa_workspace_bytes. */
int bsa_bwd_ds_capacity(const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, int64_t* pairs);
/* Total kernels launched through libbsa by this process (always counted; cheap). */
int64_t bsa_launch_count(void);
/* When enabled (process-wide: autograd runs the backward on its own thread), every libbsa kernel launch is
 * bracketed by a CUDA event pair recorded on the launch stream (events are created lazily; this is a
 * profiling aid, not for graph capture). */
int bsa_timing_enable(int on);
/* Synchronises on the recorded events, writes per-kernel-id summed milliseconds ms[id] and launch
 * counts launches[id] for id < n (either may be NULL), then clears the record. */
int bsa_timing_read(double* ms, int32_t* launches, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* BSA_H_ */
