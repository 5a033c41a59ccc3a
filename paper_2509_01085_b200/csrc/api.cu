// api.cu — the extern "C" boundary of libbsa.so (declared and documented in include/bsa.h).
// Validates every argument on the host, sizes workspaces, and enqueues the kernels of
// select.cu / attn_fwd.cu / attn_bwd.cu on the caller's stream. Never allocates or synchronises.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include "../../include/bsa.h"
#include "kernels.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(BSA_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// ---- instrumentation: launch counter (always) and optional per-kernel CUDA events
struct TimedRec {
  int id;
  cudaEvent_t a, b;
};
// Process-wide (autograd runs the backward on its own worker thread, which must be counted and timed too).
std::atomic<int64_t> g_launches{0};
std::atomic<int> g_bwd_path{BSA_BWD_REDUCE};  // bsa_set_bwd_path
std::atomic<int> g_fwd_min_slot{-1};          // bsa_set_fwd_tiling (-1: not set, the environment decides)
std::atomic<int> g_fwd_order{-1};
std::atomic<bool> g_timing{false};
std::mutex g_recs_mu;
std::vector<TimedRec> g_recs;

// Runs one launcher (which may enqueue `nk` kernels) under kernel id `id`.
template <class F>
cudaError_t timed(int id, int nk, cudaStream_t st, F&& f) {
  g_launches += nk;
  if (!g_timing.load(std::memory_order_relaxed)) return f();
  TimedRec r{id, nullptr, nullptr};
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, st);
  cudaError_t e = f();
  cudaEventRecord(r.b, st);
  std::lock_guard<std::mutex> lk(g_recs_mu);
  g_recs.push_back(r);
  return e;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// A strided [B, Hh, L, d] operand (include/bsa.h bsa_tensor) -> kernel view. NULL pointers pass when !required.
int check_tensor(const bsa_tensor& t, const char* name, int Hh, int d, bool required, bsa::Rows* out) {
  if (!t.ptr) {
    if (required) return fail(BSA_ERR_SELECTION_MISMATCH, "tensor %s is NULL", name);
    *out = bsa::Rows{nullptr, 0, 0, 0, Hh};
    return BSA_OK;
  }
  if (!aligned16(t.ptr)) return fail(BSA_ERR_INVALID_SHAPE, "tensor %s is not 16-byte aligned", name);
  if (t.sb < 0 || t.sh < 0 || t.sl < d || (t.sb | t.sh | t.sl) & 7 || t.sb >= (1LL << 38) || t.sh >= (1LL << 38) ||
      t.sl >= (1LL << 30))
    return fail(BSA_ERR_INVALID_SHAPE,
                "tensor %s: strides (sb, sh, sl) = (%lld, %lld, %lld) must be non-negative multiples of 8 elements "
                "with sl >= d = %d", name, (long long)t.sb, (long long)t.sh, (long long)t.sl, d);
  *out = bsa::Rows{static_cast<bsa::bf16*>(t.ptr), t.sb, t.sh, t.sl, Hh};
  return BSA_OK;
}

// Host geometry + validation shared by every entry point.
int check_geom(const bsa_geom* g, bsa::Geo* out) {
  if (!g) return fail(BSA_ERR_INVALID_SHAPE, "geometry is NULL");
  if (g->T < 1 || g->H < 1 || g->W < 1 || g->ct < 1 || g->ch < 1 || g->cw < 1)
    return fail(BSA_ERR_INVALID_SHAPE, "grid and block extents must be >= 1 (got T,H,W=%d,%d,%d block=%d,%d,%d)",
                g->T, g->H, g->W, g->ct, g->ch, g->cw);
  if (g->ut < 0 || g->uh < 0 || g->uw < 0) return fail(BSA_ERR_CONFIG, "unit dims must be >= 0");
  int ut = g->ut ? g->ut : g->ct, uh = g->uh ? g->uh : g->ch, uw = g->uw ? g->uw : g->cw;
  if (g->ct % ut || g->ch % uh || g->cw % uw)
    return fail(BSA_ERR_CONFIG, "unit (%d,%d,%d) must divide the block (%d,%d,%d) (P:168 'evenly dividing')", ut, uh,
                uw, g->ct, g->ch, g->cw);
  long long L = 1LL * g->T * g->H * g->W;
  if (L > (1LL << 30)) return fail(BSA_ERR_INVALID_SHAPE, "L too large");
  if (g->ct * g->ch * g->cw > 128) return fail(BSA_ERR_INVALID_SHAPE, "block of more than 128 tokens");
  *out = bsa::make_geo(g->T, g->H, g->W, g->ct, g->ch, g->cw, g->ut, g->uh, g->uw);
  return BSA_OK;
}

int check_r(double r) {
  if (!(r > 0.0 && r <= 1.0)) return fail(BSA_ERR_CONFIG, "r must be in (0,1] (got %g)", r);
  return BSA_OK;
}

int check_dims(int B, int Hh, int d) {
  if (B < 1 || Hh < 1) return fail(BSA_ERR_INVALID_SHAPE, "B and Hh must be >= 1");
  if (d != 64 && d != 128) return fail(BSA_ERR_INVALID_SHAPE, "d must be 64 or 128 (got %d)", d);
  return BSA_OK;
}

int check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(BSA_ERR_UNSUPPORTED_DEVICE, "libbsa is built for sm_100a (B200); device %d is sm_%d%d", dev, major,
                minor);
  return BSA_OK;
}

void host_sizes(const bsa::Geo& g, double r, int* Lq, int* maxk) {
  int s = 0, m = 0;
  for (int b = 0; b < g.N; ++b) {
    int k = bsa::block_kept(g, bsa::block_box(g, b), r);
    s += k;
    if (k > m) m = k;
  }
  *Lq = s;
  *maxk = m;
}

struct SelKvWs {
  size_t kc, qc, s, bits, kvbits, ovf, total;
};
SelKvWs selkv_ws(const bsa::Geo& g, size_t BH, int d) {
  SelKvWs w;
  size_t N = g.N, NW = (N + 31) / 32;
  w.kc = 0;
  w.qc = w.kc + align256(BH * N * d * 8);
  w.s = w.qc + align256(BH * N * d * 8);
  w.bits = w.s + align256(BH * N * N * 8);
  w.kvbits = w.bits + align256(BH * N * NW * 4);  // admission row bitmaps
  w.ovf = w.kvbits + align256(BH * N * NW * 4);   // their transpose
  w.total = w.ovf + align256((BH * N + 1) * 4);  // overflow row list of the warp admission kernel
  return w;
}

// Forward tiles grouped by KV-list similarity (group.cu): opt-in with BSA_FWD_GROUPING=1 in the environment.
// Measured at 32k: attn_fwd 0.866 -> 0.752 ms with grouped tiles, but the grouping kernels
// cost 0.147 ms, so consecutive query blocks per tile stay the default.
bool fwd_grouping() {
  static const bool on = [] {
    const char* e = std::getenv("BSA_FWD_GROUPING");
    return e && e[0] == '1';
  }();
  return on;
}

// Packed forward tiles (attn_fwd.cu k_fwd_union): a query block takes its kept count rounded up to a power of
// two >= 16 rows, tiles of the smallest slots first. Measured (attn_fwd ms, unpacked -> packed):
// 32k 0.814 -> 0.799, 75k 10.02 -> 9.65, 147k 31.88 -> 31.32, own dense path 9.09 -> 7.53. An 8-row minimum packs
// 16 ragged blocks per tile, whose KV union grows as fast as the rows shrink (32k 0.826, 147k 32.00).
// BSA_FWD_PACK=0 (one SR-row slot per block), =8 (8-row minimum), BSA_FWD_ORDER=large: the alternatives.
int env_flag(const char* name, const char* on_value) {
  const char* e = std::getenv(name);
  return e && std::strcmp(e, on_value) == 0;
}

// Forward workspace: K|V block images (always) + gathered Q^s (only used when q_packed is NULL) + the tile
// grouping's scratch and tile table (G >= 2).
struct FwdWs {
  size_t kv, qs, grp, perm, ul, uc, ctr, tab, tcount, total;
};
FwdWs fwd_ws(const bsa::Geo& g, size_t BH, size_t Lq, int d, int SR) {
  FwdWs w;
  const int G = 128 / SR;
  w.kv = 0;
  w.qs = w.kv + align256(BH * g.N * 2 * static_cast<size_t>(g.BT) * d * 2);
  w.grp = w.qs + align256(BH * Lq * d * 2);
  w.perm = w.grp + align256(G >= 2 ? bsa::group_ws_bytes(g.N, static_cast<int>(BH)) : 0);
  w.ul = w.perm + align256(G >= 2 ? BH * static_cast<size_t>(bsa::group_ntiles(g.N, G)) * G * 4 : 0);
  // union lists of the forward tiles (enough for the grouped tiling, which has the most tiles)
  const size_t ntiles = std::max(static_cast<size_t>(G >= 2 ? bsa::group_ntiles(g.N, G) : 0),
                                 static_cast<size_t>(bsa::fwd_max_tiles(g.N, SR)));
  w.uc = w.ul + align256(BH * ntiles * g.N * 4);
  w.ctr = w.uc + align256(BH * ntiles * 4);
  w.tab = w.ctr + 256;  // packed tile entries, then their count
  w.tcount = w.tab + align256(ntiles * 16 * 4);
  w.total = w.tcount + 256;
  return w;
}

// Backward workspace: gathered Q^s (only when q_packed is NULL), Q^s|dO^s query-block images
// (N * SR padded rows per head), D = rowsum(dO^s O^s), fp32 dQ accumulator.
// dS path capacity (admitted (query block, KV block) pairs whose bf16 dS tiles the workspace holds): a pair
// density of 1/8 (the paper's settings admit ~4-8% of the pairs), at most 24 GiB of tiles. A
// selection with more pairs takes the reduce path (fp32 dQ partials reduced in L2); the switch is on the device.
long long ds_capacity(const bsa::Geo& g, size_t BH, int SR) {
  const long long per_row = std::max<long long>(8, (g.N + 7) / 8);
  const long long dens = static_cast<long long>(BH) * g.N * per_row;
  const long long bytes_cap = (24LL << 30) / (static_cast<long long>(SR) * 128);
  return std::min(dens, bytes_cap);
}
struct BwdWs {
  size_t qs, img, dv, dq, ctr, qoff, ord, ptot, slot, ds, total;
  long long cap;
};
BwdWs bwd_ws(const bsa::Geo& g, size_t BH, size_t Lq, int SR, int d) {
  BwdWs w;
  w.qs = 0;
  w.img = w.qs + align256(BH * Lq * d * 2);
  w.dv = w.img + align256(BH * g.N * static_cast<size_t>(SR) * d * 4);
  w.dq = w.dv + align256(BH * g.N * static_cast<size_t>(SR) * 8);
  w.ctr = w.dq + align256(BH * Lq * d * 4);
  w.qoff = w.ctr + align256(BH * 4);  // work counters of the main kernel (one per launch, <= B <= BH)
  w.ord = w.qoff + align256(BH * g.N * 4);  // the main kernel's claim order
  w.ptot = w.ord + align256(BH * g.N * 4);
  w.slot = w.ptot + align256((BH + 1) * 4);  // per-head pair counts, then the total
  const bool ds = g_bwd_path.load() == BSA_BWD_DS;
  w.ds = w.slot + (ds ? align256(BH * g.N * static_cast<size_t>(g.N) * 4) : 0);
  // the dS region only under BSA_BWD_DS (24 GiB at the 147k workload otherwise allocated for nothing): a layer
  // must be built after bsa_set_bwd_path; a too-small workspace is rejected by bsa_attn_bwd
  w.cap = ds ? ds_capacity(g, BH, SR) : 0;
  w.total = w.ds + align256(static_cast<size_t>(w.cap) * SR * 128);
  return w;
}

int check_attn_geom(const bsa::Geo& G, double r, int* Lq, int* SR) {
  if (G.BT != 32 && G.BT != 64)
    return fail(BSA_ERR_INVALID_SHAPE, "attention kernels need ct*ch*cw in {32, 64} (got %d)", G.BT);
  if (G.N > 4096) return fail(BSA_ERR_INVALID_SHAPE, "attention kernels need N <= 4096 blocks (got %d)", G.N);
  int maxk = 0;
  host_sizes(G, r, Lq, &maxk);
  *SR = bsa::slot_rows(maxk);
  if (*SR > 128) return fail(BSA_ERR_INVALID_SHAPE, "more than 128 kept queries per block");
  return BSA_OK;
}

// Eq.3's U(1 - k/n) with the argument clamped to [1/(2n), 1 - 1/(2n)] (reading C14).
double eq3_z(int k, int N) {
  double u = 1.0 - static_cast<double>(k) / N;
  const double lo = 1.0 / (2.0 * N), hi = 1.0 - 1.0 / (2.0 * N);
  u = u < lo ? lo : (u > hi ? hi : u);
  return bsa::normal_quantile(u);
}

}  // namespace

#define CHECK(x)                 \
  do {                           \
    int _rc = (x);               \
    if (_rc != BSA_OK) return _rc; \
  } while (0)

extern "C" {

int bsa_version(void) { return 2; }

int bsa_resolve_k(double f, int32_t N, int32_t* k) {
  if (N < 1) return fail(BSA_ERR_INVALID_SHAPE, "N must be >= 1 (got %d)", N);
  if (!(f > 0.0 && f <= 1.0)) return fail(BSA_ERR_CONFIG, "key fraction f must be in (0,1] (got %g)", f);
  if (!k) return fail(BSA_ERR_SELECTION_MISMATCH, "k is NULL");
  *k = bsa::keep_count(f, N);
  return BSA_OK;
}

int bsa_kv_quantile(int32_t k, int32_t N, double* z) {
  if (N < 1) return fail(BSA_ERR_INVALID_SHAPE, "N must be >= 1 (got %d)", N);
  if (k < 1 || k > N) return fail(BSA_ERR_CONFIG, "k must be in [1, N=%d] (got %d)", N, k);
  if (!z) return fail(BSA_ERR_SELECTION_MISMATCH, "z is NULL");
  *z = eq3_z(k, N);
  return BSA_OK;
}

const char* bsa_strerror(int s) {
  switch (s) {
    case BSA_OK: return "ok";
    case BSA_ERR_INVALID_SHAPE: return "invalid shape";
    case BSA_ERR_CONFIG: return "invalid configuration";
    case BSA_ERR_SELECTION_MISMATCH: return "selection / buffer mismatch";
    case BSA_ERR_UNSUPPORTED_DEVICE: return "unsupported device (needs sm_100a)";
    case BSA_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

const char* bsa_last_error(void) { return g_last_error.c_str(); }

int bsa_sizes(const bsa_geom* g, double r, int32_t* N, int32_t* Lq, int32_t* max_block_kept) {
  bsa::Geo G;
  CHECK(check_geom(g, &G));
  CHECK(check_r(r));
  int lq = 0, mk = 0;
  host_sizes(G, r, &lq, &mk);
  if (N) *N = G.N;
  if (Lq) *Lq = lq;
  if (max_block_kept) *max_block_kept = mk;
  return BSA_OK;
}

int bsa_workspace_bytes(int op, const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, size_t* bytes) {
  bsa::Geo G;
  CHECK(check_geom(g, &G));
  CHECK(check_dims(B, Hh, d));
  if (!bytes) return fail(BSA_ERR_SELECTION_MISMATCH, "bytes is NULL");
  size_t BH = static_cast<size_t>(B) * Hh;
  if (op == BSA_OP_SELECT_KV) {
    *bytes = selkv_ws(G, BH, d).total;
    return BSA_OK;
  }
  CHECK(check_r(r));
  int lq = 0, mk = 0;
  host_sizes(G, r, &lq, &mk);
  if (op == BSA_OP_ATTN_FWD) {
    *bytes = fwd_ws(G, BH, lq, d, bsa::slot_rows(mk)).total;
    return BSA_OK;
  }
  if (op == BSA_OP_ATTN_BWD) {
    *bytes = bwd_ws(G, BH, lq, bsa::slot_rows(mk), d).total;
    return BSA_OK;
  }
  return fail(BSA_ERR_CONFIG, "unknown op %d", op);
}

int bsa_bwd_ds_capacity(const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, int64_t* pairs) {
  bsa::Geo G;
  CHECK(check_geom(g, &G));
  CHECK(check_dims(B, Hh, d));
  CHECK(check_r(r));
  if (!pairs) return fail(BSA_ERR_SELECTION_MISMATCH, "pairs is NULL");
  int lq = 0, mk = 0;
  host_sizes(G, r, &lq, &mk);
  *pairs = g_bwd_path.load() != BSA_BWD_DS ? -1 : bwd_ws(G, static_cast<size_t>(B) * Hh, lq, bsa::slot_rows(mk), d).cap;
  return BSA_OK;
}

int bsa_block_partition(const bsa_geom* g, double r, int32_t* block_off, int32_t* block_tok, int32_t* block_ext,
                        int32_t* kept_off, void* stream) {
  bsa::Geo G;
  CHECK(check_geom(g, &G));
  CHECK(check_r(r));
  CHECK(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = timed(BSA_K_PARTITION, (block_tok ? 1 : 0) + ((block_off || block_ext || kept_off) ? 1 : 0), st,
                        [&] { return bsa::launch_partition(G, r, block_off, block_tok, block_ext, kept_off, st); });
  if (e != cudaSuccess) return cuda_fail(e, "partition");
  return BSA_OK;
}

int bsa_select_queries(const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q,
                       const int32_t* kept_off, int32_t* kept_tok, int32_t* donor, double* q_pooled, void* q_packed,
                       void* stream) {
  bsa::Geo G;
  CHECK(check_geom(g, &G));
  CHECK(check_r(r));
  CHECK(check_dims(B, Hh, d));
  bsa::Rows Qv;
  CHECK(check_tensor(Q, "Q", Hh, d, true, &Qv));
  if (!kept_off || !kept_tok || !donor)
    return fail(BSA_ERR_SELECTION_MISMATCH, "kept_off, kept_tok and donor are required");
  if (q_packed && !aligned16(q_packed)) return fail(BSA_ERR_INVALID_SHAPE, "misaligned q_packed");
  CHECK(check_device());
  int lq = 0, mk = 0;
  host_sizes(G, r, &lq, &mk);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = timed(BSA_K_SELECT_Q, 1, st, [&] {
    return bsa::launch_select_queries(G, r, B * Hh, d, lq, Qv, kept_off, kept_tok, donor, q_pooled,
                                      static_cast<bsa::bf16*>(q_packed), st);
  });
  if (e != cudaSuccess) return cuda_fail(e, "select_queries");
  return BSA_OK;
}

int bsa_select_kv_blocks(const bsa_geom* g, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q, const double* q_pooled,
                         bsa_tensor K, int32_t k, double tau, int32_t* q2k_num, int32_t* q2k_idx, int32_t* k2q_num,
                         int32_t* k2q_idx, double* thresh, void* ws, size_t ws_bytes, void* stream) {
  return bsa_select_kv_blocks_ex(g, B, Hh, d, Q, q_pooled, K, k, tau, BSA_KV_TWO_STAGE, q2k_num, q2k_idx, k2q_num,
                                 k2q_idx, thresh, ws, ws_bytes, stream);
}

int bsa_select_kv_blocks_ex(const bsa_geom* g, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q,
                            const double* q_pooled, bsa_tensor K, int32_t k, double tau, int32_t mode,
                            int32_t* q2k_num, int32_t* q2k_idx, int32_t* k2q_num, int32_t* k2q_idx, double* thresh,
                            void* ws, size_t ws_bytes, void* stream) {
  if (mode != BSA_KV_TWO_STAGE && mode != BSA_KV_UNIFIED_PROB) return fail(BSA_ERR_CONFIG, "unknown KV mode %d", mode);
  bsa::Geo G;
  CHECK(check_geom(g, &G));
  CHECK(check_dims(B, Hh, d));
  if (G.N > 4096)
    return fail(BSA_ERR_INVALID_SHAPE, "KV selection supports N <= 4096 blocks (got %d)", G.N);
  if (k < 1 || k > G.N) return fail(BSA_ERR_CONFIG, "k must be in [1, N=%d] (got %d)", G.N, k);
  if (!(tau > 0.0 && tau <= 1.0)) return fail(BSA_ERR_CONFIG, "tau must be in (0,1] (got %g)", tau);
  bsa::Rows Qv, Kv;
  CHECK(check_tensor(K, "K", Hh, d, true, &Kv));
  CHECK(check_tensor(Q, "Q", Hh, d, q_pooled == nullptr, &Qv));
  if (!q2k_num || !q2k_idx) return fail(BSA_ERR_SELECTION_MISMATCH, "q2k_num and q2k_idx are required");
  if ((k2q_num == nullptr) != (k2q_idx == nullptr))
    return fail(BSA_ERR_SELECTION_MISMATCH, "k2q_num and k2q_idx must be both given or both NULL");
  size_t BH = static_cast<size_t>(B) * Hh;
  SelKvWs w = selkv_ws(G, BH, d);
  if (!ws || ws_bytes < w.total)
    return fail(BSA_ERR_SELECTION_MISMATCH, "workspace of %zu bytes < required %zu", ws_bytes, w.total);
  CHECK(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  double* Kc = reinterpret_cast<double*>(base + w.kc);
  double* Qc = q_pooled ? const_cast<double*>(q_pooled) : reinterpret_cast<double*>(base + w.qc);
  double* S = reinterpret_cast<double*>(base + w.s);
  uint32_t* bits = reinterpret_cast<uint32_t*>(base + w.bits);
  int* ovf = reinterpret_cast<int*>(base + w.ovf);
  cudaError_t e = timed(BSA_K_POOL, 1, st, [&] {
    return bsa::launch_pool(G, static_cast<int>(BH), d, Kv, Kc, st);
  });
  if (e == cudaSuccess && !q_pooled)
    e = timed(BSA_K_POOL, 1, st, [&] { return bsa::launch_pool(G, static_cast<int>(BH), d, Qv, Qc, st); });
  if (e == cudaSuccess)
    e = timed(BSA_K_SCORES, 1, st, [&] { return bsa::launch_scores(G.N, static_cast<int>(BH), d, Qc, Kc, S, st); });
  const double z = (k < G.N || mode == BSA_KV_UNIFIED_PROB) ? eq3_z(k, G.N) : 0.0;  // unified: no k = N bypass
  if (e == cudaSuccess)
    e = timed(BSA_K_ADMIT, (k < G.N && mode == BSA_KV_TWO_STAGE) ? 2 : 1, st, [&] {
      return bsa::launch_admit(G.N, static_cast<int>(BH), S, k, z, tau, mode == BSA_KV_UNIFIED_PROB ? 1 : 0, q2k_num,
                               q2k_idx, thresh, bits, ovf, st);
    });
  if (e == cudaSuccess && k2q_num)
    e = timed(BSA_K_K2Q, 2, st, [&] {
      return bsa::launch_k2q(G.N, static_cast<int>(BH), bits, reinterpret_cast<uint32_t*>(base + w.kvbits), k2q_num,
                             k2q_idx, st);
    });
  if (e != cudaSuccess) return cuda_fail(e, "select_kv_blocks");
  return BSA_OK;
}

int bsa_attn_fwd(const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q, bsa_tensor K,
                 bsa_tensor V, const void* q_packed, const int32_t* kept_off, const int32_t* kept_tok,
                 const int32_t* donor, const int32_t* q2k_num, const int32_t* q2k_idx, float scale, bsa_tensor O,
                 float* lse, void* ws, size_t ws_bytes, void* stream) {
  bsa::Geo G;
  CHECK(check_geom(g, &G));
  CHECK(check_r(r));
  CHECK(check_dims(B, Hh, d));
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(BSA_ERR_CONFIG, "scale must be positive and finite");
  bsa::Rows Qv, Kv, Vv, Ov;
  CHECK(check_tensor(Q, "Q", Hh, d, q_packed == nullptr, &Qv));
  CHECK(check_tensor(K, "K", Hh, d, true, &Kv));
  CHECK(check_tensor(V, "V", Hh, d, true, &Vv));
  CHECK(check_tensor(O, "O", Hh, d, true, &Ov));
  if (!kept_off || !kept_tok || !donor || !q2k_num || !q2k_idx || !lse)
    return fail(BSA_ERR_SELECTION_MISMATCH, "missing required pointer");
  if (q_packed && !aligned16(q_packed)) return fail(BSA_ERR_INVALID_SHAPE, "misaligned q_packed");
  int Lq = 0, SR = 0;
  CHECK(check_attn_geom(G, r, &Lq, &SR));
  size_t BH = static_cast<size_t>(B) * Hh;
  const bsa::bf16* Qs = static_cast<const bsa::bf16*>(q_packed);
  FwdWs w = fwd_ws(G, BH, Lq, d, SR);
  if (!ws || ws_bytes < w.total)
    return fail(BSA_ERR_SELECTION_MISMATCH, "workspace %zu < required %zu bytes", ws_bytes, w.total);
  CHECK(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint8_t* kv_img = base + w.kv;
  static const int no_pack = env_flag("BSA_FWD_PACK", "0"), pack8 = env_flag("BSA_FWD_PACK", "8"),
                   large_first = env_flag("BSA_FWD_ORDER", "large");
  const int min_slot = g_fwd_min_slot.load() >= 0 ? g_fwd_min_slot.load() : (no_pack ? 128 : (pack8 ? 8 : 0));
  bsa::FwdTiling tl;
  tl.kept_off = kept_off;
  tl.SR = SR;
  tl.pack_min = min_slot == 0 ? (SR < 16 ? SR : 16) : (min_slot < SR ? min_slot : SR);
  tl.small_first = g_fwd_order.load() >= 0 ? g_fwd_order.load() == BSA_FWD_SMALL_FIRST : !large_first;
  tl.max_tiles = bsa::fwd_max_tiles(G.N, SR);
  tl.tab = reinterpret_cast<int*>(base + w.tab);
  tl.tcount = reinterpret_cast<int*>(base + w.tcount);
  cudaError_t e = timed(BSA_K_KV_IMAGE, 1, st, [&] {
    return bsa::launch_kv_image(G, static_cast<int>(BH), d, Kv, Vv, kv_img, tl, st);
  });
  if (e == cudaSuccess && !Qs) {
    bsa::bf16* dst = reinterpret_cast<bsa::bf16*>(base + w.qs);
    e = timed(BSA_K_GATHER, 1, st, [&] {
      return bsa::launch_gather_rows(static_cast<int>(BH), Lq, d, Qv, kept_tok, dst, st);
    });
    Qs = dst;
  }
  bsa::FwdArgs a;
  a.g = G;
  a.BH = static_cast<int>(BH);
  a.d = d;
  a.Lq = Lq;
  a.SR = SR;
  a.K = Kv;
  a.V = Vv;
  a.Qs = Qs;
  a.kept_off = kept_off;
  a.kept_tok = kept_tok;
  a.donor = donor;
  a.q2k_num = q2k_num;
  a.q2k_idx = q2k_idx;
  a.scale = scale;
  a.O = Ov;
  a.lse = lse;
  a.kv_img = kv_img;
  a.perm = nullptr;
  a.ntiles = 0;
  const int Gt = 128 / SR;
  if (e == cudaSuccess && Gt >= 2 && fwd_grouping()) {
    int* perm = reinterpret_cast<int*>(base + w.perm);
    e = timed(BSA_K_GROUP, 3, st, [&] {
      return bsa::launch_group(G.N, static_cast<int>(BH), Gt, q2k_num, q2k_idx, base + w.grp, perm, st);
    });
    a.perm = perm;
    a.ntiles = bsa::group_ntiles(G.N, Gt);
  }
  a.ulists = reinterpret_cast<uint32_t*>(base + w.ul);
  a.ucount = reinterpret_cast<int*>(base + w.uc);
  a.work_ctr = reinterpret_cast<int*>(base + w.ctr);
  a.tab = tl.tab;
  a.tcount = tl.tcount;
  a.pack_min = tl.pack_min;
  if (e == cudaSuccess)
    e = timed(BSA_K_FWD_UNION, 1, st, [&] { return bsa::launch_fwd_union(a, a.ulists, a.ucount, st); });
  if (e == cudaSuccess) e = timed(BSA_K_ATTN_FWD, 1, st, [&] { return bsa::launch_attn_fwd(a, st); });
  if (e == cudaSuccess) e = timed(BSA_K_FILL, 1, st, [&] { return bsa::launch_fill(a.BH, G.L, d, donor, a.O, st); });
  if (e != cudaSuccess) return cuda_fail(e, "attn_fwd");
  return BSA_OK;
}

int bsa_attn_bwd(const bsa_geom* g, double r, int32_t B, int32_t Hh, int32_t d, bsa_tensor Q, bsa_tensor K,
                 bsa_tensor V, bsa_tensor O, bsa_tensor dO, const void* q_packed, const int32_t* kept_off,
                 const int32_t* kept_tok, const int32_t* donor, const int32_t* q2k_num, const int32_t* q2k_idx,
                 const int32_t* k2q_num, const int32_t* k2q_idx, const float* lse, float scale, bsa_tensor dQ,
                 bsa_tensor dK, bsa_tensor dV, void* ws, size_t ws_bytes, void* stream) {
  bsa::Geo G;
  CHECK(check_geom(g, &G));
  CHECK(check_r(r));
  CHECK(check_dims(B, Hh, d));
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(BSA_ERR_CONFIG, "scale must be positive and finite");
  bsa::Rows Qv, Kv, Vv, Ov, dOv, dQv, dKv, dVv;
  CHECK(check_tensor(Q, "Q", Hh, d, q_packed == nullptr, &Qv));
  CHECK(check_tensor(K, "K", Hh, d, true, &Kv));
  CHECK(check_tensor(V, "V", Hh, d, true, &Vv));
  CHECK(check_tensor(O, "O", Hh, d, true, &Ov));
  CHECK(check_tensor(dO, "dO", Hh, d, true, &dOv));
  CHECK(check_tensor(dQ, "dQ", Hh, d, true, &dQv));
  CHECK(check_tensor(dK, "dK", Hh, d, true, &dKv));
  CHECK(check_tensor(dV, "dV", Hh, d, true, &dVv));
  if (!kept_off || !kept_tok || !donor || !q2k_num || !q2k_idx || !k2q_num || !k2q_idx || !lse)
    return fail(BSA_ERR_SELECTION_MISMATCH, "missing required pointer");
  if (q_packed && !aligned16(q_packed)) return fail(BSA_ERR_INVALID_SHAPE, "misaligned q_packed");
  int Lq = 0, SR = 0;
  CHECK(check_attn_geom(G, r, &Lq, &SR));
  size_t BH = static_cast<size_t>(B) * Hh;
  BwdWs w = bwd_ws(G, BH, Lq, SR, d);
  if (!ws || ws_bytes < w.total)
    return fail(BSA_ERR_SELECTION_MISMATCH, "workspace of %zu bytes < required %zu", ws_bytes, w.total);
  CHECK(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  cudaError_t e = cudaSuccess;
  const bsa::bf16* Qs = static_cast<const bsa::bf16*>(q_packed);
  if (!Qs) {
    bsa::bf16* dst = reinterpret_cast<bsa::bf16*>(base + w.qs);
    e = timed(BSA_K_GATHER, 1, st, [&] {
      return bsa::launch_gather_rows(static_cast<int>(BH), Lq, d, Qv, kept_tok, dst, st);
    });
    Qs = dst;
  }
  bsa::BwdArgs a;
  a.g = G;
  a.B = B;
  a.Hh = Hh;
  a.BH = static_cast<int>(BH);
  a.d = d;
  a.Lq = Lq;
  a.SR = SR;
  a.K = Kv;
  a.V = Vv;
  a.O = Ov;
  a.dO = dOv;
  a.Qs = Qs;
  a.kept_off = kept_off;
  a.kept_tok = kept_tok;
  a.donor = donor;
  a.k2q_num = k2q_num;
  a.k2q_idx = k2q_idx;
  a.lse = lse;
  a.scale = scale;
  a.dQ = dQv;
  a.dK = dKv;
  a.dV = dVv;
  a.qdo_img = base + w.img;
  a.lsed = reinterpret_cast<float*>(base + w.dv);
  a.dQacc = reinterpret_cast<float*>(base + w.dq);
  a.work_ctr = reinterpret_cast<int*>(base + w.ctr);
  // longest-first claim order of the main kernel (BSA_BWD_ORDER=index: claim in index order)
  static const bool index_order = env_flag("BSA_BWD_ORDER", "index");
  static const int bwd_short_pct = [] {  // BSA_BWD_SHORT_PCT: percent of the items claimed last (default 5)
    const char* e = std::getenv("BSA_BWD_SHORT_PCT");
    const int v = e ? std::atoi(e) : 5;
    return v < 1 ? 1 : (v > 100 ? 100 : v);
  }();
  a.item_order = index_order ? nullptr : reinterpret_cast<int*>(base + w.ord);
  a.short_pct = bwd_short_pct;
  a.q2k_num = q2k_num;
  a.q2k_idx = q2k_idx;
  a.q2k_off = reinterpret_cast<int*>(base + w.qoff);
  a.pair_tot = reinterpret_cast<int*>(base + w.ptot);
  const bool ds_mode = g_bwd_path.load() == BSA_BWD_DS;
  a.pair_total = ds_mode ? a.pair_tot + BH : nullptr;  // NULL: reduce path, nothing for the device to decide
  a.k2q_slot = reinterpret_cast<int*>(base + w.slot);
  a.ds_buf = base + w.ds;
  a.ds_cap = w.cap;
  if (e == cudaSuccess && ds_mode) e = timed(BSA_K_BWD_PAIRS, 2, st, [&] { return bsa::launch_bwd_pairs(a, st); });
  if (e == cudaSuccess) e = timed(BSA_K_BWD_PREP, 1, st, [&] { return bsa::launch_bwd_prep(a, st); });
  const bool one_launch = (B == 1) || (Kv.sb == Hh * Kv.sh && Vv.sb == Hh * Vv.sh && dKv.sb == Hh * dKv.sh &&
                                       dVv.sb == Hh * dVv.sh);
  if (e == cudaSuccess)
    e = timed(BSA_K_ATTN_BWD, (ds_mode ? 2 : 1) * (one_launch ? 1 : B), st, [&] { return bsa::launch_bwd_main(a, st); });
  if (e == cudaSuccess) e = timed(BSA_K_BWD_FINAL, 1, st, [&] { return bsa::launch_bwd_finalize(a, st); });
  const bool k_uniform = (B == 1) || Kv.sb == Hh * Kv.sh;
  if (e == cudaSuccess && ds_mode)
    e = timed(BSA_K_BWD_DQ, k_uniform ? 1 : B, st, [&] { return bsa::launch_bwd_dq(a, st); });
  if (e != cudaSuccess) return cuda_fail(e, "attn_bwd");
  return BSA_OK;
}

int bsa_set_bwd_path(int mode) {
  if (mode != BSA_BWD_REDUCE && mode != BSA_BWD_DS) return fail(BSA_ERR_CONFIG, "unknown backward path %d", mode);
  g_bwd_path.store(mode);
  return BSA_OK;
}

int bsa_set_fwd_tiling(int min_slot_rows, int order) {
  if (min_slot_rows != 0 && min_slot_rows != 8 && min_slot_rows != 16 && min_slot_rows != 32 && min_slot_rows != 64 &&
      min_slot_rows != 128)
    return fail(BSA_ERR_CONFIG, "forward min slot rows must be 0, 8, 16, 32, 64 or 128 (got %d)", min_slot_rows);
  if (order != BSA_FWD_SMALL_FIRST && order != BSA_FWD_LARGE_FIRST)
    return fail(BSA_ERR_CONFIG, "unknown forward tile order %d", order);
  g_fwd_min_slot.store(min_slot_rows);
  g_fwd_order.store(order);
  return BSA_OK;
}

int64_t bsa_launch_count(void) { return g_launches.load(); }

int bsa_sp_relayout(int mode, int32_t B, int32_t Ls, int32_t Hh, int32_t d, int32_t P, const void* src, void* dst,
                    void* stream) {
  if (B < 1 || Ls < 1 || Hh < 1 || P < 1) return fail(BSA_ERR_INVALID_SHAPE, "B, Ls, Hh, P must be >= 1");
  if (d < 8 || d % 8) return fail(BSA_ERR_INVALID_SHAPE, "d must be a positive multiple of 8 (got %d)", d);
  if (Hh % P) return fail(BSA_ERR_CONFIG, "Hh = %d heads do not split over P = %d ranks", Hh, P);
  if (mode < BSA_SP_SEQ_TO_SEND || mode > BSA_SP_RECV_T_TO_SEQ) return fail(BSA_ERR_CONFIG, "unknown mode %d", mode);
  if (!src || !dst || !aligned16(src) || !aligned16(dst))
    return fail(BSA_ERR_INVALID_SHAPE, "src/dst must be non-NULL and 16-byte aligned");
  CHECK(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = timed(BSA_K_SP_RELAYOUT, 1, st, [&] { return bsa::launch_sp_relayout(mode, B, Ls, Hh, d, P, src, dst, st); });
  if (e != cudaSuccess) return cuda_fail(e, "sp_relayout");
  return BSA_OK;
}

int bsa_sp_relayout_group(int mode, int32_t Ls, int32_t Hh, int32_t d, int32_t P, int32_t hoff, int32_t Hs,
                          const void* src, void* dst, void* stream) {
  if (Ls < 1 || Hh < 1 || P < 1) return fail(BSA_ERR_INVALID_SHAPE, "Ls, Hh, P must be >= 1");
  if (d < 8 || d % 8) return fail(BSA_ERR_INVALID_SHAPE, "d must be a positive multiple of 8 (got %d)", d);
  if (Hh % P) return fail(BSA_ERR_CONFIG, "Hh = %d heads do not split over P = %d ranks", Hh, P);
  if (hoff < 0 || Hs < 1 || hoff + Hs > Hh / P)
    return fail(BSA_ERR_CONFIG, "head group [%d, %d) outside the %d heads of a rank", hoff, hoff + Hs, Hh / P);
  if (mode != BSA_SP_GROUP_SEND && mode != BSA_SP_GROUP_RECV) return fail(BSA_ERR_CONFIG, "unknown mode %d", mode);
  if (!src || !dst || !aligned16(src) || !aligned16(dst))
    return fail(BSA_ERR_INVALID_SHAPE, "src/dst must be non-NULL and 16-byte aligned");
  CHECK(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = timed(BSA_K_SP_RELAYOUT, 1, st, [&] {
    return bsa::launch_sp_group(mode == BSA_SP_GROUP_SEND ? 0 : 1, Ls, Hh, d, P, hoff, Hs, src, dst, st);
  });
  if (e != cudaSuccess) return cuda_fail(e, "sp_relayout_group");
  return BSA_OK;
}

// Debug aid (not in bsa.h): per-step timeline of one forward CTA, see attn_fwd.cu FWD_TRACE.
int bsa_debug_trace_fwd(void* dev_buf, int cta) {
  cudaError_t e = bsa::debug_trace_fwd(dev_buf, cta);
  return e == cudaSuccess ? BSA_OK : cuda_fail(e, "bsa_debug_trace_fwd");
}
int bsa_debug_progress_bwd(void* dev_ptr) {
  cudaError_t e = bsa::debug_progress_bwd(dev_ptr);
  return e == cudaSuccess ? BSA_OK : cuda_fail(e, "bsa_debug_progress_bwd");
}
int bsa_debug_trace_bwd(void* dev_buf, int cta) {
  cudaError_t e = bsa::debug_trace_bwd(dev_buf, cta);
  return e == cudaSuccess ? BSA_OK : cuda_fail(e, "bsa_debug_trace_bwd");
}

int bsa_timing_enable(int on) {
  g_timing = on != 0;
  return BSA_OK;
}

int bsa_timing_read(double* ms, int32_t* launches, int32_t n) {
  std::lock_guard<std::mutex> lk(g_recs_mu);
  if (ms)
    for (int i = 0; i < n; ++i) ms[i] = 0.0;
  if (launches)
    for (int i = 0; i < n; ++i) launches[i] = 0;
  int rc = BSA_OK;
  for (TimedRec& r : g_recs) {
    float t = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess && rc == BSA_OK) rc = cuda_fail(e, "bsa_timing_read");
    if (r.id < n) {
      if (ms) ms[r.id] += t;
      if (launches) launches[r.id] += 1;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_recs.clear();
  return rc;
}

}  // extern "C"
