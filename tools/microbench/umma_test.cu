// Scratch micro-test: validates the UMMA descriptor / TMA / TMEM conventions used by the BSA
// attention kernels against a CPU reference. Not part of the product.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;

// Q: [128][128] bf16 row-major (2D map, box 64x128)
// K,V: raster [T=4][H=4][W=8][d=128]; block 1 = (t 0..3, h 0..3, w 4..7) via 5D map box (64,4,4,4,1)
// P: [128][64] bf16 row-major (written by threads into swizzled smem)
// dO: [128][128] (2D map) ; dS: [128][64]
struct Out { float s[128*64]; float o[128*128]; float dvt[128*64]; float dq[128*128]; };

__global__ void __launch_bounds__(128, 1) k_test(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
    const __nv_bfloat16* P, const __nv_bfloat16* dS, float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;               // 32 KB : 2 blocks [128][64]
  uint8_t* sK = sQ + 32768;       // 16 KB : 2 blocks [64][64]
  uint8_t* sV = sK + 16384;       // 16 KB
  uint8_t* sdO = sV + 16384;      // 32 KB
  uint8_t* sP = sdO + 32768;      // 16 KB [128][64]
  uint8_t* sdS = sP + 16384;      // 16 KB
  __shared__ uint64_t bar_ld, bar_mma;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid / 32;
  if (tid == 0) { mbar_init(&bar_ld, 1); mbar_init(&bar_mma, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  // threads write P and dS (row = tid) into swizzled layout
  for (int c16 = 0; c16 < 8; ++c16) {
    const uint4* src = reinterpret_cast<const uint4*>(P + tid * 64 + c16 * 8);
    *reinterpret_cast<uint4*>(sP + sw128_off(tid, c16)) = *src;
    const uint4* src2 = reinterpret_cast<const uint4*>(dS + tid * 64 + c16 * 8);
    *reinterpret_cast<uint4*>(sdS + sw128_off(tid, c16)) = *src2;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tbase;
  if (tid == 0) {
    mbar_expect_tx(&bar_ld, 32768 + 16384 + 16384 + 32768);
    tma_load_2d(sQ, &mq, &bar_ld, 0, 0);
    tma_load_2d(sQ + 16384, &mq, &bar_ld, 64, 0);
    tma_load_5d(sK, &mk, &bar_ld, 0, 4, 0, 0, 0);
    tma_load_5d(sK + 8192, &mk, &bar_ld, 64, 4, 0, 0, 0);
    tma_load_5d(sV, &mv, &bar_ld, 0, 4, 0, 0, 0);
    tma_load_5d(sV + 8192, &mv, &bar_ld, 64, 4, 0, 0, 0);
    tma_load_2d(sdO, &mdo, &bar_ld, 0, 0);
    tma_load_2d(sdO + 16384, &mdo, &bar_ld, 64, 0);
    mbar_wait(&bar_ld, 0);
    tc_fence_after();
    // test1: S = Q K^T  (M=128,N=64, both K-major)
    uint32_t id1 = umma_idesc_bf16(128, 64, 0, 0);
    for (int k = 0; k < 8; ++k) {
      uint32_t blk = k / 4, kk = k % 4;
      uint64_t a = umma_desc_sw128(smem_u32(sQ + blk * 16384) + kk * 32, 16, 1024);
      uint64_t b = umma_desc_sw128(smem_u32(sK + blk * 8192) + kk * 32, 16, 1024);
      umma_ss(tb + 0, a, b, id1, k > 0);
    }
    // test2: O = P V (M=128, N=128, K=64); A=P K-major, B=V MN-major (LBO=8192 between d-chunks)
    uint32_t id2 = umma_idesc_bf16(128, 128, 0, 1);
    for (int k = 0; k < 4; ++k) {
      uint64_t a = umma_desc_sw128(smem_u32(sP) + k * 32, 16, 1024);
      uint64_t b = umma_desc_sw128(smem_u32(sV) + k * 2048, 8192, 1024);
      umma_ss(tb + 64, a, b, id2, k > 0);
    }
    // test3: dV^T = dO^T P  (M=d=128, N=64 keys, K=128 queries); A=dO MN-major (LBO=16384), B=P MN-major
    uint32_t id3 = umma_idesc_bf16(128, 64, 1, 1);
    for (int k = 0; k < 8; ++k) {
      uint64_t a = umma_desc_sw128(smem_u32(sdO) + k * 2048, 16384, 1024);
      uint64_t b = umma_desc_sw128(smem_u32(sP) + k * 2048, 8192, 1024);
      umma_ss(tb + 192, a, b, id3, k > 0);
    }
    // test4: dQ = dS K (M=128, N=128 (d), K=64 keys); A=dS K-major, B=K MN-major
    uint32_t id4 = umma_idesc_bf16(128, 128, 0, 1);
    for (int k = 0; k < 4; ++k) {
      uint64_t a = umma_desc_sw128(smem_u32(sdS) + k * 32, 16, 1024);
      uint64_t b = umma_desc_sw128(smem_u32(sK) + k * 2048, 8192, 1024);
      umma_ss(tb + 256, a, b, id4, k > 0);
    }
    umma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  int row = tid;
  uint32_t lane_base = tb + ((uint32_t)(warp * 32) << 16);
  float v[16];
  Out* o = reinterpret_cast<Out*>(out);
  for (int c = 0; c < 64; c += 16) { tmem_ld16(lane_base + 0 + c, v); tmem_wait_ld(); for (int i = 0; i < 16; ++i) o->s[row * 64 + c + i] = v[i]; }
  for (int c = 0; c < 128; c += 16) { tmem_ld16(lane_base + 64 + c, v); tmem_wait_ld(); for (int i = 0; i < 16; ++i) o->o[row * 128 + c + i] = v[i]; }
  for (int c = 0; c < 64; c += 16) { tmem_ld16(lane_base + 192 + c, v); tmem_wait_ld(); for (int i = 0; i < 16; ++i) o->dvt[row * 64 + c + i] = v[i]; }
  for (int c = 0; c < 128; c += 16) { tmem_ld16(lane_base + 256 + c, v); tmem_wait_ld(); for (int i = 0; i < 16; ++i) o->dq[row * 128 + c + i] = v[i]; }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static float bf(float x) { __nv_bfloat16 b = __float2bfloat16(x); return __bfloat162float(b); }

int main() {
  EncodeFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  srand(1);
  auto rnd = [] { return bf((rand() / (float)RAND_MAX) * 2.f - 1.f); };
  std::vector<float> Q(128 * 128), K(4 * 4 * 8 * 128), V(4 * 4 * 8 * 128), dO(128 * 128), P(128 * 64), dS(128 * 64);
  for (auto& x : Q) x = rnd(); for (auto& x : K) x = rnd(); for (auto& x : V) x = rnd();
  for (auto& x : dO) x = rnd(); for (auto& x : P) x = rnd(); for (auto& x : dS) x = rnd();
  auto up = [](const std::vector<float>& h) { std::vector<__nv_bfloat16> b(h.size()); for (size_t i = 0; i < h.size(); ++i) b[i] = __float2bfloat16(h[i]);
    void* d; cudaMalloc(&d, b.size() * 2); cudaMemcpy(d, b.data(), b.size() * 2, cudaMemcpyHostToDevice); return d; };
  void *dQ = up(Q), *dK = up(K), *dV = up(V), *ddO = up(dO), *dP = up(P), *ddS = up(dS);
  CUtensorMap mq, mk, mv, mdo;
  { cuuint64_t dims[2] = {128, 128}, str[1] = {256}; cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dQ, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&mdo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ddO, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  { cuuint64_t dims[5] = {128, 8, 4, 4, 1}, str[4] = {256, 256 * 8, 256 * 32, 256 * 128}; cuuint32_t box[5] = {64, 4, 4, 4, 1}, es[5] = {1, 1, 1, 1, 1};
    CUresult r1 = enc(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, dK, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(&mv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, dV, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d %d\n", r1, r2); }
  float* dout; cudaMalloc(&dout, sizeof(Out)); cudaMemset(dout, 0, sizeof(Out));
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k_test<<<1, 128, 140 * 1024>>>(mq, mk, mv, mdo, (const __nv_bfloat16*)dP, (const __nv_bfloat16*)ddS, dout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  Out* h = new Out; cudaMemcpy(h, dout, sizeof(Out), cudaMemcpyDeviceToHost);
  // key j of block 1 -> raster token (t, h, 4 + w), j = (t*4+h)*4+w
  auto kidx = [](int j) { int t = j / 16, hh = (j / 4) % 4, w = j % 4; return ((t * 4 + hh) * 8 + 4 + w) * 128; };
  double e1 = 0, e2 = 0, e3 = 0, e4 = 0;
  for (int i = 0; i < 128; ++i) for (int j = 0; j < 64; ++j) { double s = 0; for (int c = 0; c < 128; ++c) s += Q[i * 128 + c] * K[kidx(j) + c]; e1 = fmax(e1, fabs(s - h->s[i * 64 + j])); }
  for (int i = 0; i < 128; ++i) for (int c = 0; c < 128; ++c) { double s = 0; for (int j = 0; j < 64; ++j) s += P[i * 64 + j] * V[kidx(j) + c]; e2 = fmax(e2, fabs(s - h->o[i * 128 + c])); }
  for (int c = 0; c < 128; ++c) for (int j = 0; j < 64; ++j) { double s = 0; for (int i = 0; i < 128; ++i) s += dO[i * 128 + c] * P[i * 64 + j]; e3 = fmax(e3, fabs(s - h->dvt[c * 64 + j])); }
  for (int i = 0; i < 128; ++i) for (int c = 0; c < 128; ++c) { double s = 0; for (int j = 0; j < 64; ++j) s += dS[i * 64 + j] * K[kidx(j) + c]; e4 = fmax(e4, fabs(s - h->dq[i * 128 + c])); }
  printf("maxerr S=%g O=%g dVt=%g dQ=%g   (sample S[0]=%f O[0]=%f)\n", e1, e2, e3, e4, h->s[0], h->o[0]);
  printf("%s\n", (e1 < 1e-2 && e2 < 1e-2 && e3 < 1e-2 && e4 < 1e-2) ? "UMMA_TEST_PASS" : "UMMA_TEST_FAIL");
  return 0;
}
