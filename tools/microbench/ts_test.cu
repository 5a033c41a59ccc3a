// Scratch micro-test: tcgen05.mma with the A operand in TMEM (the ".kind::f16 [d], [a], b_desc" form).
// (a) S = Q K^T : A = Q [128 x 128] packed bf16x2 in TMEM (64 cols), B = K [64 x 128] K-major SW128 smem
// (b) O = P V   : A = P [128 x 64] packed in TMEM (32 cols),       B = V [64 x 128] MN-major SW128 smem
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;

__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__global__ void __launch_bounds__(128, 1) k_test(const __nv_bfloat16* Q, const __nv_bfloat16* K, const __nv_bfloat16* P,
                                                 const __nv_bfloat16* V, float* S_out, float* O_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;          // [64 keys][128 d] as 2 chunks of [64][64] SW128 (chunk stride 8 KB)
  uint8_t* sV = sm + 16384;  // same layout (rows = keys) read MN-major for PV
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tbase, 512);
  for (int i = tid; i < 64 * 16; i += 128) {  // 64 rows x 16 chunks of 8 bf16
    const int r = i / 16, c16 = i % 16, cb = c16 / 8, cc = c16 % 8;
    *reinterpret_cast<uint4*>(sK + cb * 8192 + sw128_off(r, cc)) = *reinterpret_cast<const uint4*>(K + r * 128 + c16 * 8);
    *reinterpret_cast<uint4*>(sV + cb * 8192 + sw128_off(r, cc)) = *reinterpret_cast<const uint4*>(V + r * 128 + c16 * 8);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  // TMEM layout: S at cols [0,64), O at [64,192), Q at [256, 320), P at [320, 352)
  const uint32_t trow = tb + ((uint32_t)(warp * 32) << 16);
  {
    uint32_t v[16];
    for (int c0 = 0; c0 < 64; c0 += 16) {  // Q: 64 packed columns
      for (int e = 0; e < 16; ++e) {
        __nv_bfloat162 h = __halves2bfloat162(Q[tid * 128 + 2 * (c0 + e)], Q[tid * 128 + 2 * (c0 + e) + 1]);
        v[e] = *reinterpret_cast<uint32_t*>(&h);
      }
      tmem_st16u(trow + 256 + c0, v);
    }
    for (int c0 = 0; c0 < 32; c0 += 16) {  // P: 32 packed columns
      for (int e = 0; e < 16; ++e) {
        __nv_bfloat162 h = __halves2bfloat162(P[tid * 64 + 2 * (c0 + e)], P[tid * 64 + 2 * (c0 + e) + 1]);
        v[e] = *reinterpret_cast<uint32_t*>(&h);
      }
      tmem_st16u(trow + 320 + c0, v);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if (elect_one()) {
      const uint64_t dK = umma_desc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dV = umma_desc_sw128(smem_u32(sV), 8192, 1024);
      constexpr uint32_t id_qk = umma_idesc_bf16(128, 64, 0, 0);
      constexpr uint32_t id_pv = umma_idesc_bf16(128, 128, 0, 1);
      for (int kk = 0; kk < 8; ++kk) {
        const int cb = kk >> 2, ko = (kk & 3) * 32;
        umma_ts(tb + 0, tb + 256 + kk * 8, dK + ((cb * 8192 + ko) >> 4), id_qk, kk > 0);
      }
      for (int kk = 0; kk < 4; ++kk) umma_ts(tb + 64, tb + 320 + kk * 8, dV + ((kk * 2048) >> 4), id_pv, kk > 0);
      umma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float f[16];
  for (int c0 = 0; c0 < 64; c0 += 16) {
    tmem_ld16(trow + c0, f);
    tmem_wait_ld();
    for (int e = 0; e < 16; ++e) S_out[tid * 64 + c0 + e] = f[e];
  }
  for (int c0 = 0; c0 < 128; c0 += 16) {
    tmem_ld16(trow + 64 + c0, f);
    tmem_wait_ld();
    for (int e = 0; e < 16; ++e) O_out[tid * 128 + c0 + e] = f[e];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

int main() {
  std::vector<__nv_bfloat16> Q(128 * 128), K(64 * 128), P(128 * 64), V(64 * 128);
  std::vector<float> q(Q.size()), k(K.size()), p(P.size()), v(V.size());
  srand(1);
  auto fill = [](std::vector<__nv_bfloat16>& X, std::vector<float>& x) {
    for (size_t i = 0; i < X.size(); ++i) { X[i] = __float2bfloat16((rand() / (float)RAND_MAX) * 2 - 1); x[i] = __bfloat162float(X[i]); }
  };
  fill(Q, q); fill(K, k); fill(P, p); fill(V, v);
  __nv_bfloat16 *dQ, *dK, *dP, *dV; float *dS, *dO;
  cudaMalloc(&dQ, Q.size() * 2); cudaMalloc(&dK, K.size() * 2); cudaMalloc(&dP, P.size() * 2); cudaMalloc(&dV, V.size() * 2);
  cudaMalloc(&dS, 128 * 64 * 4); cudaMalloc(&dO, 128 * 128 * 4);
  cudaMemcpy(dQ, Q.data(), Q.size() * 2, cudaMemcpyHostToDevice); cudaMemcpy(dK, K.data(), K.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice); cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  k_test<<<1, 128, 40 * 1024>>>(dQ, dK, dP, dV, dS, dO);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> S(128 * 64), O(128 * 128);
  cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost); cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 64; ++j) {
      double r = 0; for (int c = 0; c < 128; ++c) r += q[i * 128 + c] * k[j * 128 + c];
      es = fmax(es, fabs(r - S[i * 64 + j]));
    }
  for (int i = 0; i < 128; ++i)
    for (int n = 0; n < 128; ++n) {
      double r = 0; for (int c = 0; c < 64; ++c) r += p[i * 64 + c] * v[c * 128 + n];
      eo = fmax(eo, fabs(r - O[i * 128 + n]));
    }
  printf("%s: TS QK max err %.3e (S[0]=%f), TS PV max err %.3e  -> %s\n", cudaGetErrorString(e), es, S[0], eo,
         (es < 1e-2 && eo < 1e-2) ? "PASS" : "FAIL");
}
