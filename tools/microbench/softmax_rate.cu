// Debug micro-benchmark: cycles per forward softmax step (64 columns, thread == row) in isolation,
// 4 warps per SM, data from TMEM like the kernel. Variants: plain MUFU, half the columns by polynomial.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;

__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
// 2^x for x <= 0 on the FMA pipe: Cody-Waite split, degree-3 minimax on [0,1) (rel err < 9e-5)
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float j = floorf(x);
  const float f = x - j;
  const float p = fmaf(fmaf(fmaf(0.0790199f, f, 0.2243755f), f, 0.6962318f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (static_cast<int>(j) << 23));
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(int steps, unsigned long long* out, float* sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tb, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t trow = tb + ((uint32_t)(warp * 32) << 16);
  {
    float init[16];
    for (int e = 0; e < 16; ++e) init[e] = 0.01f * (threadIdx.x + e);
    for (int c = 0; c < 64; c += 16) tmem_st16(trow + c, init);
    tmem_wait_st();
  }
  float m_run = -INFINITY, l_run = 0.f;
  const float sl2 = 0.127f;
  unsigned long long t0 = clock64();
  for (int u = 0; u < steps; ++u) {
    float sv[64];
#pragma unroll
    for (int c = 0; c < 64; c += 16) tmem_ld16(trow + c, sv + c);
    tmem_wait_ld();
    float mp[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int c = 0; c < 64; ++c) mp[c & 3] = fmaxf(mp[c & 3], sv[c]);
    float mx = fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])) * sl2;
    if (mx > m_run + 8.f) { l_run *= ex2(m_run - mx); m_run = mx; }
    float sp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      const float x = fmaf(sv[c], sl2, -m_run);
      sv[c] = (MODE == 1 && (c & 3) == 3) ? ex2_poly(x) : ex2(x);
      sp[c & 7] += sv[c];
    }
    l_run += ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
    float w[16];
#pragma unroll
    for (int c0 = 0; c0 < 32; c0 += 16) {
#pragma unroll
      for (int e = 0; e < 16; ++e) w[e] = __uint_as_float(pack_bf16(sv[2 * (c0 + e)], sv[2 * (c0 + e) + 1]));
      tmem_st16(trow + 128 + c0, w);
    }
    tmem_wait_st();
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 4 + warp] = (t1 - t0) / steps;
  sink[blockIdx.x * 128 + threadIdx.x] = l_run;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 256);
}

int main() {
  unsigned long long* out; cudaMalloc(&out, 148 * 4 * 8);
  float* sink; cudaMalloc(&sink, 148 * 128 * 4);
  auto run = [&](auto kern, const char* name) {
    kern<<<148, 128>>>(2000, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(148 * 4); cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
    double a = 0; for (auto v : h) a += v; a /= h.size();
    printf("%-34s %.0f cycles per 64-column softmax step (%s)\n", name, a, cudaGetErrorString(e));
  };
  run(k<0>, "all MUFU ex2");
  run(k<1>, "1/4 of columns polynomial");
}
