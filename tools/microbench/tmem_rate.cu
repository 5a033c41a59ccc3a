// Debug micro-benchmark: TMEM read (tcgen05.ld 32x32b.x16) and write throughput per SM, with 4 or 8
// warps, optionally while one warp keeps the tensor pipe busy with SS MMAs (128x128x16) into other columns.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;

__global__ void __launch_bounds__(384, 1) k(int nwarps, int reps, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  __shared__ int s_done;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); s_done = 0; }
  if (warp == 8) tmem_alloc(&tb, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp < nwarps) {
    const uint32_t trow = tb + ((uint32_t)((warp % 4) * 32) << 16) + (warp / 4) * 64;
    float v[16], acc = 0.f;
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (mode & 1) {
#pragma unroll
        for (int c = 0; c < 64; c += 16) tmem_st16(trow + c, v);
        tmem_wait_st();
      } else {
#pragma unroll
        for (int c = 0; c < 64; c += 16) { tmem_ld16(trow + c, v); acc += v[c / 16]; }
        tmem_wait_ld();
      }
    }
    unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + warp] = t1 - t0;
    if (acc == 1234.5f) out[0] = 0;
  } else if (warp == 11 && (mode & 2)) {
    const bool leader = elect_one();
    const uint64_t dA = umma_desc_sw128(smem_u32(sm), 16, 1024), dB = umma_desc_sw128(smem_u32(sm + 32768), 16, 1024);
    constexpr uint32_t idesc = umma_idesc_bf16(128, 128, 0, 0);
    int it = 0;
    while (*((volatile int*)&s_done) == 0 && it < 100000) {
      if (leader) {
        for (int i = 0; i < 16; ++i) umma_ss(tb + 384, dA + (((i & 3) * 32) >> 4), dB + (((i & 3) * 32) >> 4), idesc, 1);
        umma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, it & 1);
      ++it;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) s_done = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc(tb, 512);
}

int main() {
  unsigned long long* out; cudaMalloc(&out, 148 * 8 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int reps = 2000;
  for (int mode : {0, 1, 2, 3}) for (int nw : {1, 4, 8}) {
    cudaMemset(out, 0, 148 * 64);
    k<<<148, 384, 80 * 1024>>>(nw, reps, mode, out);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(148 * 8); cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int b = 0; b < 148; ++b) for (int w = 0; w < nw; ++w) mx += h[b * 8 + w];
    mx /= 148 * nw;
    double bytes = (double)nw * 32 * 64 * 4 * reps;
    printf("%s%s warps=%d: %.0f cycles, %.1f B/clk/SM (%s)\n", (mode & 1) ? "tcgen05.st" : "tcgen05.ld",
           (mode & 2) ? " + MMA stream" : "", nw, mx, bytes / mx, cudaGetErrorString(e));
  }
}
