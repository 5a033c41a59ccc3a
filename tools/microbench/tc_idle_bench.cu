// Debug micro-benchmark: tcgen05.mma burst completion latency vs the idle gap before the burst.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;

__global__ void __launch_bounds__(256, 1) k(int gap_cycles, int iters, unsigned long long* out, int mode, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += 256) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tb, 256);
  __shared__ int s_done;
  __shared__ __align__(8) uint64_t lbar;
  if (threadIdx.x == 0) { s_done = 0; mbar_init(&lbar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    const bool leader = elect_one();
    const uint64_t dA = umma_desc_sw128(smem_u32(sm), 16, 1024), dB = umma_desc_sw128(smem_u32(sm + 32768), 16, 1024);
    constexpr uint32_t idesc = umma_idesc_bf16(128, 64, 0, 0);
    unsigned long long tot = 0, mx = 0, slow = 0;
    for (int it = 0; it < iters; ++it) {
      unsigned long long t0 = clock64();
      while (clock64() - t0 < (unsigned long long)gap_cycles) {}
      unsigned long long t1 = clock64();
      if (leader) {
        for (int kk = 0; kk < 8; ++kk) umma_ss(tb + 64, dA + ((kk * 32) >> 4), dB + ((kk * 32) >> 4), idesc, kk > 0);
        if (mode & 4) {
          constexpr uint32_t idesc_pv = umma_idesc_bf16(128, 128, 0, 1);
          const uint64_t dP = umma_desc_sw128(smem_u32(sm + 49152), 16, 1024);
          const uint64_t dV = umma_desc_sw128(smem_u32(sm + 32768), 8192, 1024);
          for (int kk = 0; kk < 4; ++kk) umma_ss(tb + 128, dP + ((kk * 32) >> 4), dV + ((kk * 2048) >> 4), idesc_pv, kk > 0);
        }
        umma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, it & 1);
      unsigned long long d = clock64() - t1;
      tot += d; if (d > mx) mx = d; if (d > 4000) ++slow;
    }
    if (leader) { out[blockIdx.x * 3] = tot / iters; out[blockIdx.x * 3 + 1] = mx; out[blockIdx.x * 3 + 2] = slow; }
    if (leader) atomicExch(&s_done, 1);
  } else if (warp >= 4 && (mode & 8)) {
    // softmax-like: write a 128x64 bf16 P tile rows with swizzle + fence.proxy.async, continuously
    const int row = (warp - 4) * 32 + (threadIdx.x & 31);
    int n = 0;
    while (*((volatile int*)&s_done) == 0) {
      for (int c16 = 0; c16 < 8; ++c16)
        *reinterpret_cast<uint4*>(sm + 49152 + sw128_off(row, c16)) = make_uint4(n, n, n, n);
      fence_proxy_async_smem();
      ++n;
    }
  } else if (warp >= 4 && (mode & 1)) {
    // TMEM readers on columns [0, 64) (S-like), lane quadrant warp%4
    const uint32_t trow = tb + ((uint32_t)((warp % 4) * 32) << 16);
    float v[16]; float acc = 0.f;
    while (*((volatile int*)&s_done) == 0) {
      for (int c = 0; c < 64; c += 16) { tmem_ld16(trow + c, v); }
      tmem_wait_ld();
      acc += v[0];
    }
    if (acc == 12345.f) out[0] = 1;
  } else if (warp == 2 && (mode & 2)) {
    // bulk-copy producer: 32 KB requests into smem [16K, 48K) continuously
    if (elect_one()) {
      int u = 0;
      while (*((volatile int*)&s_done) == 0) {
        mbar_expect_tx(&lbar, 32768);
        bulk_load(sm + 16384, gsrc + (size_t)((blockIdx.x * 7 + u) % 1024) * 32768, 32768, &lbar);
        mbar_wait(&lbar, u & 1);
        ++u;
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 256);
}

int main() {
  unsigned long long* out; cudaMalloc(&out, 148 * 3 * 8);
  uint8_t* gsrc; cudaMalloc(&gsrc, 1024ll * 32768); cudaMemset(gsrc, 0, 1024ll * 32768);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int mode : {4, 6, 12, 14}) for (int gap : {0, 1000}) {
    for (int rep = 0; rep < 2; ++rep) {
      k<<<148, 256, 80 * 1024>>>(gap, 300, out, mode, gsrc);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<unsigned long long> h(148 * 3); cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
      double avg = 0, mx = 0, slow = 0;
      for (int i = 0; i < 148; ++i) { avg += h[3 * i]; mx = mx > h[3 * i + 1] ? mx : h[3 * i + 1]; slow += h[3 * i + 2]; }
      if (rep) printf("mode %d (1=TMEM readers, 2=bulk loads) gap %5d cycles: burst(8 MMA 128x64x16)+commit latency avg %.0f max %.0f, slow(>4k) %.1f%% (%s)\n", mode, gap,
                      avg / 148, mx, 100.0 * slow / (148 * 300), cudaGetErrorString(e));
    }
  }
}
