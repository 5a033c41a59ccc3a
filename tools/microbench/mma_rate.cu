// Debug micro-benchmark: steady-state tcgen05.mma issue rate (cycles per MMA) for the shapes the
// attention kernels use: SS (both operands in smem) vs TS (A in TMEM), M=64/128, N=64/128/256.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;


template <int M, int N, bool TS, bool BMN>
__global__ void __launch_bounds__(128, 1) k(int nmma, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += 128) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tb, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    const bool leader = elect_one();
    const uint64_t dA = umma_desc_sw128(smem_u32(sm), 16, 1024);
    // B: K-major [N rows][64 k] (8-row groups 1 KB apart) or MN-major [64 k rows][N] (64-col chunks 8 KB apart)
    const uint64_t dB = BMN ? umma_desc_sw128(smem_u32(sm + 32768), 8192, 1024) : umma_desc_sw128(smem_u32(sm + 32768), 16, 1024);
    constexpr uint32_t idesc = umma_idesc_bf16(M, N, 0, BMN ? 1 : 0);
    unsigned long long tot = 0;
    for (int it = 0; it < iters; ++it) {
      unsigned long long t0 = clock64();
      if (leader) {
        for (int i = 0; i < nmma; ++i) {
          const int kk = i & 3;
          const uint64_t b = dB + ((BMN ? kk * 2048 : kk * 32) >> 4);
          if (TS) umma_ts(tb + 256, tb + kk * 8, b, idesc, 1);
          else umma_ss(tb + 256, dA + ((kk * 32) >> 4), b, idesc, 1);
        }
        umma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, it & 1);
      if (it > 0) tot += clock64() - t0;
    }
    if (leader) out[blockIdx.x] = tot / (iters - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 512);
}

template <int M, int N, bool TS, bool BMN>
void run(const char* name) {
  unsigned long long* out; cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k<M, N, TS, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int nmma : {16, 256}) {
    k<M, N, TS, BMN><<<148, 128, 100 * 1024>>>(nmma, 6, out);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(148); cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (auto v : h) avg += v; avg /= 148;
    printf("%-22s M=%3d N=%3d nmma=%3d: %.0f cycles total, %.1f cycles/MMA (floor %d) %s\n", name, M, N, nmma, avg, avg / nmma,
           (M < 128 ? 128 : M) * N / 256, cudaGetErrorString(e));
  }
  cudaFree(out);
}

int main() {
  run<128, 64, false, false>("SS K-major B");
  run<128, 128, false, false>("SS K-major B");
  run<128, 256, false, false>("SS K-major B");
  run<128, 64, false, true>("SS MN-major B");
  run<128, 128, false, true>("SS MN-major B");
  run<64, 64, false, false>("SS K-major B");
  run<64, 128, false, false>("SS K-major B");
  run<128, 64, true, false>("TS K-major B");
  run<128, 128, true, false>("TS K-major B");
  run<128, 128, true, true>("TS MN-major B");
  run<128, 256, true, false>("TS K-major B");
}
