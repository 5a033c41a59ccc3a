// Debug micro-benchmark: cp.async (LDGSTS) throughput per SM from a 128-thread producer warpgroup,
// 32 KB stages, depth-3 pipelining, scattered 4 KB (32 x 128 B) tiles like the BSA backward chunks.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;

__global__ void __launch_bounds__(160, 1) k(const uint8_t* src, long long nrows, int nsteps, int rows_per_tile,
                                             unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[4], empty[4];
  const int tid = threadIdx.x;
  constexpr int STAGE = 32768;
  if (tid == 0) { for (int s = 0; s < 4; ++s) { mbar_init(&full[s], 128); mbar_init(&empty[s], 1); } fence_mbar_init(); }
  __syncthreads();
  unsigned long long t0 = clock64();
  const int tiles = STAGE / (rows_per_tile * 128);
  if (tid < 128) {
    unsigned seed = blockIdx.x * 7919u + 13u;
    for (int u = 0; u < nsteps + 2; ++u) {
      if (u < nsteps) {
        int s = u & 3;
        mbar_wait(&empty[s], ((u >> 2) & 1) ^ 1);
        // every thread copies STAGE/128 = 256 B = 16 x 16 B; tile rows of 128 B
        for (int k = 0; k < 16; ++k) {
          int chunk = tid + 128 * k;             // 16-byte chunk id within the stage (2048 chunks)
          int tile = chunk / (rows_per_tile * 8), within = chunk % (rows_per_tile * 8);
          int row = within / 8, c16 = within % 8;
          unsigned sd = seed + tile * 2654435761u + u * 40503u;
          long long grow = (long long)(sd % (unsigned)(nrows / rows_per_tile)) * rows_per_tile + row;
          const uint8_t* g = src + grow * 256 + c16 * 16;
          uint32_t dst = smem_u32(sm + s * STAGE + tile * rows_per_tile * 128 + sw128_off(row, c16));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(g) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      if (u >= 2) {  // stage u-2 complete
        if (u < nsteps) asm volatile("cp.async.wait_group 2;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        fence_proxy_async_smem();
        mbar_arrive(&full[(u - 2) & 3]);
      }
    }
  } else if (tid == 128) {
    for (int u = 0; u < nsteps; ++u) {
      int s = u & 3;
      mbar_wait(&full[s], (u >> 2) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  long long nrows = 1 << 18;
  uint8_t* buf; cudaMalloc(&buf, nrows * 256); cudaMemset(buf, 1, nrows * 256);
  unsigned long long* out; cudaMalloc(&out, 296 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int rpt : {32, 64}) for (int grid : {148, 296}) for (int rep = 0; rep < 2; ++rep) {
    int nsteps = 512;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<grid, 160, grid == 148 ? 140 * 1024 : 110 * 1024>>>(buf, nrows, nsteps, rpt, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> h(grid); cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
    double cyc = 0; for (auto v : h) cyc += v; cyc /= grid;
    double bytes = (double)nsteps * 32768;
    if (rep) printf("cp.async tiles of %d rows, grid %d: %.1f B/clk/CTA, chip %.2f TB/s (%s)\n", rpt, grid, bytes / cyc,
                    bytes * grid / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
