// Debug micro-benchmark: cp.async.bulk throughput vs request size and CTAs per SM.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;
__global__ void k(const uint8_t* src, long long nbytes, int req, int stages, int nsteps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[8], empty[8];
  int tid = threadIdx.x;
  if (tid == 0) { for (int s = 0; s < 8; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); } fence_mbar_init(); }
  __syncthreads();
  unsigned long long t0 = clock64();
  if (tid == 0) {
    unsigned seed = blockIdx.x * 7919u + 13u;
    for (int u = 0; u < nsteps; ++u) {
      int s = u % stages;
      mbar_wait(&empty[s], ((u / stages) & 1) ^ 1);
      mbar_expect_tx(&full[s], req);
      seed = seed * 1664525u + 1013904223u;
      long long off = (long long)(seed % (unsigned)(nbytes / req)) * req;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(sm + s * req)), "l"(src + off), "r"(req), "r"(smem_u32(&full[s])) : "memory");
    }
  } else if (tid == 32) {
    for (int u = 0; u < nsteps; ++u) { int s = u % stages; mbar_wait(&full[s], (u / stages) & 1); mbar_arrive(&empty[s]); }
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = clock64() - t0;
}
int main() {
  long long nbytes = 64ll << 20;
  uint8_t* buf; cudaMalloc(&buf, nbytes); cudaMemset(buf, 1, nbytes);
  unsigned long long* out; cudaMalloc(&out, 4 * 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C { int req, stages, ctas; };
  C cs[] = {{16384, 4, 1}, {16384, 8, 1}, {32768, 4, 1}, {32768, 6, 1}, {65536, 3, 1}, {16384, 4, 2}, {32768, 3, 2}, {16384, 2, 4}};
  for (auto c : cs) for (int rep = 0; rep < 2; ++rep) {
    int grid = 148 * c.ctas, smem = c.req * c.stages + 1024, nsteps = 256;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<<<grid, 64, smem>>>(buf, nbytes, c.req, c.stages, nsteps, out); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> h(grid); cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
    double cyc = 0; for (auto v : h) cyc += v; cyc /= grid;
    double bytes = (double)nsteps * c.req;
    if (rep) printf("bulk req %6d stages %d ctas/SM %d: %.1f B/clk/CTA  chip %.2f TB/s (%s)\n", c.req, c.stages, c.ctas,
                    bytes / cyc, bytes * grid / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
}
