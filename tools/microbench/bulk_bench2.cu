// Debug: are bulk copies serialized per CTA or per issuing warp? 4 x 16 KB requests per stage,
// issued by 1 warp vs by 4 different warps.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;
__global__ void k(const uint8_t* src, long long nbytes, int nwarps_issue, int nsteps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[3], empty[3];
  const int req = 16384, per_stage = 4, stages = 3;
  int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  if (tid == 0) { for (int s = 0; s < 3; ++s) { mbar_init(&full[s], nwarps_issue); mbar_init(&empty[s], 1); } fence_mbar_init(); }
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp < nwarps_issue && lane == 0) {
    unsigned seed = blockIdx.x * 7919u + 13u + warp * 77u;
    for (int u = 0; u < nsteps; ++u) {
      int s = u % stages;
      mbar_wait(&empty[s], ((u / stages) & 1) ^ 1);
      int mine = per_stage / nwarps_issue;
      mbar_expect_tx(&full[s], req * mine);
      for (int r = 0; r < mine; ++r) {
        seed = seed * 1664525u + 1013904223u;
        long long off = (long long)(seed % (unsigned)(nbytes / req)) * req;
        int slot = warp * mine + r;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_u32(sm + (s * per_stage + slot) * req)), "l"(src + off), "r"(req), "r"(smem_u32(&full[s])) : "memory");
      }
    }
  } else if (warp == 4 && lane == 0) {
    for (int u = 0; u < nsteps; ++u) { int s = u % stages; mbar_wait(&full[s], (u / stages) & 1); mbar_arrive(&empty[s]); }
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = clock64() - t0;
}
int main() {
  long long nbytes = 64ll << 20;
  uint8_t* buf; cudaMalloc(&buf, nbytes); cudaMemset(buf, 1, nbytes);
  unsigned long long* out; cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nw : {1, 2, 4}) for (int rep = 0; rep < 2; ++rep) {
    int nsteps = 256;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k<<<148, 160, 3 * 4 * 16384 + 1024>>>(buf, nbytes, nw, nsteps, out); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> h(148); cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
    double cyc = 0; for (auto v : h) cyc += v; cyc /= 148;
    double bytes = (double)nsteps * 4 * 16384;
    if (rep) printf("4 x 16 KB per stage issued by %d warp(s): %.1f B/clk/CTA chip %.2f TB/s (%s)\n", nw, bytes / cyc,
                    bytes * 148 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
}
