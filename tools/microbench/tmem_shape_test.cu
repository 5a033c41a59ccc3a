// Micro-test: element mapping of tcgen05.ld.16x256b (and the lane offset within a warp's quadrant).
// TMEM is filled with value = 1000 * lane + column via 32x32b stores; each thread of warp 0 then loads
// with .16x256b.x2 at lane offsets 0 and 16 and prints what it got.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;

__global__ void k(float* out) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&tb, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t trow = tb + ((uint32_t)(warp * 32) << 16);
  float v[16];
  for (int e = 0; e < 16; ++e) v[e] = 1000.f * (warp * 32 + lane) + e;
  tmem_st16(trow, v);
  for (int e = 0; e < 16; ++e) v[e] = 1000.f * (warp * 32 + lane) + 16 + e;
  tmem_st16(trow + 16, v);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) {  // tcgen05.st.16x128b.x2: thread t writes value 100*t + reg index
    uint32_t w[4];
    for (int e = 0; e < 4; ++e) w[e] = __float_as_uint(100.f * lane + e);
    asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1,%2,%3,%4};" ::"r"(tb + (64u << 16) + 24u),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
    tmem_wait_st();
    float rv[8];  // read back lanes 64..95, cols 24..31 with 32x32b
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tb + (64u << 16) + 24u));
    tmem_wait_ld();
    for (int e = 0; e < 8; ++e) rv[e] = __uint_as_float(r[e]);
    for (int e = 0; e < 8; ++e) out[512 + lane * 8 + e] = rv[e];
  }
  if (warp == 1) {
    for (int off = 0; off < 2; ++off) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tb + ((uint32_t)(32 + 16 * off) << 16)));
      tmem_wait_ld();
      for (int e = 0; e < 8; ++e) out[(off * 32 + lane) * 8 + e] = __uint_as_float(r[e]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 32);
}

int main() {
  float* d; cudaMalloc(&d, 4 * 32 * 8 * 4);
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  float h[4 * 32 * 8]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  for (int off = 0; off < 2; ++off)
    for (int t = 0; t < 32; t += 1) {
      printf("off %d thread %2d:", off, t);
      for (int e = 0; e < 8; ++e) {
        float x = h[(off * 32 + t) * 8 + e];
        printf(" (L%d,c%d)", (int)(x / 1000), (int)x % 1000);
      }
      printf("\n");
    }
  printf("16x128b.x2 store: TMEM lane (64+i), cols 24..31 hold (thread*100 + reg):\n");
  for (int i = 0; i < 16; ++i) {
    printf(" lane %2d:", 64 + i);
    for (int e = 0; e < 8; ++e) { float x = h[512 + i * 8 + e]; printf(" t%d.r%d", (int)(x / 100), (int)x % 100); }
    printf("\n");
  }
}
