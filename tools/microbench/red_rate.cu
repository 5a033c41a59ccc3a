// Debug micro-benchmark: fp32 add-reduction throughput into a large global buffer (like dQacc):
//   mode 0: red.global.add.v4.f32 from registers (128 threads/CTA, each thread a 512 B row)
//   mode 1: cp.reduce.async.bulk (non-tensor) of whole 32-row x 512 B = 16 KB blocks from smem
//   mode 2: plain st.global.v4 (baseline write bandwidth)
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <cuda.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void bulk_reduce_add_f32(void* gdst, const void* src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(128, 1) k(float* buf, size_t nrows, int iters, int mode, unsigned long long* cyc, const __grid_constant__ CUtensorMap map, int boxc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* sm = reinterpret_cast<float*>(smem_raw);
  for (int i = threadIdx.x; i < 4 * 32 * 128; i += 128) sm[i] = 1.0f;
  fence_proxy_async_smem();
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // pseudo-random 32-row block
    size_t blk = (static_cast<size_t>(blockIdx.x) * 7919u + it * 104729u) % (nrows / 32);
    float* base = buf + blk * 32 * 128;
    if (mode == 0) {
      // 4 rows per warp-iteration... each thread owns row (tid % 32) of the block, 32 v4 reds over the row
      const int r = threadIdx.x & 31, q = threadIdx.x >> 5;
      float* row = base + r * 128 + q * 32;
      for (int e = 0; e < 32; e += 4)
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(row + e), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                     : "memory");
    } else if (mode == 1) {
      if (threadIdx.x == 0) {
        bulk_reduce_add_f32(base, sm + (it & 3) * 32 * 128, 32 * 128 * 4);
        bulk_commit_group();
        bulk_wait_group_read<3>();
      }
    } else if (mode >= 3) {
      // tensor reduce: boxes of {boxc cols, 32 rows} covering the 32 x 128 block, issued by lane 0 of each warp
      const int w = threadIdx.x >> 5, nb = 128 / boxc;
      if ((threadIdx.x & 31) == 0) {
        for (int b = w; b < nb; b += 4) {
          uint8_t* src = reinterpret_cast<uint8_t*>(sm) + ((it & 1) * 4 + (b & 3)) * 32 * boxc * 4 % 65536;
          if (mode == 6) {
            tma_reduce_add_2d(&map, src, b * boxc, static_cast<int>(blk * 32));
            tma_reduce_add_2d(&map, src + 2048, b * boxc, static_cast<int>(blk * 32 + 16));
          } else {
            tma_reduce_add_2d(&map, src, b * boxc, static_cast<int>(blk * 32));
          }
        }
        bulk_commit_group();
        bulk_wait_group_read<1>();
      }
    } else {
      const int r = threadIdx.x & 31, q = threadIdx.x >> 5;
      float4* row = reinterpret_cast<float4*>(base + r * 128 + q * 32);
      for (int e = 0; e < 8; ++e) row[e] = make_float4(1.f, 1.f, 1.f, 1.f);
    }
  }
  if ((mode == 1 || mode >= 3) && (threadIdx.x & 31) == 0) bulk_wait_group<0>();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const size_t nrows = 12ull * 16384;  // ~ BH * Lq rows of 128 fp32 = 100 MB
  float* buf; cudaMalloc(&buf, nrows * 128 * 4);
  unsigned long long* cyc; cudaMalloc(&cyc, 148 * 2 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  EncodeTiledFn enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  for (int mode : {0, 1, 2, 3, 4, 5, 6}) for (int ctas : {148, 296}) {
    CUtensorMap map; int boxc = mode == 3 ? 16 : (mode == 4 || mode == 6) ? 32 : 128; int boxr = mode == 6 ? 16 : 32;
    {
      cuuint64_t dims[2] = {128, nrows}; cuuint64_t str[1] = {512}; cuuint32_t box[2] = {(cuuint32_t)boxc, (cuuint32_t)boxr}; cuuint32_t es[2] = {1, 1};
      CUtensorMapSwizzle sw = mode == 3 ? CU_TENSOR_MAP_SWIZZLE_64B : (mode == 4 || mode == 6) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    }
    cudaMemset(buf, 0, nrows * 512);
    const int iters = 400;
    k<<<ctas, 128, 70 * 1024>>>(buf, nrows, 20, mode, cyc, map, boxc);
    cudaEventRecord(a);
    k<<<ctas, 128, 70 * 1024>>>(buf, nrows, iters, mode, cyc, map, boxc);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)ctas * iters * 16384;
    printf("mode %d (%s) ctas %d: %.3f ms, %.0f GB/s of fp32 reduce traffic (%s)\n", mode,
           mode == 0 ? "red.global.v4" : mode == 1 ? "bulk reduce 16KB" : mode == 2 ? "st.global.v4" : mode == 3 ? "tensor box16x32 sw64" : mode == 4 ? "tensor box32x32 sw128" : mode == 5 ? "tensor box128x32 nosw" : "tensor box32x16 sw128", ctas, ms, bytes / ms / 1e6,
           cudaGetErrorString(e));
  }
}
