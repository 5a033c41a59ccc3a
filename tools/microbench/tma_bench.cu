// Debug micro-benchmark: TMA throughput per SM vs box shape (4-stage ring, no compute).
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2509_01085_b200/csrc/ptx.cuh"
using namespace bsa;

struct P { CUtensorMap m; int boxes_per_stage; int box_bytes; int rows_per_box; int nsteps; int mode; const uint8_t* src; long long nrows; };

__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ P p, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[4], empty[4];
  int tid = threadIdx.x;
  if (tid == 0) { for (int s = 0; s < 4; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); } fence_mbar_init(); }
  __syncthreads();
  const int stage_bytes = p.boxes_per_stage * p.box_bytes;
  unsigned long long t0 = clock64();
  if (tid < 32) {
    unsigned seed = blockIdx.x * 7919u + 13u + tid * 101u;
    for (int u = 0; u < p.nsteps; ++u) {
      int s = u & 3;
      mbar_wait(&empty[s], ((u >> 2) & 1) ^ 1);
      if (tid == 0) mbar_expect_tx(&full[s], stage_bytes);
      __syncwarp();
      for (int b = 0; b < p.boxes_per_stage; ++b) {
        if (p.mode == 2 ? (b % 32) != tid : tid != 0) continue;
        seed = seed * 1664525u + 1013904223u;
        long long row = (long long)(seed % (unsigned)(p.nrows / p.rows_per_box)) * p.rows_per_box;
        uint8_t* dst = sm + s * stage_bytes + b * p.box_bytes;
        if (p.mode != 1) {
          tma_load_2d(dst, &p.m, &full[s], 0, (int)row);
        } else {
          const uint8_t* src = p.src + row * 256;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(smem_u32(dst)), "l"(src), "r"(p.box_bytes), "r"(smem_u32(&full[s])) : "memory");
        }
      }
    }
  }
  if (tid == 32) {
    for (int u = 0; u < p.nsteps; ++u) {
      int s = u & 3;
      mbar_wait(&full[s], (u >> 2) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  EncodeFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  long long nrows = 1 << 18;  // 256K rows x 256 B = 64 MB (L2 resident after first touch)
  uint8_t* buf; cudaMalloc(&buf, nrows * 256); cudaMemset(buf, 1, nrows * 256);
  unsigned long long* out; cudaMalloc(&out, 296 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int mode, box_rows, boxes; const char* name; };
  Cfg cfgs[] = {{2, 32, 8, "2D 4 KB x8, 8 issuing lanes"}, {2, 64, 4, "2D 8 KB x4, 4 issuing lanes"},{0, 32, 8, "2D box 64x32 (4 KB) x8"}, {0, 64, 4, "2D box 64x64 (8 KB) x4"}, {0, 128, 2, "2D box 64x128 (16 KB) x2"},
                {0, 256, 1, "2D box 64x256 (32 KB) x1"}, {1, 32, 4, "bulk 8 KB x4"}, {1, 64, 2, "bulk 16 KB x2"}};
  for (auto& c : cfgs) {
    P p; p.nsteps = 512; p.mode = c.mode; p.src = buf; p.nrows = nrows;
    p.rows_per_box = c.mode == 0 ? c.box_rows : c.box_rows;
    p.box_bytes = c.mode == 1 ? c.box_rows * 256 : c.box_rows * 128;
    p.boxes_per_stage = c.boxes;
    cuuint64_t dims[2] = {128, (cuuint64_t)nrows}, str[1] = {256};
    cuuint32_t box[2] = {64, (cuuint32_t)c.box_rows}, es[2] = {1, 1};
    enc(&p.m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int grid : {148, 296}) for (int rep = 0; rep < 2; ++rep) {
      int smem_b = grid == 148 ? 200 * 1024 : 100 * 1024;
      if (grid == 296 && p.boxes_per_stage * p.box_bytes * 4 + 2048 > smem_b) continue;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<grid, 64, smem_b>>>(p, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      std::vector<unsigned long long> h(grid); cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
      double cyc = 0; for (auto v : h) cyc += v; cyc /= grid;
      double bytes = (double)p.nsteps * p.boxes_per_stage * p.box_bytes;
      if (rep) printf("%-32s grid %d stage %6d B: %.1f B/clk/CTA, chip %.2f TB/s (%s)\n", c.name, grid, p.boxes_per_stage * p.box_bytes,
                      bytes / cyc, bytes * grid / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
