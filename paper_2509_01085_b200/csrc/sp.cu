// sp.cu — layout changes around the Ulysses all-to-all (SURVEY.md §8(e) mode 2).
//
// A sequence-parallel DiT hands each of P ranks a contiguous chunk of Ls = L/P raster tokens of every
// head, [B][Ls][Hh][d]. BSA's selection needs all N pooled blocks of a head, so the
// sequence is regathered per head group: rank p owns heads [p Hp, (p+1) Hp), Hp = Hh/P, over the whole
// sequence. One all-to-all (NCCL, outside this library) moves equal-sized contiguous chunks; these
// kernels only reorder rows of d channels into and out of its send/receive buffers:
//
//   SEQ_TO_SEND    [B][Ls][Hh][d]        -> [P][B][Hp][Ls][d]   chunk p = head group p (fwd: Q, K, V; bwd: dO)
//   RECV_TO_HEADS  [P][B][Hp][Ls][d]     -> [B][Hp][P Ls][d]    chunk s = sequence chunk s (BSA layout)
//   HEADS_TO_SEND  [B][Hp][P Ls][d]      -> [P][B][Hp][Ls][d]   chunk s = sequence chunk s (fwd: O; bwd: dQ, dK, dV)
//   RECV_TO_SEQ    [P][B][Hp][Ls][d]     -> [B][Ls][Hh][d]      chunk p = head group p (back to the model)
//   SEQ_TO_SEND_T  [B][Ls][Hh][d]        -> [P][B][Ls][Hp][d]   token-major chunks (B = 1: what arrives is the
//                                                                whole sequence of Hp heads as [L][Hp][d], a
//                                                                strided [1, Hp, L, d] view BSA reads in place)
//   RECV_T_TO_SEQ  [P][B][Ls][Hp][d]     -> [B][Ls][Hh][d]      back to the model from token-major chunks
//
// Pure data movement, HBM-bound: one 16-byte vector per thread, destination-ordered so the writes are
// fully coalesced and every source row (2 d bytes, >= 128 B) is read as whole sectors.
#include "kernels.h"

namespace bsa {

template <int MODE>
__global__ void __launch_bounds__(256) k_sp_relayout(int B, int Ls, int Hh, int P, int vpr, const uint4* __restrict__ src,
                                                     uint4* __restrict__ dst, size_t total) {
  const size_t v = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= total) return;
  const size_t row = v / vpr;
  const int c = static_cast<int>(v % vpr);
  const int Hp = Hh / P;
  size_t srow;
  if (MODE == 0 || MODE == 2) {
    // dst [P][B][Hp][Ls]
    const int l = static_cast<int>(row % Ls);
    size_t t = row / Ls;
    const int h = static_cast<int>(t % Hp);
    t /= Hp;
    const int b = static_cast<int>(t % B);
    const int p = static_cast<int>(t / B);
    if (MODE == 0) srow = (static_cast<size_t>(b) * Ls + l) * Hh + static_cast<size_t>(p) * Hp + h;  // [B][Ls][Hh]
    else srow = (static_cast<size_t>(b) * Hp + h) * (static_cast<size_t>(P) * Ls) + static_cast<size_t>(p) * Ls + l;  // [B][Hp][P Ls]
  } else if (MODE == 1) {
    // dst [B][Hp][P Ls]  <-  src [P][B][Hp][Ls]
    const size_t L = static_cast<size_t>(P) * Ls;
    const size_t n = row % L;
    const size_t t = row / L;
    const int h = static_cast<int>(t % Hp), b = static_cast<int>(t / Hp);
    const int s = static_cast<int>(n / Ls), l = static_cast<int>(n % Ls);
    srow = ((static_cast<size_t>(s) * B + b) * Hp + h) * Ls + l;
  } else if (MODE == 3) {
    // dst [B][Ls][Hh]  <-  src [P][B][Hp][Ls]
    const int hh = static_cast<int>(row % Hh);
    const size_t t = row / Hh;
    const int l = static_cast<int>(t % Ls), b = static_cast<int>(t / Ls);
    const int p = hh / Hp, h = hh % Hp;
    srow = ((static_cast<size_t>(p) * B + b) * Hp + h) * Ls + l;
  } else if (MODE == 4) {
    // dst [P][B][Ls][Hp]  <-  src [B][Ls][Hh]
    const int h = static_cast<int>(row % Hp);
    size_t t = row / Hp;
    const int l = static_cast<int>(t % Ls);
    t /= Ls;
    const int b = static_cast<int>(t % B), p = static_cast<int>(t / B);
    srow = (static_cast<size_t>(b) * Ls + l) * Hh + static_cast<size_t>(p) * Hp + h;
  } else {
    // dst [B][Ls][Hh]  <-  src [P][B][Ls][Hp]
    const int hh = static_cast<int>(row % Hh);
    const size_t t = row / Hh;
    const int l = static_cast<int>(t % Ls), b = static_cast<int>(t / Ls);
    const int p = hh / Hp, h = hh % Hp;
    srow = ((static_cast<size_t>(p) * B + b) * Ls + l) * Hp + h;
  }
  dst[row * vpr + c] = src[srow * vpr + c];
}

// Head-group token-major exchange (B = 1 pipelining, ulysses.py head_groups): each rank's chunk carries only
// heads [p Hp + hoff, p Hp + hoff + Hs) of head group p, so a sub-group can be exchanged and attended while the
// next one is in flight.
//   GROUP_SEND (0)  dst [P][Ls][Hs][d]  <-  src [Ls][Hh][d] heads p Hp + hoff + h
//   GROUP_RECV (1)  dst [Ls][Hh][d] heads p Hp + hoff + h  <-  src [P][Ls][Hs][d]   (other heads untouched)
template <int MODE>
__global__ void __launch_bounds__(256) k_sp_group(int Ls, int Hh, int P, int hoff, int Hs, int vpr,
                                                  const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                  size_t total) {
  const size_t v = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= total) return;
  const size_t row = v / vpr;  // enumerates [P][Ls][Hs]
  const int c = static_cast<int>(v % vpr);
  const int h = static_cast<int>(row % Hs);
  const size_t t = row / Hs;
  const int l = static_cast<int>(t % Ls), p = static_cast<int>(t / Ls);
  const size_t mrow = static_cast<size_t>(l) * Hh + static_cast<size_t>(p) * (Hh / P) + hoff + h;  // [Ls][Hh]
  if (MODE == 0) dst[row * vpr + c] = src[mrow * vpr + c];
  else dst[mrow * vpr + c] = src[row * vpr + c];
}

cudaError_t launch_sp_group(int mode, int Ls, int Hh, int d, int P, int hoff, int Hs, const void* src, void* dst,
                            cudaStream_t st) {
  const int vpr = d / 8;
  const size_t total = static_cast<size_t>(P) * Ls * Hs * vpr;
  if (total == 0) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>((total + 255) / 256);
  const uint4* s = static_cast<const uint4*>(src);
  uint4* o = static_cast<uint4*>(dst);
  if (mode == 0) k_sp_group<0><<<blocks, 256, 0, st>>>(Ls, Hh, P, hoff, Hs, vpr, s, o, total);
  else k_sp_group<1><<<blocks, 256, 0, st>>>(Ls, Hh, P, hoff, Hs, vpr, s, o, total);
  return cudaGetLastError();
}

cudaError_t launch_sp_relayout(int mode, int B, int Ls, int Hh, int d, int P, const void* src, void* dst,
                               cudaStream_t st) {
  const int vpr = d / 8;  // 16-byte vectors per row of d bf16
  const size_t total = static_cast<size_t>(B) * Ls * P * (Hh / P) * vpr;
  if (total == 0) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>((total + 255) / 256);
  const uint4* s = static_cast<const uint4*>(src);
  uint4* o = static_cast<uint4*>(dst);
  switch (mode) {
    case 0: k_sp_relayout<0><<<blocks, 256, 0, st>>>(B, Ls, Hh, P, vpr, s, o, total); break;
    case 1: k_sp_relayout<1><<<blocks, 256, 0, st>>>(B, Ls, Hh, P, vpr, s, o, total); break;
    case 2: k_sp_relayout<2><<<blocks, 256, 0, st>>>(B, Ls, Hh, P, vpr, s, o, total); break;
    case 3: k_sp_relayout<3><<<blocks, 256, 0, st>>>(B, Ls, Hh, P, vpr, s, o, total); break;
    case 4: k_sp_relayout<4><<<blocks, 256, 0, st>>>(B, Ls, Hh, P, vpr, s, o, total); break;
    default: k_sp_relayout<5><<<blocks, 256, 0, st>>>(B, Ls, Hh, P, vpr, s, o, total); break;
  }
  return cudaGetLastError();
}

}  // namespace bsa
