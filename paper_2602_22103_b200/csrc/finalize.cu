// finalize.cu -- S3: unique-page bitmap + popcount, per-kernel footprint / WS, and
// the bitmap OR used by the multi-GPU merge (DESIGN.md sections 3-5).
//
//  * bitmap: one warp per 64 pages: two coalesced 8-byte loads per lane, two
//    __ballot_sync(count != 0) make the 64-bit word (low half = first 32 pages), lane
//    0 stores it and adds __popcll; block reduce, one atomicAdd per block into
//    totals[UNIQUE_PAGES] (P:795 working set by pages, north star part 3; R14).
//  * footprint: one warp per kernel row: sum of registered sizes over ids with a
//    non-zero count; atomicMax of the rows into totals[WS_OBJ]
//    (P:795); the row's page-bitmap popcount (per-kernel unique pages). The same kernel
//    gives tensor footprints and totals[WS_TENSOR] from the tensor rows (NEXT f3).
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace pasta {
namespace {

using namespace dev;

constexpr int kBlock = 256;

__global__ void __launch_bounds__(kBlock) bitmap_kernel(const uint64_t* __restrict__ pc, uint64_t P,
                                                        uint64_t* __restrict__ bitmap,
                                                        uint64_t* __restrict__ unique_out) {
  __shared__ uint64_t part[kBlock / 32];
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t W = (P + 63) / 64;
  const uint64_t gw = (uint64_t)blockIdx.x * (kBlock / 32) + wib;
  const uint64_t nw = (uint64_t)gridDim.x * (kBlock / 32);
  uint64_t local = 0;
  constexpr int kU = 4;  // bitmap words per warp iteration (8 loads per lane in flight)
  for (uint64_t w0 = gw * kU; w0 < W; w0 += nw * kU) {
    uint64_t c[2 * kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t p0 = 64 * (w0 + u) + lane, p1 = p0 + 32;
      c[2 * u] = p0 < P ? __ldg(pc + p0) : 0;
      c[2 * u + 1] = p1 < P ? __ldg(pc + p1) : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const unsigned b0 = __ballot_sync(kFull, c[2 * u] != 0);
      const unsigned b1 = __ballot_sync(kFull, c[2 * u + 1] != 0);
      const uint64_t word = (uint64_t)b0 | ((uint64_t)b1 << 32);
      if (lane == u && w0 + u < W) {
        if (bitmap) bitmap[w0 + u] = word;
        local += __popcll(word);
      }
    }
  }
  local = warp_sum_u64(local);
  if (lane == 0) part[wib] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (int i = 0; i < kBlock / 32; ++i) s += part[i];
    if (s) red_add_u64(unique_out, s);
  }
}

// One CTA per kernel row (grid-stride over rows): every thread strides over the row with
// 4 loads in flight, block reduction of the footprint and of the row's page-bitmap
// popcount. (A warp per row starved at wide rows: 3,000 x 65,536 ids = 1.6 GB streamed
// by 3,000 warps at ~2 TB/s.)
__global__ void __launch_bounds__(kBlock) footprint_kernel(const uint64_t* __restrict__ kac, uint32_t K,
                                                           uint64_t max_ids, const uint64_t* __restrict__ id_size,
                                                           const uint64_t* __restrict__ kpb, uint32_t words,
                                                           uint64_t* __restrict__ fp_out, uint32_t fp_stride,
                                                           uint64_t* __restrict__ up_out, uint32_t up_stride,
                                                           uint64_t* __restrict__ ws_out) {
  __shared__ uint64_t part[2][kBlock / 32];
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint64_t wmax = 0;
  for (uint64_t k = blockIdx.x; k < K; k += gridDim.x) {
    const uint64_t* row = kac + k * max_ids;
    uint64_t f = 0;
    constexpr int kFU = 4;
    for (uint64_t i0 = threadIdx.x; i0 < max_ids; i0 += (uint64_t)kBlock * kFU) {
      uint64_t v[kFU];
#pragma unroll
      for (int u = 0; u < kFU; ++u) v[u] = i0 + (uint64_t)kBlock * u < max_ids ? __ldg(row + i0 + kBlock * u) : 0;
#pragma unroll
      for (int u = 0; u < kFU; ++u)
        if (v[u] != 0) f += __ldg(id_size + i0 + kBlock * u);
    }
    uint64_t up = 0;
    if (kpb) {
      const uint64_t* brow = kpb + k * words;
      for (uint64_t w = threadIdx.x; w < words; w += kBlock) up += __popcll(__ldg(brow + w));
    }
    f = warp_sum_u64(f);
    up = warp_sum_u64(up);
    if (lane == 0) {
      part[0][wib] = f;
      part[1][wib] = up;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t F = 0, U = 0;
      for (int i = 0; i < kBlock / 32; ++i) {
        F += part[0][i];
        U += part[1][i];
      }
      fp_out[k * fp_stride] = F;
      if (up_out) up_out[k * up_stride] = U;
      wmax = F > wmax ? F : wmax;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && wmax) atomic_max_u64(ws_out, wmax);
}

__global__ void __launch_bounds__(kBlock) bitmap_or_kernel(const uint64_t* gathered, uint32_t g,
                                                           uint64_t words, uint64_t* out, uint64_t* popcount) {
  __shared__ uint64_t part[kBlock / 32];
  const uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * kBlock;
  uint64_t local = 0;
  for (uint64_t w = tid; w < words; w += nt) {
    uint64_t x = 0;
    for (uint32_t r = 0; r < g; ++r) x |= gathered[(uint64_t)r * words + w];
    out[w] = x;
    local += __popcll(x);
  }
  if (!popcount) return;
  local = warp_sum_u64(local);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (int i = 0; i < kBlock / 32; ++i) s += part[i];
    if (s) red_add_u64(popcount, s);
  }
}

// MAX_MEM_REFERENCED_KERNEL (R24): one block, argmax of attributed +
// unattributed records per kernel row, ties to the lowest row.
// out[0] = row0 + argmax, out[1] = that row's records (the (index, records) pair that
// kernel-aligned shards merge with pasta_peer_reduce(PASTA_PEER_ARGMAX)).
__global__ void __launch_bounds__(1024) max_kernel_kernel(const uint64_t* __restrict__ kstats, uint32_t K,
                                                          uint64_t row0, uint64_t* __restrict__ out) {
  __shared__ uint64_t sv[32];
  __shared__ uint32_t si[32];
  uint64_t bv = 0;
  uint32_t bi = 0xFFFFFFFFu;
  // 8 rows per thread in flight at once (one block: the loads' latency is the cost)
  for (uint32_t k0 = threadIdx.x; k0 < K; k0 += 8u * blockDim.x) {
    uint64_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t k = k0 + (uint32_t)u * blockDim.x;
      v[u] = k < K ? __ldg(kstats + 4ull * k) + __ldg(kstats + 4ull * k + 1) : 0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t k = k0 + (uint32_t)u * blockDim.x;
      if (k < K && (bi == 0xFFFFFFFFu || v[u] > bv)) {  // rows visited in increasing order: the first max stays
        bv = v[u];
        bi = k;
      }
    }
  }
  // warp then block reduction of (value desc, index asc)
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t v = __shfl_xor_sync(kFull, bv, o);
    const uint32_t i = __shfl_xor_sync(kFull, bi, o);
    if (i != 0xFFFFFFFFu && (bi == 0xFFFFFFFFu || v > bv || (v == bv && i < bi))) {
      bv = v;
      bi = i;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (si[w] != 0xFFFFFFFFu && (si[0] == 0xFFFFFFFFu || sv[w] > sv[0] || (sv[w] == sv[0] && si[w] < si[0]))) {
        sv[0] = sv[w];
        si[0] = si[w];
      }
    out[0] = row0 + (si[0] == 0xFFFFFFFFu ? 0 : si[0]);
    out[1] = si[0] == 0xFFFFFFFFu ? 0 : sv[0];
  }
}

int grid_for(uint64_t items, int per_block, int max_grid) {
  uint64_t b = (items + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > (uint64_t)max_grid) b = max_grid;
  return (int)b;
}

}  // namespace

cudaError_t launch_finalize_bitmap(const uint64_t* page_counts, uint64_t P, uint64_t* bitmap, uint64_t* unique_out,
                                   int grid, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(unique_out, 0, sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  const uint64_t W = (P + 63) / 64;
  bitmap_kernel<<<grid_for(W, kBlock / 32, grid), kBlock, 0, st>>>(page_counts, P, bitmap, unique_out);
  return cudaGetLastError();
}

cudaError_t launch_footprint(const uint64_t* kac, uint32_t n_kernels, uint64_t max_ids, const uint64_t* id_size,
                             const uint64_t* kpb, uint32_t words, uint64_t* fp_out, uint32_t fp_stride,
                             uint64_t* up_out, uint32_t up_stride, uint64_t* ws_out, int grid, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(ws_out, 0, sizeof(uint64_t), st);
  if (e != cudaSuccess) return e;
  footprint_kernel<<<grid_for(n_kernels, 1, grid), kBlock, 0, st>>>(
      kac, n_kernels, max_ids, id_size, kpb, words, fp_out, fp_stride, up_out, up_stride, ws_out);
  return cudaGetLastError();
}

cudaError_t launch_max_kernel(const uint64_t* kstats, uint32_t n_kernels, uint64_t row0, uint64_t* out,
                              cudaStream_t st) {
  max_kernel_kernel<<<1, 1024, 0, st>>>(kstats, n_kernels, row0, out);
  return cudaGetLastError();
}

cudaError_t launch_bitmap_or(const uint64_t* gathered, uint32_t g, uint64_t words, uint64_t* out,
                             uint64_t* popcount, int grid, cudaStream_t st) {
  if (popcount) {
    cudaError_t e = cudaMemsetAsync(popcount, 0, sizeof(uint64_t), st);
    if (e != cudaSuccess) return e;
  }
  bitmap_or_kernel<<<grid_for(words, kBlock, grid), kBlock, 0, st>>>(gathered, g, words, out, popcount);
  return cudaGetLastError();
}

}  // namespace pasta
