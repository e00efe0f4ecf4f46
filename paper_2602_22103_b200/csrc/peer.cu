// peer.cu -- S5 merge over peer memory: one kernel reads every
// rank's partial counts directly (NVLink / NVSwitch loads through CUDA IPC mappings)
// and reduces them, fused with the bitmap and unique-page count of the reduced range.
//
// Every count output is a pointwise sum over any partition of the records (SPEC
// S:291-299), so the merged page count of page p is sum_r counts_r[p]; the bitmap
// bit p is merged_count[p] != 0 (R14); working sets merge by MAX (R11). The NCCL path
// (reduce_scatter, then all_gather of bitmaps, then pasta_bitmap_or) needs three
// passes and a gathered copy of every rank's bitmap; here rank r reads its shard of
// pages from all g ranks once and emits counts, bitmap words and popcount together.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace pasta {
namespace {

using namespace dev;

constexpr int kBlock = 256;

// Words of 64 pages: warp w of the grid takes word w (grid-stride); lane l sums pages
// 64w + l and 64w + 32 + l over the g sources (coalesced 256-byte rows per source, 2g
// loads in flight per lane), writes them, and the two ballots are the bitmap word.
__global__ void __launch_bounds__(kBlock) peer_sum_bitmap_kernel(PeerSrc src, uint32_t g, uint64_t lo,
                                                                 uint64_t words, uint64_t* __restrict__ out,
                                                                 uint64_t* __restrict__ out_bitmap,
                                                                 uint64_t* __restrict__ out_popcount) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp0 = ((uint64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * kBlock) >> 5;
  uint64_t pop = 0;
  for (uint64_t w = warp0; w < words; w += nwarps) {
    const uint64_t i0 = 64 * w + lane, i1 = i0 + 32;
    uint64_t v0[kMaxPeers], v1[kMaxPeers];
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r) {
      if (r < (int)g) {
        v0[r] = ld_stream_u64(src.p[r] + lo + i0);
        v1[r] = ld_stream_u64(src.p[r] + lo + i1);
      }
    }
    uint64_t c0 = 0, c1 = 0;
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r) {
      if (r < (int)g) {
        c0 += v0[r];
        c1 += v1[r];
      }
    }
    out[i0] = c0;
    out[i1] = c1;
    const uint64_t word = (uint64_t)__ballot_sync(kFull, c0 != 0) | ((uint64_t)__ballot_sync(kFull, c1 != 0) << 32);
    if (lane == 0) {
      if (out_bitmap) out_bitmap[w] = word;
      pop += (uint64_t)__popcll(word);
    }
  }
  if (out_popcount) {
    __shared__ unsigned long long part[kBlock / 32];
    if (lane == 0) part[threadIdx.x >> 5] = pop;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int i = 0; i < kBlock / 32; ++i) s += part[i];
      if (s) atomicAdd(reinterpret_cast<unsigned long long*>(out_popcount), s);
    }
  }
}

// Elementwise SUM or MAX of n values from g sources (small parts, WS slots).
template <bool kMax>
__global__ void __launch_bounds__(kBlock) peer_elementwise_kernel(PeerSrc src, uint32_t g, uint64_t lo, uint64_t n,
                                                                   uint64_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kBlock) {
    uint64_t acc = 0;
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r) {  // static indices: the sources stay in the parameter bank
      if (r < (int)g) {
        const uint64_t v = ld_stream_u64(src.p[r] + lo + i);
        acc = kMax ? (v > acc ? v : acc) : acc + v;
      }
    }
    out[i] = acc;
  }
}

// (index, value) pairs of g sources -> the pair with the largest value, ties to the
// smallest index (the merged MAX_MEM_REFERENCED_KERNEL of kernel-aligned shards, R24).
__global__ void peer_argmax_kernel(PeerSrc src, uint32_t g, uint64_t lo, uint64_t* __restrict__ out) {
  uint64_t bi = 0, bv = 0;
  bool any = false;
#pragma unroll
  for (int r = 0; r < kMaxPeers; ++r) {
    if (r < (int)g) {
      const uint64_t i = ld_stream_u64(src.p[r] + lo), v = ld_stream_u64(src.p[r] + lo + 1);
      if (!any || v > bv || (v == bv && i < bi)) {
        bi = i;
        bv = v;
        any = true;
      }
    }
  }
  out[0] = bi;
  out[1] = bv;
}

// Small part of g shards in one pass: SUM except the listed slots (MAX, ARGMAX pair, ZERO).
__global__ void __launch_bounds__(kBlock) peer_small_kernel(PeerSrc src, uint32_t g, uint64_t lo, uint64_t n,
                                                            PeerSlots sl, uint64_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kBlock) {
    uint32_t op = 0, half = 0;  // 0 SUM, 1 MAX, 2 ARGMAX (half: 0 index, 1 value), 3 ZERO
    for (uint32_t s = 0; s < sl.n; ++s) {
      if (sl.idx[s] == i) op = sl.op[s];
      if (sl.op[s] == 2u && (uint64_t)sl.idx[s] + 1 == i) {
        op = 2;
        half = 1;
      }
    }
    uint64_t acc = 0;
    if (op == 2u) {
      const uint64_t at = lo + i - half;
      uint64_t bi = 0, bv = 0;
      bool any = false;
#pragma unroll
      for (int r = 0; r < kMaxPeers; ++r) {
        if (r < (int)g) {
          const uint64_t x = ld_stream_u64(src.p[r] + at), v = ld_stream_u64(src.p[r] + at + 1);
          if (!any || v > bv || (v == bv && x < bi)) {
            bi = x;
            bv = v;
            any = true;
          }
        }
      }
      acc = half ? bv : bi;
    } else if (op != 3u) {
#pragma unroll
      for (int r = 0; r < kMaxPeers; ++r) {
        if (r < (int)g) {
          const uint64_t v = ld_stream_u64(src.p[r] + lo + i);
          acc = op == 1u ? (v > acc ? v : acc) : acc + v;
        }
      }
    }
    out[i] = acc;
  }
}

// Up to kMaxCopies copies / atomic adds in one launch (grid-stride inside every entry).
__global__ void __launch_bounds__(kBlock) peer_gather_kernel(const __grid_constant__ PeerCopyTable t) {
  const uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x, nt = (uint64_t)gridDim.x * kBlock;
  for (uint32_t j = 0; j < t.count; ++j) {
    const uint64_t* __restrict__ src = t.e[j].src;
    uint64_t* __restrict__ dst = t.e[j].dst;
    const uint64_t n = t.e[j].n;
    if (t.e[j].op == 0u) {
      for (uint64_t i = tid; i < n; i += nt) dst[i] = ld_stream_u64(src + i);
    } else {
      for (uint64_t i = tid; i < n; i += nt) {
        const uint64_t v = ld_stream_u64(src + i);
        if (v) red_add_u64(dst + i, v);
      }
    }
  }
}

int grid_for(uint64_t items, int per_block, int cap) {
  const uint64_t b = (items + per_block - 1) / per_block;
  return (int)(b < 1 ? 1 : (b > (uint64_t)cap ? cap : b));
}

}  // namespace

cudaError_t launch_peer_small(const PeerSrc& src, uint32_t g, uint64_t lo, uint64_t n, const PeerSlots& sl,
                              uint64_t* out, int grid, cudaStream_t st) {
  peer_small_kernel<<<grid_for(n, kBlock, grid), kBlock, 0, st>>>(src, g, lo, n, sl, out);
  return cudaGetLastError();
}

cudaError_t launch_peer_gather(const PeerCopyTable& t, int grid, cudaStream_t st) {
  uint64_t most = 1;
  for (uint32_t j = 0; j < t.count; ++j) most = t.e[j].n > most ? t.e[j].n : most;
  peer_gather_kernel<<<grid_for(most, kBlock, grid), kBlock, 0, st>>>(t);
  return cudaGetLastError();
}

cudaError_t launch_peer_reduce(const PeerSrc& src, uint32_t g, uint64_t lo, uint64_t n, uint32_t op, uint64_t* out,
                               uint64_t* out_bitmap, uint64_t* out_popcount, int grid, cudaStream_t st) {
  if (op == 2) {
    peer_argmax_kernel<<<1, 1, 0, st>>>(src, g, lo, out);
  } else if (op == 0 && (out_bitmap || out_popcount)) {
    const uint64_t words = n / 64;
    peer_sum_bitmap_kernel<<<grid_for(words, kBlock / 32, grid), kBlock, 0, st>>>(src, g, lo, words, out,
                                                                                 out_bitmap, out_popcount);
  } else if (op == 0) {
    peer_elementwise_kernel<false><<<grid_for(n, kBlock, grid), kBlock, 0, st>>>(src, g, lo, n, out);
  } else {
    peer_elementwise_kernel<true><<<grid_for(n, kBlock, grid), kBlock, 0, st>>>(src, g, lo, n, out);
  }
  return cudaGetLastError();
}

}  // namespace pasta
