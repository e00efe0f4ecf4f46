// topk.cu -- S4: top-K hot pages by radix select, deterministic ties.
//
// The paper motivates the list ("long-lived hot data ... good candidates for
// prefetching and can be pinned in device memory using ... cudaMemPrefetchAsync and
// cudaMemAdvise") but gives no algorithm. Result order (R10): count
// descending, then page ascending; only non-zero pages; K' = min(K, nnz).
//
// Pipeline (all on the device, no host synchronization; the host never learns nnz):
//  1. stats: nnz and max count (block reduce + atomics);
//  2. plan: K' = min(K, nnz); first 8-bit digit = the one holding max's MSB;
//  3. up to 8 MSD radix passes: per-CTA shared 256-bin histogram of the current digit
//     over the non-zero counts that match the selected prefix, global sum, then a
//     1-CTA select picks the digit where the running count from the top reaches the
//     remaining rank; after the last digit T = the K'-th largest count exactly and
//     `need` = how many pages with count == T are taken;
//  4. gather: pages with count > T go to atomically reserved slots (their order is
//     fixed by the sort); pages with count == T are ranked in ascending page order by
//     a per-CTA count pass + block exclusive scans (no atomics decide which are
//     taken), and the first `need` are kept;
//  5. bitonic sort of the K' (padded to a power of two with (0, UINT64_MAX) sentinels
//     that sort last) by (count desc, page asc): shared-memory tiles of 2048, global
//     compare-exchange steps for the larger strides; sentinels fill slots [K', K).
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace pasta {
namespace {

using namespace dev;

constexpr int kBlock = 256;
constexpr int kTile = 2048;  // bitonic shared-memory tile (elements)

struct State {
  unsigned long long nnz, maxc, kprime, remaining, prefix, mask;
  long long shift;
  unsigned long long done;  // 0 running, 1 nothing to select, 2 threshold found
  unsigned long long T, need, gt_slots;
  unsigned long long pad[5];
};

struct Scratch {
  State* st;
  unsigned* hist;              // [256]
  unsigned long long* blkcnt;  // [grid]
  uint64_t* key_c;             // [Kp] counts
  uint64_t* key_p;             // [Kp] pages
};

__device__ __forceinline__ bool before(uint64_t c1, uint64_t p1, uint64_t c2, uint64_t p2) {
  return c1 > c2 || (c1 == c2 && p1 < p2);
}

__global__ void __launch_bounds__(kBlock) stats_kernel(const uint64_t* __restrict__ pc, uint64_t P, State* st) {
  uint64_t nz = 0, mx = 0;
  for (uint64_t p = (uint64_t)blockIdx.x * kBlock + threadIdx.x; p < P; p += (uint64_t)gridDim.x * kBlock) {
    const uint64_t c = __ldg(pc + p);
    nz += (c != 0);
    mx = c > mx ? c : mx;
  }
  nz = warp_sum_u64(nz);
  mx = warp_max_u64(mx);
  if ((threadIdx.x & 31) == 0) {
    if (nz) atomicAdd(&st->nnz, (unsigned long long)nz);
    if (mx) atomicMax(&st->maxc, (unsigned long long)mx);
  }
}

__global__ void plan_kernel(State* st, uint64_t K) {
  if (threadIdx.x != 0) return;
  const uint64_t kp = st->nnz < K ? st->nnz : K;
  st->kprime = kp;
  st->remaining = kp;
  st->prefix = 0;
  st->mask = 0;
  st->gt_slots = 0;
  if (kp == 0) {
    st->done = 1;
    st->T = ~0ull;
    st->need = 0;
    return;
  }
  const int msb = 63 - __clzll((long long)st->maxc);
  st->shift = (msb / 8) * 8;
  st->done = 0;
}

__global__ void __launch_bounds__(kBlock) hist_kernel(const uint64_t* __restrict__ pc, uint64_t P, State* st,
                                                      unsigned* hist) {
  if (st->done) return;
  __shared__ unsigned h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t prefix = st->prefix, mask = st->mask;
  const int shift = (int)st->shift;
  for (uint64_t p = (uint64_t)blockIdx.x * kBlock + threadIdx.x; p < P; p += (uint64_t)gridDim.x * kBlock) {
    const uint64_t c = __ldg(pc + p);
    if (c != 0 && (c & mask) == prefix) atomicAdd(&h[(c >> shift) & 0xFF], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void select_kernel(State* st, unsigned* hist) {
  __shared__ unsigned long long suf[256];  // suf[d] = sum of hist[d'] for d' > d
  if (st->done) return;
  const int t = threadIdx.x;
  // inclusive suffix sums by a simple serial pass in thread 0 (256 entries)
  if (t == 0) {
    unsigned long long acc = 0;
    for (int d = 255; d >= 0; --d) {
      suf[d] = acc;
      acc += hist[d];
    }
  }
  __syncthreads();
  const unsigned long long rem = st->remaining;
  const unsigned long long above = suf[t], here = hist[t];
  __syncthreads();
  if (above < rem && rem <= above + here) {
    const int shift = (int)st->shift;
    st->remaining = rem - above;
    st->prefix |= (unsigned long long)t << shift;
    st->mask |= 0xFFull << shift;
    if (shift == 0) {
      st->T = st->prefix;
      st->need = rem - above;
      st->done = 2;
    } else {
      st->shift = shift - 8;
    }
  }
  hist[t] = 0;
}

// Pages with count == T per CTA over a contiguous page range.
__global__ void __launch_bounds__(kBlock) eq_count_kernel(const uint64_t* __restrict__ pc, uint64_t P, State* st,
                                                          unsigned long long* blkcnt) {
  if (st->done != 2) return;
  const uint64_t T = st->T;
  const uint64_t b0 = (uint64_t)blockIdx.x * P / gridDim.x, b1 = (uint64_t)(blockIdx.x + 1) * P / gridDim.x;
  uint64_t n = 0;
  for (uint64_t p = b0 + threadIdx.x; p < b1; p += kBlock) n += (__ldg(pc + p) == T);
  n = warp_sum_u64(n);
  __shared__ unsigned long long part[kBlock / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int i = 0; i < kBlock / 32; ++i) s += part[i];
    blkcnt[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kBlock) gather_kernel(const uint64_t* __restrict__ pc, uint64_t P, State* st,
                                                        const unsigned long long* blkcnt, uint64_t* key_c,
                                                        uint64_t* key_p) {
  if (st->done != 2) return;
  const uint64_t T = st->T, need = st->need, kp = st->kprime;
  const uint64_t eq_base_slot = kp - need;
  __shared__ unsigned long long part[kBlock / 32];
  __shared__ unsigned long long running;
  // exclusive prefix of the ==T counts of the CTAs before this one
  unsigned long long pre = 0;
  for (unsigned i = threadIdx.x; i < blockIdx.x; i += kBlock) pre += blkcnt[i];
  pre = warp_sum_u64(pre);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = pre;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int i = 0; i < kBlock / 32; ++i) s += part[i];
    running = s;
  }
  __syncthreads();
  const uint64_t b0 = (uint64_t)blockIdx.x * P / gridDim.x, b1 = (uint64_t)(blockIdx.x + 1) * P / gridDim.x;
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (uint64_t t0 = b0; t0 < b1; t0 += kBlock) {
    const uint64_t p = t0 + threadIdx.x;
    const uint64_t c = p < b1 ? __ldg(pc + p) : 0;
    if (p < b1 && c > T) {
      const unsigned long long slot = atomicAdd(&st->gt_slots, 1ull);
      key_c[slot] = c;
      key_p[slot] = p;
    }
    const bool eq = p < b1 && c == T;
    const unsigned bal = __ballot_sync(kFull, eq);
    const unsigned long long rank_w = __popc(bal & ((1u << lane) - 1));
    __syncthreads();
    if (lane == 0) part[wib] = __popc(bal);
    __syncthreads();
    unsigned long long off = running;
    for (unsigned i = 0; i < wib; ++i) off += part[i];
    if (eq) {
      const unsigned long long r = off + rank_w;
      if (r < need) {
        key_c[eq_base_slot + r] = c;
        key_p[eq_base_slot + r] = p;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int i = 0; i < kBlock / 32; ++i) s += part[i];
      running += s;
    }
    __syncthreads();
  }
}

__global__ void pad_kernel(State* st, uint64_t* key_c, uint64_t* key_p, uint64_t Kp) {
  const uint64_t kp = st->kprime;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Kp; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i >= kp) {
      key_c[i] = 0;
      key_p[i] = ~0ull;
    }
  }
}

// Bitonic network restricted to one tile in shared memory: for sizes in
// [size_lo, size_hi] and, for each size, strides from min(size/2, stride_hi) down to 1.
__global__ void __launch_bounds__(1024) bitonic_tile_kernel(uint64_t* key_c, uint64_t* key_p, uint64_t Kp,
                                                            uint64_t size_lo, uint64_t size_hi, uint64_t stride_hi) {
  __shared__ uint64_t sc[kTile], sp[kTile];
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
    const uint64_t g = t0 + i;
    sc[i] = g < Kp ? key_c[g] : 0;
    sp[i] = g < Kp ? key_p[g] : ~0ull;
  }
  __syncthreads();
  for (uint64_t size = size_lo; size <= size_hi; size <<= 1) {
    uint64_t s0 = size >> 1;
    if (s0 > stride_hi) s0 = stride_hi;
    for (uint64_t stride = s0; stride > 0; stride >>= 1) {
      for (int q = threadIdx.x; q < kTile / 2; q += blockDim.x) {
        // pair index q -> element i with bit `stride` clear
        const uint64_t lo = q & (stride - 1);
        const uint64_t i = ((q - lo) << 1) | lo;
        const uint64_t j = i | stride;
        const bool asc = ((t0 + i) & size) == 0;
        const bool swap = asc ? before(sc[j], sp[j], sc[i], sp[i]) : before(sc[i], sp[i], sc[j], sp[j]);
        if (swap) {
          const uint64_t c = sc[i], p = sp[i];
          sc[i] = sc[j];
          sp[i] = sp[j];
          sc[j] = c;
          sp[j] = p;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
    const uint64_t g = t0 + i;
    if (g < Kp) {
      key_c[g] = sc[i];
      key_p[g] = sp[i];
    }
  }
}

__global__ void __launch_bounds__(kBlock) bitonic_global_kernel(uint64_t* key_c, uint64_t* key_p, uint64_t Kp,
                                                                uint64_t size, uint64_t stride) {
  for (uint64_t q = (uint64_t)blockIdx.x * kBlock + threadIdx.x; q < Kp / 2; q += (uint64_t)gridDim.x * kBlock) {
    const uint64_t lo = q & (stride - 1);
    const uint64_t i = ((q - lo) << 1) | lo;
    const uint64_t j = i | stride;
    const bool asc = (i & size) == 0;
    const uint64_t ci = key_c[i], pi = key_p[i], cj = key_c[j], pj = key_p[j];
    const bool swap = asc ? before(cj, pj, ci, pi) : before(ci, pi, cj, pj);
    if (swap) {
      key_c[i] = cj;
      key_p[i] = pj;
      key_c[j] = ci;
      key_p[j] = pi;
    }
  }
}

__global__ void write_kernel(const State* st, const uint64_t* key_c, const uint64_t* key_p, uint64_t K,
                             uint64_t* out_page, uint64_t* out_count, uint64_t* out_found) {
  const uint64_t kp = st->kprime;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K; i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < kp) {
      out_page[i] = key_p[i];
      out_count[i] = key_c[i];
    } else {
      out_page[i] = ~0ull;
      out_count[i] = 0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_found = kp;
}

uint64_t pow2_ceil(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

Scratch carve(void* base, uint64_t Kp, int grid) {
  char* b = static_cast<char*>(base);
  Scratch s;
  s.st = reinterpret_cast<State*>(b);
  b += 256;
  s.hist = reinterpret_cast<unsigned*>(b);
  b += 256 * sizeof(unsigned);
  s.blkcnt = reinterpret_cast<unsigned long long*>(b);
  b += ((size_t)grid * 8 + 255) / 256 * 256;
  s.key_c = reinterpret_cast<uint64_t*>(b);
  b += Kp * 8;
  s.key_p = reinterpret_cast<uint64_t*>(b);
  return s;
}

}  // namespace

size_t topk_scratch_bytes(uint64_t k, int grid) {
  const uint64_t Kp = pow2_ceil(k < 2 ? 2 : k);
  return 256 + 256 * sizeof(unsigned) + ((size_t)grid * 8 + 255) / 256 * 256 + 2 * Kp * 8;
}

#define PASTA_TRY(x)                         \
  do {                                       \
    cudaError_t e_ = (x);                    \
    if (e_ != cudaSuccess) return e_;        \
    if (n_launches) ++*n_launches;           \
  } while (0)

cudaError_t run_topk(const uint64_t* pc, uint64_t P, uint32_t k, uint64_t* out_page, uint64_t* out_count,
                     uint64_t* out_found, void* scratch, int grid, cudaStream_t st, int* n_launches) {
  const uint64_t Kp = pow2_ceil(k < 2 ? 2 : k);
  Scratch s = carve(scratch, Kp, grid);
  cudaError_t e = cudaMemsetAsync(scratch, 0, 256 + 256 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  int g = (int)((P + kBlock - 1) / kBlock);
  if (g > grid) g = grid;
  if (g < 1) g = 1;
  stats_kernel<<<g, kBlock, 0, st>>>(pc, P, s.st);
  PASTA_TRY(cudaGetLastError());
  plan_kernel<<<1, 32, 0, st>>>(s.st, k);
  PASTA_TRY(cudaGetLastError());
  for (int pass = 0; pass < 8; ++pass) {
    hist_kernel<<<g, kBlock, 0, st>>>(pc, P, s.st, s.hist);
    PASTA_TRY(cudaGetLastError());
    select_kernel<<<1, 256, 0, st>>>(s.st, s.hist);
    PASTA_TRY(cudaGetLastError());
  }
  eq_count_kernel<<<grid, kBlock, 0, st>>>(pc, P, s.st, s.blkcnt);
  PASTA_TRY(cudaGetLastError());
  gather_kernel<<<grid, kBlock, 0, st>>>(pc, P, s.st, s.blkcnt, s.key_c, s.key_p);
  PASTA_TRY(cudaGetLastError());
  const int pg = (int)((Kp + 1023) / 1024 < 1024 ? (Kp + 1023) / 1024 : 1024);
  pad_kernel<<<pg, 1024, 0, st>>>(s.st, s.key_c, s.key_p, Kp);
  PASTA_TRY(cudaGetLastError());
  // bitonic sort of Kp keys
  const uint64_t tile = Kp < (uint64_t)kTile ? Kp : (uint64_t)kTile;
  const int tiles = (int)((Kp + kTile - 1) / kTile);
  bitonic_tile_kernel<<<tiles, 1024, 0, st>>>(s.key_c, s.key_p, Kp, 2, tile, ~0ull);
  PASTA_TRY(cudaGetLastError());
  for (uint64_t size = 2 * (uint64_t)kTile; size <= Kp; size <<= 1) {
    for (uint64_t stride = size >> 1; stride >= (uint64_t)kTile; stride >>= 1) {
      int gg = (int)((Kp / 2 + kBlock - 1) / kBlock);
      if (gg > grid) gg = grid;
      bitonic_global_kernel<<<gg, kBlock, 0, st>>>(s.key_c, s.key_p, Kp, size, stride);
      PASTA_TRY(cudaGetLastError());
    }
    bitonic_tile_kernel<<<tiles, 1024, 0, st>>>(s.key_c, s.key_p, Kp, size, size, kTile / 2);
    PASTA_TRY(cudaGetLastError());
  }
  int wg = (int)((k + 255) / 256);
  if (wg > grid) wg = grid;
  write_kernel<<<wg, 256, 0, st>>>(s.st, s.key_c, s.key_p, k, out_page, out_count, out_found);
  PASTA_TRY(cudaGetLastError());
  return cudaSuccess;
}

}  // namespace pasta
