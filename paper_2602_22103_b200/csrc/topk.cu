// topk.cu -- S4: top-K hot pages by radix select, deterministic ties.
//
// The paper motivates the list ("long-lived hot data ... good candidates for
// prefetching and can be pinned in device memory using ... cudaMemPrefetchAsync and
// cudaMemAdvise") but gives no algorithm. Result order (R10): count
// descending, then page ascending; only non-zero pages; K' = min(K, nnz).
//
// Pipeline (all on the device, no host synchronization; the host never learns nnz):
//  1. one pass: per-CTA shared histogram of a monotone 11-bit "float" key of every
//     non-zero count (bit length + the 5 bits below the leading one); block 0 derives
//     nnz, K' = min(K, nnz) and the bin holding the K'-th largest count;
//  2. up to six MSD radix passes of 11 bits over the counts inside the selected bin,
//     each followed by a 1-CTA select of the digit where the running count from the
//     top reaches the remaining rank; they stop as soon as a bin is taken whole, so
//     T (take every count > T) and `need` (how many pages with count == T) are fixed;
//  3. gather: pages with count > T go to atomically reserved slots (their order is
//     fixed by the sort) in the same pass that counts each CTA's `== T` pages; only if
//     ties are cut, the CTAs that hold needed ties re-read their range and rank those
//     pages in ascending page order with block exclusive scans (no atomics decide
//     which are taken);
//  4. bitonic sort of the K' (padded to a power of two with (0, UINT64_MAX) sentinels
//     that sort last) by (count desc, page asc): shared-memory tiles of 2048, global
//     compare-exchange steps for the larger strides; sentinels fill slots [K', K).
#include <cstdint>

#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace pasta {
namespace {

using namespace dev;

constexpr int kBlock = 256;
constexpr int kTile = 2048;  // bitonic shared-memory tile (elements)

struct State {
  unsigned long long nnz, kprime;
  unsigned long long lo;         // selected bin: counts in [lo, lo + 2^(shift+width) - 1]
  unsigned long long above;      // pages with a count above the bin (all taken)
  unsigned long long remaining;  // pages still to take from the bin
  long long shift;               // low bit of the next digit
  long long width;               // bits in the next digit
  unsigned long long done;       // 0 refining, 1 nothing to select, 2 threshold fixed
  unsigned long long T, need;    // take every count > T and the first `need` pages with count == T
  unsigned long long gt_slots;
  unsigned long long pad[5];
};

constexpr int kDigitBits = 11;
constexpr int kBins = 1 << kDigitBits;

struct Scratch {
  State* st;
  unsigned* hist;              // [kBins]
  unsigned long long* blkcnt;  // [grid]
  uint64_t* key_c;             // [Kp] counts
  uint64_t* key_p;             // [Kp] pages
};

__device__ __forceinline__ bool before(uint64_t c1, uint64_t p1, uint64_t c2, uint64_t p2) {
  return c1 > c2 || (c1 == c2 && p1 < p2);
}

// Warp-aggregated shared-memory histogram increment: lanes with equal bins are grouped
// with __match_any_sync and the group leader adds the group size (counts are heavily
// tied, so plain per-lane atomics would serialize on one bin).
// Shared-memory histogram increment.
__device__ __forceinline__ void hist_add(unsigned* h, bool valid, unsigned bin) {
  if (valid) atomicAdd(&h[bin], 1u);
}

// Streaming helper: visit every pair index i < n2 of this grid with kU 16-byte loads in
// flight per thread (enough memory-level parallelism to stream P x 8 bytes at HBM speed).
#ifndef PASTA_TOPK_U
#define PASTA_TOPK_U 8
#endif
constexpr int kU = PASTA_TOPK_U;
#ifndef PASTA_TOPK_CTAS_PER_SM
#define PASTA_TOPK_CTAS_PER_SM 4  // co-resident CTAs per SM of the cooperative selection kernel
#endif  // 16-byte loads in flight per thread in the streaming passes
template <typename F>
__device__ __forceinline__ void stream_pairs(const ulonglong2* __restrict__ pc2, uint64_t n2, F f) {
  const uint64_t stride = (uint64_t)gridDim.x * kBlock * kU;
  for (uint64_t base = (uint64_t)blockIdx.x * kBlock * kU + threadIdx.x; base < n2; base += stride) {
    ulonglong2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = base + (uint64_t)u * kBlock;
      v[u] = i < n2 ? __ldg(pc2 + i) : make_ulonglong2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = base + (uint64_t)u * kBlock;
      if (i < n2) f(i, v[u]);
    }
  }
}

// ---- selection passes (device functions of the one cooperative selection kernel) ----

// Pass 1 key: a monotone 11-bit "float" of a non-zero count c with bit length L:
// c itself for L <= 6 (exact bins 1..63), else 64 + 32 (L - 7) + the 5 bits below the
// leading one (bins 64..1919, each covering 2^(L-6) consecutive counts). One pass
// resolves the bit length and five more bits.
constexpr int kFirstBins = 64 + 58 * 32;  // 1920
static_assert(kFirstBins <= kBins, "pass-1 bins share the digit histogram buffers");
__device__ __forceinline__ unsigned first_key(uint64_t c) {
  const int L = 64 - __clzll((long long)c);
  return L <= 6 ? (unsigned)c : 64u + (unsigned)(L - 7) * 32u + (unsigned)((c >> (L - 6)) & 31u);
}

// Pass 1: histogram of first_key over the non-zero counts.
__device__ void dev_first(const uint64_t* __restrict__ pc, uint64_t P, unsigned* h, unsigned* hist) {
  for (int i = threadIdx.x; i < kFirstBins; i += kBlock) h[i] = 0;
  __syncthreads();
  stream_pairs(reinterpret_cast<const ulonglong2*>(pc), P / 2, [&](uint64_t, const ulonglong2& v) {
    hist_add(h, v.x != 0, first_key(v.x));
    hist_add(h, v.y != 0, first_key(v.y));
  });
  if ((P & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint64_t c = pc[P - 1];
    if (c) atomicAdd(&h[first_key(c)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kFirstBins; i += kBlock)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// Block-wide search (block 0, all threads) for the bin d of hist[0, nb) holding rank
// `rem` counted from the top: suffix(d + 1) < rem <= suffix(d). Thread t sums bins
// [t * per, (t + 1) * per); a block suffix scan of those sums (warp shuffles + one
// shared step) finds the one thread whose chunk holds d, which walks its <= per bins.
// Returns true in that thread only, with d, the count above bin d and the rank left
// inside it. `total` (every thread) = the sum of all bins.
__device__ bool block_find_bin(const unsigned* hist, int nb, int per, unsigned long long rem,
                               unsigned long long* sm, unsigned long long& total, int& d_out,
                               unsigned long long& above_out, unsigned long long& rem_out) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  unsigned long long mine = 0;
  for (int j = 0; j < per; ++j) {
    const int d = t * per + j;
    if (d < nb) mine += hist[d];
  }
  unsigned long long v = mine;  // suffix sum within the warp (lanes >= lane)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long x = __shfl_down_sync(kFull, v, o);
    if (lane + o < 32) v += x;
  }
  if (lane == 0) sm[w] = v;
  __syncthreads();
  unsigned long long after = 0;  // warps above this one
  total = 0;
  for (int i = 0; i < kBlock / 32; ++i) {
    total += sm[i];
    if (i > w) after += sm[i];
  }
  __syncthreads();
  const unsigned long long S = v + after, S_next = S - mine;  // suffix from my chunk / the next
  if (!(S_next < rem && rem <= S)) return false;
  rem -= S_next;
  unsigned long long above = S_next;
  int d = t * per + per - 1;
  if (d > nb - 1) d = nb - 1;
  for (; d > t * per; --d) {
    if (hist[d] >= rem) break;
    rem -= hist[d];
    above += hist[d];
  }
  d_out = d;
  above_out = above;
  rem_out = rem;
  return true;
}

// Pick the pass-1 bin holding the K'-th largest count (block 0, all threads): nnz,
// K' = min(K, nnz) and the bin; then the threshold state.
__device__ void dev_select_first(volatile State* st, unsigned* hist, uint64_t K, uint64_t Kp, unsigned long long* sm) {
  constexpr int per = (kFirstBins + kBlock - 1) / kBlock;  // bins per thread
  unsigned long long nnz = 0, above = 0, rem = 0;
  int d = 0;
  // the rank is only known after the total: first pass for nnz, the search inside
  unsigned long long part = 0;
  for (int j = 0; j < per; ++j) {
    const int b = threadIdx.x * per + j;
    if (b < kFirstBins) part += hist[b];
  }
  part = warp_sum_u64(part);
  if ((threadIdx.x & 31) == 0) sm[kBlock / 32 + (threadIdx.x >> 5)] = part;
  __syncthreads();
  for (int i = 0; i < kBlock / 32; ++i) nnz += sm[kBlock / 32 + i];
  const unsigned long long kp = nnz < K ? nnz : K;
  if (kp == 0) {
    if (threadIdx.x == 0) {
      st->nnz = 0;
      st->kprime = 0;
      st->gt_slots = 0;
      st->need = 0;
      st->done = 1;
      st->T = ~0ull;
    }
  } else if (block_find_bin(hist, kFirstBins, per, kp, sm, nnz, d, above, rem)) {
    const unsigned long long here = hist[d];
    int bits = 0;  // the bin is [lo, lo + 2^bits - 1]
    unsigned long long lo = (unsigned long long)d;
    if (d >= 64) {
      const int L = (d - 64) / 32 + 7;
      bits = L - 6;
      lo = (32ull + (unsigned)((d - 64) % 32)) << bits;
    }
    st->nnz = nnz;
    st->kprime = kp;
    st->gt_slots = 0;
    st->need = 0;
    st->lo = lo;
    st->above = above;
    st->remaining = rem;
    if (rem == here) {  // the whole bin is taken: no ties to break
      st->done = 2;
      st->T = lo - 1;
    } else if (above + here <= Kp) {  // every count >= lo fits the sort: it picks the first K'
      st->done = 2;
      st->T = lo - 1;
    } else if (bits == 0) {  // exact value: take the first `rem` pages with this count
      st->done = 2;
      st->T = lo;
      st->need = rem;
    } else {
      const int w = bits < kDigitBits ? bits : kDigitBits;
      st->width = w;
      st->shift = bits - w;
      st->done = 0;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += kBlock) hist[i] = 0;
}

// One radix digit among the counts of the selected bin.
__device__ void dev_digit(const uint64_t* __restrict__ pc, uint64_t P, volatile State* st, unsigned* h,
                          unsigned* hist) {
  const uint64_t lo = st->lo;
  const int shift = (int)st->shift, width = (int)st->width;
  for (int i = threadIdx.x; i < (1 << width); i += kBlock) h[i] = 0;
  __syncthreads();
  const uint64_t span = (1ull << (shift + width)) - 1;  // bin = [lo, lo + span]
  stream_pairs(reinterpret_cast<const ulonglong2*>(pc), P / 2, [&](uint64_t, const ulonglong2& v) {
    hist_add(h, v.x - lo <= span, (unsigned)((v.x - lo) >> shift));
    hist_add(h, v.y - lo <= span, (unsigned)((v.y - lo) >> shift));
  });
  if ((P & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint64_t c = pc[P - 1];
    if (c - lo <= span) atomicAdd(&h[(c - lo) >> shift], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (1 << width); i += kBlock)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// Choose the digit (block 0, all threads) where the running count from the top
// reaches the remaining rank.
__device__ void dev_select_digit(volatile State* st, unsigned* hist, uint64_t Kp, unsigned long long* sm) {
  const int shift = (int)st->shift, width = (int)st->width;
  const unsigned long long rem0 = st->remaining, above0 = st->above, lo0 = st->lo;
  __syncthreads();  // every thread has read the state before the winner rewrites it
  const int nb = 1 << width;
  const int per = (nb + kBlock - 1) / kBlock;  // bins per thread (<= 8)
  unsigned long long total = 0, above = 0, rem = 0;
  int d = 0;
  if (block_find_bin(hist, nb, per, rem0, sm, total, d, above, rem)) {
    const unsigned long long here = hist[d];
    const unsigned long long lo = lo0 + ((unsigned long long)d << shift);
    st->lo = lo;
    st->above = above0 + above;
    st->remaining = rem;
    if (rem == here || above0 + above + here <= Kp) {  // whole bin, or all counts >= lo fit the sort
      st->done = 2;
      st->T = lo - 1;
    } else if (shift == 0) {  // exact value: take the first `rem` pages with this count
      st->done = 2;
      st->T = lo;
      st->need = rem;
    } else {
      const int w = shift < kDigitBits ? shift : kDigitBits;
      st->width = w;
      st->shift = shift - w;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += kBlock) hist[i] = 0;
}

// Gather (one pass over this CTA's contiguous page range): every page with count > T
// to an atomically reserved slot (the sort fixes the order), and the number of pages
// with count == T to blkcnt[cta].
__device__ void dev_gather_gt(const uint64_t* __restrict__ pc, uint64_t P, volatile State* st,
                              unsigned long long* blkcnt, uint64_t* key_c, uint64_t* key_p,
                              unsigned long long* part) {
  const uint64_t T = st->T;
  const uint64_t b0 = (uint64_t)blockIdx.x * P / gridDim.x, b1 = (uint64_t)(blockIdx.x + 1) * P / gridDim.x;
  uint64_t n = 0;
  for (uint64_t p0 = b0 + threadIdx.x; p0 < b1; p0 += (uint64_t)kBlock * kU) {
    uint64_t v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t p = p0 + (uint64_t)u * kBlock;
      v[u] = p < b1 ? __ldg(pc + p) : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t p = p0 + (uint64_t)u * kBlock;
      n += (p < b1 && v[u] == T) ? 1u : 0u;
      if (v[u] > T) {
        const unsigned long long slot = atomicAdd((unsigned long long*)&st->gt_slots, 1ull);
        key_c[slot] = v[u];
        key_p[slot] = p;
      }
    }
  }
  n = warp_sum_u64(n);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s2 = 0;
    for (int i = 0; i < kBlock / 32; ++i) s2 += part[i];
    blkcnt[blockIdx.x] = s2;
  }
}

// Ties (after a grid barrier): pages with count == T ranked in ascending page order
// (block exclusive scans over the CTA ranges, no atomics decide which), the first
// `need` kept in slots [K' - need, K'). Only CTAs whose range holds such pages and whose
// predecessors do not already supply `need` re-read their range (at most `need` CTAs).
__device__ void dev_gather_eq(const uint64_t* __restrict__ pc, uint64_t P, volatile State* st,
                              const unsigned long long* blkcnt, uint64_t* key_c, uint64_t* key_p,
                              unsigned long long* part, unsigned long long* running_s) {
  const uint64_t T = st->T, need = st->need, kp = st->kprime;
  if (blkcnt[blockIdx.x] == 0) return;
  const uint64_t eq_base_slot = kp - need;
  const uint64_t b0 = (uint64_t)blockIdx.x * P / gridDim.x, b1 = (uint64_t)(blockIdx.x + 1) * P / gridDim.x;
  unsigned long long pre = 0;
  for (unsigned i = threadIdx.x; i < blockIdx.x; i += kBlock) pre += blkcnt[i];
  pre = warp_sum_u64(pre);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = pre;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s2 = 0;
    for (int i = 0; i < kBlock / 32; ++i) s2 += part[i];
    *running_s = s2;
  }
  __syncthreads();
  bool ties = *running_s < need;
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (uint64_t t0 = b0; ties && t0 < b1; t0 += kBlock) {
    const uint64_t p = t0 + threadIdx.x;
    const bool eq = p < b1 && __ldg(pc + p) == T;
    const unsigned bal = __ballot_sync(kFull, eq);
    const unsigned long long rank_w = __popc(bal & ((1u << lane) - 1));
    __syncthreads();
    if (lane == 0) part[wib] = __popc(bal);
    __syncthreads();
    unsigned long long off = *running_s;
    for (unsigned i = 0; i < wib; ++i) off += part[i];
    if (eq) {
      const unsigned long long r = off + rank_w;
      if (r < need) {
        key_c[eq_base_slot + r] = T;
        key_p[eq_base_slot + r] = p;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s2 = 0;
      for (int i = 0; i < kBlock / 32; ++i) s2 += part[i];
      *running_s += s2;
    }
    __syncthreads();
    ties = *running_s < need;
  }
}

// The whole selection in ONE cooperative launch: the float-key pass, up to six 11-bit
// digit passes (stopping as soon as the threshold is fixed), the gather of counts > T
// with per-CTA tie counts and, if ties are cut, the ordered tie gather, separated by
// grid-wide barriers.
__global__ void __launch_bounds__(kBlock) select_coop_kernel(const uint64_t* __restrict__ pc, uint64_t P,
                                                             uint64_t K, uint64_t Kp, State* st_, unsigned* hist,
                                                             unsigned long long* blkcnt, uint64_t* key_c,
                                                             uint64_t* key_p) {
  cg::grid_group grid = cg::this_grid();
  volatile State* st = st_;
  __shared__ unsigned h[kBins];
  __shared__ unsigned long long sm[kBlock];
  __shared__ unsigned long long running_s;
  dev_first(pc, P, h, hist);
  grid.sync();
  if (blockIdx.x == 0) dev_select_first(st, hist, K, Kp, sm);
  grid.sync();
  for (int pass = 0; pass < (63 + kDigitBits - 1) / kDigitBits; ++pass) {
    if (st->done) break;  // grid-uniform: read after the barrier
    dev_digit(pc, P, st, h, hist);
    grid.sync();
    if (blockIdx.x == 0) dev_select_digit(st, hist, Kp, sm);
    grid.sync();
  }
  if (st->done != 2) return;
  dev_gather_gt(pc, P, st, blkcnt, key_c, key_p, sm);
  if (st->need == 0) return;  // grid-uniform
  grid.sync();
  dev_gather_eq(pc, P, st, blkcnt, key_c, key_p, sm, &running_s);
}

__global__ void pad_kernel(State* st, uint64_t* key_c, uint64_t* key_p, uint64_t Kp) {
  // filled slots: K' (threshold + ties) or every candidate >= the bin (need = 0)
  const uint64_t kp = st->need ? st->kprime : st->gt_slots;
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

// Whole bitonic sort of Kp <= 1024 keys in one CTA, one key per thread: strides below
// 32 exchange through warp shuffles (no shared memory, no barrier), larger strides
// through shared memory. Same network and order as bitonic_tile_kernel.
__global__ void __launch_bounds__(1024) bitonic_small_kernel(uint64_t* key_c, uint64_t* key_p, uint32_t Kp) {
  __shared__ uint64_t sc[1024], sp[1024];
  const uint32_t i = threadIdx.x;
  const unsigned mask = Kp >= 32 ? kFull : (1u << Kp) - 1u;  // the one partial warp when Kp < 32
  uint64_t c = key_c[i], p = key_p[i];
  for (uint32_t size = 2; size <= Kp; size <<= 1) {
    const bool asc = (i & size) == 0;
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      uint64_t oc, op;
      if (stride >= 32) {
        sc[i] = c;
        sp[i] = p;
        __syncthreads();
        oc = sc[i ^ stride];
        op = sp[i ^ stride];
        __syncthreads();
      } else {
        oc = __shfl_xor_sync(mask, c, stride);
        op = __shfl_xor_sync(mask, p, stride);
      }
      // the lower index of the pair keeps the element that comes first (asc) or last
      const bool other_first = before(oc, op, c, p);
      const bool lower = (i & stride) == 0;
      if (lower == asc ? other_first : !other_first) {
        c = oc;
        p = op;
      }
    }
  }
  key_c[i] = c;
  key_p[i] = p;
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
                             uint64_t* out_page, uint64_t* out_count, uint64_t* out_found, int from_nnz) {
  const uint64_t kp = from_nnz ? (st->nnz < K ? st->nnz : K) : st->kprime;
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

// Candidates of g shard-local top-K lists (rank-major, k entries each) -> sort keys with
// global page ids (page + r * shard_pages); empty slots (count 0) become sentinels.
__global__ void merge_load_kernel(const uint64_t* __restrict__ cand_page, const uint64_t* __restrict__ cand_count,
                                  uint32_t g, uint32_t k, uint64_t shard_pages, State* st, uint64_t* key_c,
                                  uint64_t* key_p, uint64_t Kp) {
  uint64_t nz = 0;
  const uint64_t n = (uint64_t)g * k;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Kp; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = 0, p = ~0ull;
    if (i < n) {
      c = cand_count[i];
      if (c) p = cand_page[i] + (i / k) * shard_pages;
    }
    key_c[i] = c;
    key_p[i] = c ? p : ~0ull;
    nz += (c != 0);
  }
  nz = warp_sum_u64(nz);
  if ((threadIdx.x & 31) == 0 && nz) atomicAdd(&st->nnz, (unsigned long long)nz);
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
  b += kBins * sizeof(unsigned);
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
  return 256 + kBins * sizeof(unsigned) + ((size_t)grid * 8 + 255) / 256 * 256 + 2 * Kp * 8;
}

#define PASTA_TRY(x)                         \
  do {                                       \
    cudaError_t e_ = (x);                    \
    if (e_ != cudaSuccess) return e_;        \
    if (n_launches) ++*n_launches;           \
  } while (0)

// Bitonic sort of Kp (power of two) keys by (count desc, page asc).
cudaError_t sort_keys(uint64_t* key_c, uint64_t* key_p, uint64_t Kp, int grid, cudaStream_t st, int* n_launches) {
  if (Kp <= 1024) {
    bitonic_small_kernel<<<1, (unsigned)Kp, 0, st>>>(key_c, key_p, (uint32_t)Kp);
    PASTA_TRY(cudaGetLastError());
    return cudaSuccess;
  }
  const uint64_t tile = Kp < (uint64_t)kTile ? Kp : (uint64_t)kTile;
  const int tiles = (int)((Kp + kTile - 1) / kTile);
  bitonic_tile_kernel<<<tiles, 1024, 0, st>>>(key_c, key_p, Kp, 2, tile, ~0ull);
  PASTA_TRY(cudaGetLastError());
  for (uint64_t size = 2 * (uint64_t)kTile; size <= Kp; size <<= 1) {
    for (uint64_t stride = size >> 1; stride >= (uint64_t)kTile; stride >>= 1) {
      int gg = (int)((Kp / 2 + kBlock - 1) / kBlock);
      if (gg > grid) gg = grid;
      bitonic_global_kernel<<<gg, kBlock, 0, st>>>(key_c, key_p, Kp, size, stride);
      PASTA_TRY(cudaGetLastError());
    }
    bitonic_tile_kernel<<<tiles, 1024, 0, st>>>(key_c, key_p, Kp, size, size, kTile / 2);
    PASTA_TRY(cudaGetLastError());
  }
  return cudaSuccess;
}

cudaError_t run_topk(const uint64_t* pc, uint64_t P, uint32_t k, uint64_t* out_page, uint64_t* out_count,
                     uint64_t* out_found, void* scratch, int grid, cudaStream_t st, int* n_launches) {
  const uint64_t Kp = pow2_ceil(k < 2 ? 2 : k);
  Scratch s = carve(scratch, Kp, grid);
  cudaError_t e = cudaMemsetAsync(scratch, 0, 256 + kBins * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  {
    static int coop_blocks = 0;  // co-resident blocks per SM for the cooperative launch
    if (coop_blocks == 0) {
      int nb = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, select_coop_kernel, kBlock, 0) != cudaSuccess || nb < 1)
        nb = 1;
      coop_blocks = nb;
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int g = sms * (coop_blocks < PASTA_TOPK_CTAS_PER_SM ? coop_blocks : PASTA_TOPK_CTAS_PER_SM);
    const uint64_t need_blocks = (P + kBlock - 1) / kBlock;
    if ((uint64_t)g > need_blocks) g = (int)(need_blocks < 1 ? 1 : need_blocks);
    if (g > grid) g = grid;
    uint64_t K64 = k, Kp64 = Kp;
    void* args[] = {(void*)&pc, (void*)&P, (void*)&K64, (void*)&Kp64, (void*)&s.st, (void*)&s.hist,
                    (void*)&s.blkcnt, (void*)&s.key_c, (void*)&s.key_p};
    PASTA_TRY(cudaLaunchCooperativeKernel((void*)select_coop_kernel, dim3(g), dim3(kBlock), args, 0, st));
  }
  const int pg = (int)((Kp + 1023) / 1024 < 1024 ? (Kp + 1023) / 1024 : 1024);
  pad_kernel<<<pg, 1024, 0, st>>>(s.st, s.key_c, s.key_p, Kp);
  PASTA_TRY(cudaGetLastError());
  e = sort_keys(s.key_c, s.key_p, Kp, grid, st, n_launches);
  if (e != cudaSuccess) return e;
  int wg = (int)((k + 255) / 256);
  if (wg > grid) wg = grid;
  write_kernel<<<wg, 256, 0, st>>>(s.st, s.key_c, s.key_p, k, out_page, out_count, out_found, 0);
  PASTA_TRY(cudaGetLastError());
  return cudaSuccess;
}

cudaError_t run_topk_merge(const uint64_t* cand_page, const uint64_t* cand_count, uint32_t g, uint32_t k,
                           uint64_t shard_pages, uint64_t* out_page, uint64_t* out_count, uint64_t* out_found,
                           void* scratch, int grid, cudaStream_t st, int* n_launches) {
  const uint64_t n = (uint64_t)g * k;
  const uint64_t Kp = pow2_ceil(n < 2 ? 2 : n);
  Scratch s = carve(scratch, Kp, grid);
  cudaError_t e = cudaMemsetAsync(scratch, 0, 256, st);
  if (e != cudaSuccess) return e;
  int lg = (int)((Kp + 255) / 256);
  if (lg > grid) lg = grid;
  merge_load_kernel<<<lg, 256, 0, st>>>(cand_page, cand_count, g, k, shard_pages, s.st, s.key_c, s.key_p, Kp);
  PASTA_TRY(cudaGetLastError());
  e = sort_keys(s.key_c, s.key_p, Kp, grid, st, n_launches);
  if (e != cudaSuccess) return e;
  int wg = (int)((k + 255) / 256);
  if (wg > grid) wg = grid;
  write_kernel<<<wg, 256, 0, st>>>(s.st, s.key_c, s.key_p, k, out_page, out_count, out_found, 1);
  PASTA_TRY(cudaGetLastError());
  return cudaSuccess;
}

}  // namespace pasta
