// topk.cu -- S4: top-K hot pages by radix select, deterministic ties.
//
// The paper motivates the list ("long-lived hot data ... good candidates for
// prefetching and can be pinned in device memory using ... cudaMemPrefetchAsync and
// cudaMemAdvise") but gives no algorithm. Result order (R10): count
// descending, then page ascending; only non-zero pages; K' = min(K, nnz).
//
// pasta_topk is ONE cooperative kernel (selection by unique composite keys, see
// topk_kernel below): at most two passes over the P counts in the common case, the
// remaining radix digits resolved over a compacted candidate buffer, and the sort of the
// K' results in the same launch. pasta_topk_merge (g shard lists, multi-GPU) sorts the
// g * K candidates with the bitonic kernels at the end of this file.
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

// ---- selection by unique composite keys (one cooperative kernel) ----
//
// key(p) = (count << pbits) | (pmask - p), pbits = bit length of P - 1: a 128-bit
// integer, unique per page, whose descending order is exactly (count desc, page asc)
// (R10). The top-K' list is then the K' largest keys: there are no ties to break, and the
// selection is an MSD radix select over keys:
//  A. one pass over the counts: per-CTA shared histogram of a monotone 11-bit "float"
//     key of every non-zero count (bit length + the 5 bits below the leading one); every
//     CTA derives nnz, K' = min(K, nnz) and the bin holding the K'-th largest count,
//     i.e. a key range [rlo, rlo + 2^w - 1] and the rank left inside it;
//  B. one pass over the counts: keys above the range go to the output slots, keys inside
//     it are appended to a candidate buffer (capacity C) and counted into the histogram
//     of the range's next 11-bit digit; the digit holding the rank narrows the range;
//  C. while the range still has more keys than C (heavy ties over > C pages), more passes
//     like B; once the buffer holds the whole range, the remaining digits are resolved
//     over the buffer alone (C keys, not P counts);
//  D. as soon as the rank covers a whole digit bucket, every key >= its lower bound is
//     taken (from the buffer, or by one last pass);
//  E. the K' gathered keys are sorted descending (bitonic: one CTA in shared memory for
//     K' <= 2048, else grid-wide steps between grid barriers) and decoded into the
//     outputs; slots [K', K) get (UINT64_MAX, 0).
// Every CTA computes each digit choice itself from the same global histogram (read after
// the grid barrier), so one barrier per pass suffices. Nothing depends on the order of
// the atomics that reserve buffer / output slots: keys are unique and sorted at the end.
using u128 = unsigned __int128;

constexpr int kTB = 512;        // threads per block
constexpr int kTU = 4;          // 16-byte count loads in flight per thread
constexpr int kMaxPass = 11;    // pass 0 (float key) + <= ceil(96 / 11) digit passes
constexpr int kSortTile = 2048; // keys per shared-memory bitonic tile
constexpr uint64_t kBufMax = 1ull << 20;
constexpr uint32_t kFastMax = 4096;  // fast finish: <= this many candidates sorted by block 0 alone

struct TkHead {  // zeroed before every call
  unsigned hist[kMaxPass][kBins];
  unsigned long long fill[kMaxPass];  // keys that fell in the range during full pass i
  unsigned overflow[kMaxPass];        // some CTA's buffer region overflowed in full pass i
  unsigned long long slots;           // keys gathered into the output list
  unsigned long long cfill;           // keys of the first range copied to the compact list
};

constexpr size_t kHeadBytes = (sizeof(TkHead) + 255) / 256 * 256;  // a head's slot in the scratch
constexpr uint32_t kHeadWords = (uint32_t)(kHeadBytes / 16);

struct TkArgs {
  const uint64_t* pc;
  uint64_t P, K;
  TkHead* head;       // zero on entry (zeroed by the previous call or a memset)
  TkHead* next_head;  // the other head: zeroed by this launch for the next call
  u128* buf;     // candidate buffer: CTA c appends to its own region [c * rcap, (c + 1) * rcap)
  uint64_t rcap; // region capacity (keys)
  u128* keys;    // gathered keys [kcap]
  u128* compact; // [kFastMax] the first range's keys, contiguous (fast finish)
  uint64_t kcap;
  uint64_t* out_page;
  uint64_t* out_count;
  uint64_t* out_found;
  int pbits;
};

// Pass-1 key: a monotone 11-bit "float" of a non-zero count c with bit length L:
// c itself for L <= 6 (exact bins 1..63), else 64 + 32 (L - 7) + the 5 bits below the
// leading one (bins 64..1919, each covering 2^(L-6) consecutive counts).
constexpr int kFirstBins = 64 + 58 * 32;  // 1920
static_assert(kFirstBins <= kBins, "pass-1 bins fit the digit histogram");
__device__ __forceinline__ unsigned first_key(uint64_t c) {
  const int L = 64 - __clzll((long long)c);
  return L <= 6 ? (unsigned)c : 64u + (unsigned)(L - 7) * 32u + (unsigned)((c >> (L - 6)) & 31u);
}

__device__ __forceinline__ u128 make_key(uint64_t c, uint64_t p, int pbits, uint64_t pmask) {
  return ((u128)c << pbits) | (u128)(pmask - p);
}

// Streams the counts: f(p, c) for every page, called by every lane of every warp in step
// (zero counts for lanes past the end), so f may use warp collectives. 16-byte loads,
// kTU in flight per thread; an unaligned head element and an odd tail element are
// visited by warp 0 of block 0 at the end. With `rev` the blocks of kTB * kTU pairs are
// visited last to first: a pass that follows a forward pass then starts on the counts
// the forward pass read last, which are still in L2 (126 MB; the llama counts are 134 MB).
template <bool rev = false, typename F>
__device__ __forceinline__ void tk_stream(const uint64_t* __restrict__ pc, uint64_t P, F&& f) {
  const uint64_t h = ((reinterpret_cast<uintptr_t>(pc) & 15u) != 0 && P > 0) ? 1 : 0;
  const ulonglong2* v2 = reinterpret_cast<const ulonglong2*>(pc + h);
  const uint64_t n2 = (P - h) / 2;
  const uint64_t rows = (n2 + (uint64_t)kTB * kTU - 1) / ((uint64_t)kTB * kTU);
  for (uint64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint64_t b0 = (rev ? rows - 1 - r : r) * (uint64_t)kTB * kTU;
    ulonglong2 v[kTU];
#pragma unroll
    for (int u = 0; u < kTU; ++u) {
      const uint64_t i = b0 + (uint64_t)u * kTB + threadIdx.x;
      v[u] = i < n2 ? __ldg(v2 + i) : make_ulonglong2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < kTU; ++u) {
      const uint64_t i = b0 + (uint64_t)u * kTB + threadIdx.x;
      f(h + 2 * i, v[u].x);
      f(h + 2 * i + 1, v[u].y);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const bool tail = ((P - h) & 1) != 0;
    uint64_t p = 0, c = 0;
    if (threadIdx.x == 0 && h) c = __ldg(pc);
    if (threadIdx.x == 1 && tail) {
      p = P - 1;
      c = __ldg(pc + P - 1);
    }
    f(p, c);
  }
}

// Warp-aggregated append of `key` (lanes with want) to dst[*ctr ...], slots >= cap
// dropped (the counter still counts them). Every lane of the warp calls it. ctr may be
// a global or a shared counter.
__device__ __forceinline__ void warp_append(bool want, u128 key, u128* dst, unsigned long long* ctr, uint64_t cap) {
  const unsigned m = __ballot_sync(kFull, want);
  if (m == 0) return;
  const unsigned lane = threadIdx.x & 31u;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if ((int)lane == leader) base = atomicAdd(ctr, (unsigned long long)__popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (want) {
    const uint64_t slot = base + __popc(m & ((1u << lane) - 1u));
    if (slot < cap) dst[slot] = key;
  }
}

// Run-length shared-histogram increments: equal consecutive bins (tied counts) cost
// one shared atomic per run.
struct RunHist {
  unsigned bin = 0xFFFFFFFFu, n = 0;
  __device__ __forceinline__ void add(unsigned* sh, unsigned b) {
    if (b != bin) {
      if (n) atomicAdd(&sh[bin], n);
      bin = b;
      n = 0;
    }
    ++n;
  }
  __device__ __forceinline__ void flush(unsigned* sh) {
    if (n) atomicAdd(&sh[bin], n);
    n = 0;
  }
};

// Shared histogram -> global histogram gh (nb bins), shared bins re-zeroed.
__device__ __forceinline__ void hist_publish(unsigned* sh, unsigned* gh, int nb) {
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += kTB) {
    const unsigned v = sh[i];
    if (v) {
      atomicAdd(&gh[i], v);
      sh[i] = 0;
    }
  }
  __syncthreads();
}

struct Pick {
  unsigned long long above;  // keys in bins above d
  unsigned long long rem;    // rank left inside bin d
  unsigned long long here;   // keys in bin d
  unsigned long long total;  // all keys in the histogram
  int d;
};

// Every thread of the block: the bin d of the global histogram gh[0, nb) holding rank
// `rank` counted from the top (suffix(d + 1) < rank <= suffix(d)); with clamp, rank is
// first replaced by min(rank, total). Thread t sums bins [4t, 4t + 4); a block suffix
// scan finds the one thread whose chunk holds d; the result is broadcast via `out`.
__device__ Pick block_pick(const unsigned* gh, int nb, unsigned long long rank, bool clamp,
                           unsigned long long* sw, Pick* out) {
  constexpr int per = kBins / kTB;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  unsigned long long b[per], mine = 0;
#pragma unroll
  for (int j = 0; j < per; ++j) {
    const int d = t * per + j;
    b[j] = d < nb ? __ldcg(gh + d) : 0u;
    mine += b[j];
  }
  unsigned long long v = mine;  // suffix sum within the warp (lanes >= lane)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long x = __shfl_down_sync(kFull, v, o);
    if (lane + o < 32) v += x;
  }
  if (lane == 0) sw[w] = v;
  __syncthreads();
  unsigned long long after = 0, total = 0;
  for (int i = 0; i < kTB / 32; ++i) {
    total += sw[i];
    if (i > w) after += sw[i];
  }
  if (clamp && rank > total) rank = total;
  const unsigned long long S = v + after, Sn = S - mine;
  if (t == 0) {
    out->total = total;
    out->d = -1;
    out->above = out->rem = out->here = 0;
  }
  __syncthreads();
  if (rank > 0 && Sn < rank && rank <= S) {
    unsigned long long r = rank - Sn, above = Sn;
    int j = per - 1;
    for (; j > 0; --j) {
      if (b[j] >= r) break;
      r -= b[j];
      above += b[j];
    }
    out->d = t * per + j;
    out->above = above;
    out->rem = r;
    out->here = b[j];
  }
  __syncthreads();
  const Pick p = *out;
  __syncthreads();
  return p;
}

struct Sel {
  u128 rlo;    // current key range [rlo, rlo + 2^w - 1]
  u128 ghi;    // every key above ghi is already in the output list
  unsigned long long rem;  // how many keys of the range to take (from the top)
  int w;
  bool done;   // take every key >= rlo
};

__device__ __forceinline__ u128 range_hi(const Sel& s) { return s.rlo + (((u128)1 << s.w) - 1); }

// What a full pass acts on (shared memory, written by one thread before the pass).
struct PassCtl {
  u128 rlo, rhi;  // the range: keys appended to the region and counted by digit
  u128 glo, ghi;  // the gather interval: keys sent to the output list
  uint64_t pmask;
  int dsh;        // the digit's shift inside the range
  int rng;        // 0 once the selection is done (gather only)
};

// The per-element work of a full pass for a warp with at least one count >= cmin, out
// of line: the hot loop then holds only the loads and the count compare (no 128-bit
// range bounds live across it). Called by all 32 lanes together.
__device__ __noinline__ void full_slow(const TkArgs* a, const PassCtl* ctl, unsigned* sh, unsigned long long* sfill,
                                       uint64_t p, uint64_t c) {
  const u128 k = make_key(c, p, a->pbits, ctl->pmask);
  const bool g = c != 0 && k >= ctl->glo && k <= ctl->ghi;
  const bool r = ctl->rng && c != 0 && k >= ctl->rlo && k <= ctl->rhi;
  if (r) atomicAdd(&sh[(unsigned)((k - ctl->rlo) >> ctl->dsh)], 1u);
  warp_append(g, k, a->keys, &a->head->slots, a->kcap);
  if (ctl->rng) warp_append(r, k, a->buf + (uint64_t)blockIdx.x * a->rcap, sfill, a->rcap);
}

// A full pass over the counts: keys in (range_hi, ghi] (or [rlo, ghi] once done) to the
// output list; keys inside the range appended to this CTA's buffer region (shared-memory
// slot counter: no global atomic hot spot) and counted by next digit. Returns the keys
// this CTA found in the range (its region holds them all when that is <= rcap).
__device__ uint64_t tk_full_pass(const TkArgs& a, const Sel& s, int ps, unsigned* sh, unsigned long long* sfill,
                                 PassCtl* ctl, bool compact) {
  const bool rng = !s.done;
  const int dw = s.w < kDigitBits ? s.w : kDigitBits;
  if (threadIdx.x == 0) {
    ctl->rlo = s.rlo;
    ctl->rhi = range_hi(s);
    ctl->glo = s.done ? s.rlo : range_hi(s) + 1;
    ctl->ghi = s.ghi;
    ctl->pmask = a.pbits ? ((~0ull) >> (64 - a.pbits)) : 0ull;
    ctl->dsh = s.w - dw;
    ctl->rng = rng ? 1 : 0;
  }
  __syncthreads();
  TkHead* hd = a.head;
  // every key this pass acts on is >= rlo, i.e. has count >= rlo >> pbits (>= 1): a warp
  // whose counts are all below skips the key arithmetic (almost every count, every pass)
  const uint64_t cmin = (uint64_t)(s.rlo >> a.pbits);
  auto visit = [&](uint64_t p, uint64_t c) {
    if (__any_sync(kFull, c >= cmin)) full_slow(&a, ctl, sh, sfill, p, c);
  };
#ifndef PASTA_TOPK_REV
#define PASTA_TOPK_REV 1
#endif
  if (PASTA_TOPK_REV && (ps & 1))
    tk_stream<true>(a.pc, a.P, visit);  // right after a forward pass: start on its L2-resident tail
  else
    tk_stream<false>(a.pc, a.P, visit);
  if (!rng) return 0;
  hist_publish(sh, hd->hist[ps], 1 << dw);  // (its barriers also complete every append)
  const uint64_t mine = *sfill;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mine) atomicAdd(&hd->fill[ps], (unsigned long long)mine);
    if (mine > a.rcap) atomicOr(&hd->overflow[ps], 1u);
    *sfill = compact && mine ? atomicAdd(&hd->cfill, (unsigned long long)mine) : 0;
  }
  if (compact) {  // this CTA's range keys -> the contiguous list (if it still has room)
    __syncthreads();
    const uint64_t off = *sfill;
    if (mine <= a.rcap && off + mine <= kFastMax) {
      PASTA_DCHECK((uint64_t)(blockIdx.x + 1) * a.rcap * 16 <= a.rcap * 16 * gridDim.x);
      const u128* region = a.buf + (uint64_t)blockIdx.x * a.rcap;
      for (uint64_t i = threadIdx.x; i < mine; i += kTB) a.compact[off + i] = region[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) *sfill = 0;
  }
  return mine;
}

// A pass over this CTA's buffer region (n keys; together the regions hold the whole range
// of the last full pass): histogram of the current range's next digit, or (done) every
// key >= rlo to the output list.
__device__ void tk_buf_pass(const TkArgs& a, const Sel& s, int ps, uint64_t n, unsigned* sh) {
  const u128 rlo = s.rlo, rhi = range_hi(s);
  const int dw = s.w < kDigitBits ? s.w : kDigitBits;
  const int dsh = s.w - dw;
  const u128* region = a.buf + (uint64_t)blockIdx.x * a.rcap;
  RunHist rh;
  for (uint64_t b0 = 0; b0 < n; b0 += (uint64_t)kTB * kTU) {
    u128 v[kTU];
#pragma unroll
    for (int u = 0; u < kTU; ++u) {
      const uint64_t i = b0 + (uint64_t)u * kTB + threadIdx.x;
      v[u] = 0;
      if (i < n) {
        const ulonglong2 x = __ldcg(reinterpret_cast<const ulonglong2*>(region + i));
        v[u] = ((u128)x.y << 64) | x.x;
      }
    }
#pragma unroll
    for (int u = 0; u < kTU; ++u) {
      const u128 k = v[u];  // 0 is never a key (counts >= 1)
      if (s.done) {
        warp_append(k != 0 && k >= rlo, k, a.keys, &a.head->slots, a.kcap);
      } else if (k >= rlo && k <= rhi && k != 0) {
        rh.add(sh, (unsigned)((k - rlo) >> dsh));
      }
    }
  }
  rh.flush(sh);
  if (!s.done) hist_publish(sh, a.head->hist[ps], 1 << dw);
}

__device__ __forceinline__ u128 ld_key(const u128* p) {
  const ulonglong2 x = __ldcg(reinterpret_cast<const ulonglong2*>(p));
  return ((u128)x.y << 64) | x.x;
}

// Bitonic steps on n keys of a shared tile whose first key has global index gbase, for
// sizes [size_lo, size_hi] and strides from min(size / 2, stride_cap) down to 1;
// descending overall (pairs with (gbase + i) & size == 0 put the larger key first).
template <typename T>
__device__ void tile_bitonic(T* t, uint32_t n, uint64_t gbase, uint64_t size_lo, uint64_t size_hi,
                             uint64_t stride_cap) {
  for (uint64_t size = size_lo; size <= size_hi; size <<= 1) {
    uint64_t s0 = size >> 1;
    if (s0 > stride_cap) s0 = stride_cap;
    for (uint64_t stride = s0; stride > 0; stride >>= 1) {
      for (uint32_t q = threadIdx.x; q < n / 2; q += kTB) {
        const uint32_t lo = q & (uint32_t)(stride - 1);
        const uint32_t i = ((q - lo) << 1) | lo, j = i | (uint32_t)stride;
        const bool desc = ((gbase + i) & size) == 0;
        const T x = t[i], y = t[j];
        if (desc ? x < y : x > y) {
          t[i] = y;
          t[j] = x;
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ void put_key(const TkArgs& a, uint64_t i, u128 k, uint64_t pmask) {
  a.out_count[i] = (uint64_t)(k >> a.pbits);
  a.out_page[i] = pmask - (uint64_t)(k & (u128)pmask);
}

// Block 0: sort tile[0, n2) (n2 a power of two <= kFastMax) descending and write the
// first kprime keys to the outputs. When every key fits 64 bits (counts below
// 2^(64 - pbits): every realistic trace) the keys are re-packed as u64 in the same
// shared buffer first: half the shared-memory traffic and one compare per exchange.
__device__ __noinline__ void block_sort_write(const TkArgs* a, u128* tile, uint32_t n2, uint64_t kprime,
                                              uint64_t pmask) {
  constexpr int kPer = kFastMax / kTB;
  bool wide = false;
  for (uint32_t i = threadIdx.x; i < n2; i += kTB) wide |= (uint64_t)(tile[i] >> 64) != 0;
  if (__syncthreads_or(wide)) {
    tile_bitonic(tile, n2, 0, 2, n2, n2);
    for (uint32_t i = threadIdx.x; i < (uint32_t)kprime; i += kTB) put_key(*a, i, tile[i], pmask);
    return;
  }
  uint64_t v[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const uint32_t i = threadIdx.x + (uint32_t)e * kTB;
    v[e] = i < n2 ? (uint64_t)tile[i] : 0;
  }
  __syncthreads();
  uint64_t* t64 = reinterpret_cast<uint64_t*>(tile);
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const uint32_t i = threadIdx.x + (uint32_t)e * kTB;
    if (i < n2) t64[i] = v[e];
  }
  __syncthreads();
  tile_bitonic(t64, n2, 0, 2, n2, n2);
  for (uint32_t i = threadIdx.x; i < (uint32_t)kprime; i += kTB) put_key(*a, i, (u128)t64[i], pmask);
}

__global__ void __launch_bounds__(kTB, 2) topk_kernel(const __grid_constant__ TkArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned sh[kBins];
  __shared__ unsigned long long sw[kTB / 32];
  __shared__ Pick pk;
  __shared__ unsigned long long sfill;
  __shared__ PassCtl ctl;
  extern __shared__ u128 tile[];  // [kFastMax] (dynamic): sort tiles, the fast finish
  for (int i = threadIdx.x; i < kBins; i += kTB) sh[i] = 0;
  if (threadIdx.x == 0) sfill = 0;
  {  // the next call's head (no memset launch per call); nothing in this launch uses it
    uint4* nh = reinterpret_cast<uint4*>(a.next_head);
    for (uint32_t i = blockIdx.x * kTB + threadIdx.x; i < kHeadWords; i += gridDim.x * kTB)
      nh[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  __syncthreads();
  TkHead* hd = a.head;
  const uint64_t pmask = a.pbits ? ((~0ull) >> (64 - a.pbits)) : 0ull;

  // A: float-key histogram of the non-zero counts
  {
    RunHist rh;
    tk_stream(a.pc, a.P, [&](uint64_t, uint64_t c) {
      if (c) rh.add(sh, first_key(c));
    });
    rh.flush(sh);
    hist_publish(sh, hd->hist[0], kFirstBins);
  }
  grid.sync();
  const Pick p0 = block_pick(hd->hist[0], kFirstBins, a.K, true, sw, &pk);
  const uint64_t kprime = a.K < p0.total ? a.K : p0.total;
  bool fast = false;
  if (kprime > 0) {
    Sel s;
    uint64_t lo = (uint64_t)p0.d;
    int bits = 0;
    if (p0.d >= 64) {
      const int L = (p0.d - 64) / 32 + 7;
      bits = L - 6;
      lo = (32ull + (uint64_t)((p0.d - 64) % 32)) << bits;
    }
    s.rlo = (u128)lo << a.pbits;
    s.w = bits + a.pbits;
    s.rem = p0.rem;
    s.done = p0.here == p0.rem;
    s.ghi = ~(u128)0;
    bool buf_ok = false;
    uint64_t nbuf = 0;
    // B / C / D
    for (int ps = 1; ps < kMaxPass; ++ps) {
      if (!buf_ok) {
        const uint64_t mine = tk_full_pass(a, s, ps, sh, &sfill, &ctl, ps == 1 && !s.done);
        grid.sync();
        if (s.done) break;
        if (ps == 1) {
          // fast finish: the keys above the first range and the range itself (compacted)
          // are few: block 0 sorts them all and keeps the first K'; the others are done
          const uint64_t above = __ldcg(&hd->slots), total = __ldcg(&hd->fill[1]);
          // (only if no CTA's region overflowed: the compact list holds whole regions)
          if (total <= kFastMax && above + total <= kFastMax && __ldcg(&hd->overflow[1]) == 0u) {
            if (blockIdx.x == 0) {
              const uint32_t n = (uint32_t)(above + total);
              uint32_t n2 = 2;
              while (n2 < n) n2 <<= 1;
              for (uint32_t i = threadIdx.x; i < n2; i += kTB)
                tile[i] = i < above ? ld_key(a.keys + i) : (i < n ? ld_key(a.compact + (i - above)) : (u128)0);
              __syncthreads();
              block_sort_write(&a, tile, n2, kprime, pmask);
            }
            fast = true;
            break;
          }
        }
        s.ghi = range_hi(s);
        if (__ldcg(&hd->overflow[ps]) == 0u) {
          buf_ok = true;
          nbuf = mine;
        }
      } else {
        tk_buf_pass(a, s, ps, nbuf, sh);
        grid.sync();
        if (s.done) break;
      }
      const int dw = s.w < kDigitBits ? s.w : kDigitBits;
      const Pick q = block_pick(hd->hist[ps], 1 << dw, s.rem, false, sw, &pk);
      s.rlo += (u128)(uint64_t)q.d << (s.w - dw);
      s.w -= dw;
      s.rem = q.rem;
      s.done = q.here == q.rem || s.w == 0;
    }
  }
  // E: sort the K' gathered keys descending and write the outputs
  uint64_t kp2 = 2;
  while (kp2 < kprime) kp2 <<= 1;
  if (fast) {
    // written by block 0 above
  } else if (kp2 <= (uint64_t)kSortTile) {
    if (blockIdx.x == 0) {
      for (uint32_t i = threadIdx.x; i < (uint32_t)kp2; i += kTB) tile[i] = i < kprime ? ld_key(a.keys + i) : (u128)0;
      __syncthreads();
      block_sort_write(&a, tile, (uint32_t)kp2, kprime, pmask);
    }
  } else {
    const uint64_t nthreads = (uint64_t)gridDim.x * kTB, tid = (uint64_t)blockIdx.x * kTB + threadIdx.x;
    for (uint64_t i = kprime + tid; i < kp2; i += nthreads) a.keys[i] = 0;
    grid.sync();
    const uint64_t ntiles = kp2 / kSortTile;
    auto tile_pass = [&](uint64_t size_lo, uint64_t size_hi, uint64_t cap) {
      for (uint64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        u128* g = a.keys + tl * kSortTile;
        for (int i = threadIdx.x; i < kSortTile; i += kTB) tile[i] = ld_key(g + i);
        __syncthreads();
        tile_bitonic(tile, kSortTile, tl * kSortTile, size_lo, size_hi, cap);
        for (int i = threadIdx.x; i < kSortTile; i += kTB) g[i] = tile[i];
        __syncthreads();
      }
      grid.sync();
    };
    tile_pass(2, kSortTile, kSortTile);
    for (uint64_t size = 2 * (uint64_t)kSortTile; size <= kp2; size <<= 1) {
      for (uint64_t stride = size >> 1; stride >= (uint64_t)kSortTile; stride >>= 1) {
        for (uint64_t q = tid; q < kp2 / 2; q += nthreads) {
          const uint64_t lo = q & (stride - 1);
          const uint64_t i = ((q - lo) << 1) | lo, j = i | stride;
          const bool desc = (i & size) == 0;
          const u128 x = ld_key(a.keys + i), y = ld_key(a.keys + j);
          if (desc ? x < y : x > y) {
            a.keys[i] = y;
            a.keys[j] = x;
          }
        }
        grid.sync();
      }
      tile_pass(size, size, kSortTile / 2);
    }
    for (uint64_t i = tid; i < kprime; i += nthreads) put_key(a, i, ld_key(a.keys + i), pmask);
  }
  // slots [K', K): sentinels; found = K'
  for (uint64_t i = kprime + (uint64_t)blockIdx.x * kTB + threadIdx.x; i < a.K; i += (uint64_t)gridDim.x * kTB) {
    a.out_page[i] = ~0ull;
    a.out_count[i] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.out_found = kprime;
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

// Top-k lists as prefixes of one top-k_max list (R10's order is total, so the first k
// entries of the top-k_max list ARE the top-k list, sentinels included): entry j copies
// k_j entries and sets found_j = min(k_j, found_max). One launch for every entry.
__global__ void topk_prefix_kernel(const __grid_constant__ TopkPrefixTable t) {
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x, tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t j = 0; j < t.count; ++j) {
    const TopkPrefix& e = t.e[j];
    PASTA_DCHECK(t.count <= kMaxTopkPrefix);
    for (uint64_t i = tid; i < e.k; i += nt) {
      e.dst_page[i] = __ldg(t.src_page + i);
      e.dst_count[i] = __ldg(t.src_count + i);
    }
    if (tid == 0) {
      const uint64_t f = *t.src_found;
      *e.dst_found = f < e.k ? f : e.k;
    }
  }
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

// Candidate buffer region per CTA: the whole range of <= 2^20 keys split over the CTAs,
// at least 256 keys each.
uint64_t topk_region_cap(uint64_t P, int max_ctas) {
  const uint64_t tot = P < kBufMax ? P : kBufMax;
  const uint64_t r = (tot + (uint64_t)max_ctas - 1) / (uint64_t)max_ctas;
  return r < 256 ? 256 : r;
}

size_t topk_scratch_bytes(uint64_t k, uint64_t P, int max_ctas) {
  const uint64_t m = k < P ? k : P;
  const uint64_t Kp = pow2_ceil(m < 2 ? 2 : m);
  return 2 * kHeadBytes + 16ull * kFastMax + 16 * topk_region_cap(P, max_ctas) * (uint64_t)max_ctas + 16 * Kp;
}

size_t topk_merge_scratch_bytes(uint64_t n, int grid) {
  const uint64_t Kp = pow2_ceil(n < 2 ? 2 : n);
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
                     uint64_t* out_found, void* scratch, int max_ctas, cudaStream_t st, int* n_launches,
                     int* head_state) {
  const uint64_t m = (uint64_t)k < P ? (uint64_t)k : P;
  TkArgs a;
  a.pc = pc;
  a.P = P;
  a.K = k;
  char* b = static_cast<char*>(scratch);
  // two heads: each call uses the one the previous call zeroed and zeroes the other;
  // *head_state = 0 (unknown: fresh scratch, or the merge used it) -> memset head 0
  TkHead* h0 = reinterpret_cast<TkHead*>(b);
  TkHead* h1 = reinterpret_cast<TkHead*>(b + kHeadBytes);
  const bool use1 = *head_state == 2;
  a.head = use1 ? h1 : h0;
  a.next_head = use1 ? h0 : h1;
  b += 2 * kHeadBytes;
  a.compact = reinterpret_cast<u128*>(b);
  b += 16ull * kFastMax;
  a.rcap = topk_region_cap(P, max_ctas);
  a.buf = reinterpret_cast<u128*>(b);
  b += 16 * a.rcap * (uint64_t)max_ctas;
  a.kcap = pow2_ceil(m < 2 ? 2 : m);
  a.keys = reinterpret_cast<u128*>(b);
  a.out_page = out_page;
  a.out_count = out_count;
  a.out_found = out_found;
  a.pbits = P > 1 ? 64 - __builtin_clzll(P - 1) : 0;
  cudaError_t e = cudaSuccess;
  if (*head_state == 0) {
    e = cudaMemsetAsync(a.head, 0, sizeof(TkHead), st);
    if (e != cudaSuccess) return e;
  }
  constexpr int kDynSmem = 16 * kFastMax;
  static int coop_blocks = 0;  // co-resident blocks per SM for the cooperative launch
  if (coop_blocks == 0) {
    e = cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
    if (e != cudaSuccess) return e;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, topk_kernel, kTB, kDynSmem) != cudaSuccess || nb < 1) nb = 1;
    coop_blocks = nb;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int g = sms * (coop_blocks < 2 ? coop_blocks : 2);
  // no more CTAs than the counts (or the sort) give work to
#ifndef PASTA_TOPK_PER_CTA
#define PASTA_TOPK_PER_CTA (2ull * kTB * kTU)  // counts per CTA below which fewer CTAs are launched
#endif
  const uint64_t want = (P + PASTA_TOPK_PER_CTA - 1) / PASTA_TOPK_PER_CTA;
  const uint64_t want_sort = a.kcap / kSortTile;
  uint64_t w = want > want_sort ? want : want_sort;
  if (w < 1) w = 1;
  if ((uint64_t)g > w) g = (int)w;
  if (g > max_ctas) g = max_ctas;
  // the candidate buffer (sized for max_ctas regions) split over the CTAs actually
  // launched: regions of >= min(P, 2^20) / g keys, so a pass over P <= 2^20 counts
  // never overflows a region (a small P runs on few CTAs)
  a.rcap = topk_region_cap(P, max_ctas) * (uint64_t)max_ctas / (uint64_t)g;
  void* args[] = {(void*)&a};
  PASTA_TRY(cudaLaunchCooperativeKernel((void*)topk_kernel, dim3(g), dim3(kTB), args, kDynSmem, st));
  *head_state = use1 ? 1 : 2;  // the head zeroed by this launch is the next call's
  return cudaSuccess;
}

cudaError_t launch_topk_prefix(const TopkPrefixTable& t, int grid, cudaStream_t st) {
  uint64_t most = 0;
  for (uint32_t j = 0; j < t.count; ++j) most = t.e[j].k > most ? t.e[j].k : most;
  uint64_t g = (most + 255) / 256;
  if (g < 1) g = 1;
  if (g > (uint64_t)grid) g = (uint64_t)grid;
  topk_prefix_kernel<<<(unsigned)g, 256, 0, st>>>(t);
  return cudaGetLastError();
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
