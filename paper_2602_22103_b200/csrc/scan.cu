// scan.cu -- the fused trace scan: S1 range lookup + S2 histograms + S3 per-kernel
// page bits in ONE pass over the records.
//
// Paper: "the profiling library records the instruction into a device buffer. A
// helper device function then processes many of these events concurrently"
// (P:322-323); "a profiling device function increments access count for each
// associated memory object upon each access". The paper's lookup / counting
// method is unstated; this is our sm_100a design:
//
//  * persistent grid, one CTA per SM, each CTA owns a contiguous run of 32 KiB
//    chunks; one producer warp streams chunks global -> shared with 1-D TMA bulk
//    copies (cp.async.bulk + mbarrier complete_tx, L2 evict_first) into a 4-stage
//    ring; 16 consumer warps read their records with conflict-free LDS.128;
//  * each consumer lane owns RPT consecutive records and keeps a *run*: the
//    interval [lo, lo+span] = (owning range or gap) intersected with (page or
//    out-of-window region) plus a count. A record inside the run costs one 64-bit
//    subtract-compare; a warp whose lanes all stay in their runs takes one vote;
//  * on a miss the lane flushes its run (warp-aggregated: __match_any_sync groups,
//    __reduce_add_sync sum, one leader atomic per distinct key) and looks the new
//    address up: page by shift, owner by binary search over the sorted boundary
//    array held in shared memory (count of boundaries <= a: odd => inside range
//    (c-1)/2, even => gap);
//  * owner counts go to a per-CTA shared-memory array (u32 per live range plus the
//    unattributed slot), flushed to global at kernel-segment boundaries and at the
//    end; page counts go straight to L2 with red.global.add.u64 (one per distinct
//    (warp, page) flush), per-kernel page bits with atom.or at the same flush.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace pasta {
namespace {

using namespace dev;

constexpr int kRPT = 8;                       // records per consumer lane per chunk
constexpr int kVec = kRPT / 2;                // LDS.128 per lane per chunk
constexpr int kConsWarps = 16;
constexpr int kCons = kConsWarps * 32;        // consumer threads
constexpr int kThreads = kCons + 32;          // + one producer warp
constexpr int kChunk = kCons * kRPT;          // records per chunk (4096 = 32 KiB)
constexpr int kStages = 4;
constexpr uint32_t kChunkBytes = kChunk * 8;
constexpr int kRingBytes = kStages * kChunkBytes;
constexpr int kMiscBytes = 2 * kStages * 8 + 16;
constexpr int kSmemLimit = 227 * 1024;

struct Lane {
  uint64_t lo, span;    // current run interval [lo, lo + span]
  uint64_t olo, ospan;  // owner (range or gap) interval
  uint32_t cnt;         // records in the run
  uint32_t page;        // page index or kOOW
  uint32_t own;         // live-range index, A = unattributed
  uint32_t kbit;        // last page whose kernel bit this lane set (KPAGES)
};

// #{ i < m : B[i] <= a } by bisection.
template <bool kGlobal>
__device__ __forceinline__ uint32_t count_le(const uint64_t* __restrict__ B, uint32_t m, uint64_t a) {
  uint32_t lo = 0, len = m;
  while (len > 0) {
    uint32_t half = len >> 1;
    uint64_t v = kGlobal ? __ldg(B + lo + half) : B[lo + half];
    if (v <= a) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return lo;
}

struct Ctx {
  uint64_t va_lo, va_hi;
  uint32_t s;
  uint32_t A;
  const uint64_t* B;  // boundary array (shared or global)
};

template <bool kBig>
__device__ __forceinline__ void lookup(Lane& L, uint64_t a, const Ctx& c) {
  if (a - L.olo > L.ospan) {
    const uint32_t m = 2 * c.A;
    const uint32_t cc = count_le<kBig>(c.B, m, a);
    const uint64_t olo = cc ? (kBig ? __ldg(c.B + cc - 1) : c.B[cc - 1]) : 0ull;
    const uint64_t olast = (cc == m) ? ~0ull : (kBig ? __ldg(c.B + cc) : c.B[cc]) - 1;
    L.olo = olo;
    L.ospan = olast - olo;
    L.own = (cc & 1u) ? (cc >> 1) : c.A;
  }
  uint64_t plo, plast;
  if (a < c.va_lo) {
    plo = 0;
    plast = c.va_lo - 1;
    L.page = kOOW;
  } else if (a >= c.va_hi) {
    plo = c.va_hi;
    plast = ~0ull;
    L.page = kOOW;
  } else {
    const uint64_t p = (a - c.va_lo) >> c.s;
    L.page = static_cast<uint32_t>(p);
    plo = c.va_lo + (p << c.s);
    plast = plo + ((1ull << c.s) - 1);
  }
  const uint64_t olast = L.olo + L.ospan;
  const uint64_t lo = L.olo > plo ? L.olo : plo;
  const uint64_t last = olast < plast ? olast : plast;
  L.lo = lo;
  L.span = last - lo;
}

struct Out {
  uint64_t* page_counts;
  uint64_t* alloc_counts;
  uint64_t* totals;
  uint64_t* kac;
  uint64_t* kstats;
  uint64_t* kpb;
  const uint32_t* ids;
  uint64_t max_ids;
  uint32_t words;
  uint32_t* own_cnt;  // shared (A+1 slots) unless kBig
  uint32_t* oow;      // shared
};

// Owner count of `s` records straight to global (kBig path and the extras kernel).
template <bool kRows>
__device__ __forceinline__ void owner_to_global(const Out& o, uint32_t own, uint32_t A, uint64_t s, uint32_t k) {
  if (own < A) {
    const uint32_t id = __ldg(o.ids + own);
    red_add_u64(o.alloc_counts + id, s);
    if (kRows) {
      red_add_u64(o.kac + (uint64_t)k * o.max_ids + id, s);
      if (o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 0, s);
    }
  } else {
    red_add_u64(o.totals + 1, s);
    if (kRows && o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 1, s);
  }
}

// Warp-collective: lanes with `pred` flush their run. Called by all 32 lanes.
template <bool kBig, bool kRows, bool kPages>
__device__ __forceinline__ void flush_runs(bool pred, Lane& L, const Out& o, uint32_t A, uint32_t k) {
  const unsigned m = __ballot_sync(kFull, pred);
  if (m == 0) return;
  if (pred) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned g1 = __match_any_sync(m, L.own);
    const uint32_t s1 = __reduce_add_sync(g1, L.cnt);
    if (lane == (unsigned)(__ffs(g1) - 1)) {
      if (kBig) owner_to_global<kRows>(o, L.own, A, s1, k);
      else atomicAdd(o.own_cnt + L.own, s1);
    }
    const unsigned g2 = __match_any_sync(m, L.page);
    const uint32_t s2 = __reduce_add_sync(g2, L.cnt);
    if (lane == (unsigned)(__ffs(g2) - 1)) {
      if (L.page == kOOW) {
        atomicAdd(o.oow, s2);
      } else {
        red_add_u64(o.page_counts + L.page, s2);
        if (kPages && L.kbit != L.page)
          red_or_u64(o.kpb + (uint64_t)k * o.words + (L.page >> 6), 1ull << (L.page & 63));
      }
    }
    if (kPages) L.kbit = L.page;
  }
}

// CTA-collective (consumer threads): flush every lane's run, then the shared owner
// counts of kernel segment k.
template <bool kBig, bool kRows, bool kPages>
__device__ void segment_flush(Lane& L, const Out& o, uint32_t A, uint32_t k) {
  flush_runs<kBig, kRows, kPages>(L.cnt > 0, L, o, A, k);
  L.cnt = 0;
  if (kPages) L.kbit = kOOW;
  named_bar_sync(1, kCons);
  uint64_t attributed = 0;
  if (!kBig) {
    for (uint32_t r = threadIdx.x; r <= A; r += kCons) {
      const uint32_t v = o.own_cnt[r];
      if (v == 0) continue;
      o.own_cnt[r] = 0;
      if (r < A) {
        const uint32_t id = __ldg(o.ids + r);
        red_add_u64(o.alloc_counts + id, v);
        if (kRows) red_add_u64(o.kac + (uint64_t)k * o.max_ids + id, v);
        attributed += v;
      } else {
        red_add_u64(o.totals + 1, v);
        if (kRows && o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 1, v);
      }
    }
    if (kRows && o.kstats) {
      attributed = warp_sum_u64(attributed);
      if ((threadIdx.x & 31) == 0 && attributed) red_add_u64(o.kstats + (uint64_t)k * 4 + 0, attributed);
    }
  }
  if (threadIdx.x == 0) {
    const uint32_t v = *o.oow;
    if (v) {
      *o.oow = 0;
      red_add_u64(o.totals + 2, v);
    }
  }
  named_bar_sync(1, kCons);
}

// Process this lane's records of the current chunk whose chunk positions lie in
// [r0, r1). a[2i], a[2i+1] are the records at positions base + 2*rot(i) (+1).
template <bool kMasked, bool kBig, bool kRows, bool kPages>
__device__ __forceinline__ void process(const uint64_t (&a)[kRPT], uint32_t base, uint32_t rsh, uint32_t r0,
                                        uint32_t r1, Lane& L, const Ctx& c, const Out& o, uint32_t k) {
  uint32_t need = 0, hits = 0;
#pragma unroll
  for (int i = 0; i < kVec; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      bool v = true;
      if (kMasked) {
        const uint32_t pos = base + 2 * ((i + rsh) % kVec) + h;
        v = pos >= r0 && pos < r1;
      }
      const bool hit = (a[2 * i + h] - L.lo) <= L.span;
      need += v;
      hits += (v && hit);
    }
  }
  if (__all_sync(kFull, hits == need)) {
    L.cnt += need;
    return;
  }
#pragma unroll
  for (int i = 0; i < kVec; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      bool v = true;
      if (kMasked) {
        const uint32_t pos = base + 2 * ((i + rsh) % kVec) + h;
        v = pos >= r0 && pos < r1;
      }
      const uint64_t x = a[2 * i + h];
      const bool miss = v && ((x - L.lo) > L.span);
      if (__any_sync(kFull, miss)) {
        flush_runs<kBig, kRows, kPages>(miss && L.cnt > 0, L, o, c.A, k);
        if (miss) {
          lookup<kBig>(L, x, c);
          L.cnt = 0;
        }
      }
      L.cnt += v;
    }
  }
}

__device__ __forceinline__ uint32_t kernel_of(const uint64_t* __restrict__ koffs, uint32_t K, uint64_t g) {
  // largest k with koffs[k] <= g among k in [0, K-1]
  uint32_t lo = 0, hi = K - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (__ldg(koffs + mid) <= g) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <bool kBig, bool kRows, bool kPages>
__global__ void __launch_bounds__(kThreads, 1) scan_kernel(const ScanArgs args) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* ring = reinterpret_cast<uint64_t*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes);
  uint64_t* empty = full + kStages;
  uint32_t* oow = reinterpret_cast<uint32_t*>(empty + kStages);
  uint64_t* sB = reinterpret_cast<uint64_t*>(smem + kRingBytes + kMiscBytes);
  uint32_t* own_cnt = reinterpret_cast<uint32_t*>(sB + 2 * (size_t)args.A);

  const uint32_t A = args.A;
  const uint64_t nchunks = (args.nbody + kChunk - 1) / kChunk;
  const uint64_t c0 = (uint64_t)blockIdx.x * nchunks / gridDim.x;
  const uint64_t c1 = (uint64_t)(blockIdx.x + 1) * nchunks / gridDim.x;
  const int warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsWarps);
    }
    *oow = 0;
    fence_mbar_init();
    if (blockIdx.x == 0 && args.add_records) red_add_u64(args.totals + 0, args.add_records);
  }
  if (!kBig) {
    for (uint32_t i = threadIdx.x; i < 2 * A; i += kThreads) sB[i] = args.bounds[i];
    for (uint32_t i = threadIdx.x; i <= A; i += kThreads) own_cnt[i] = 0;
  }
  __syncthreads();

  if (warp == kConsWarps) {
    // ---------------- producer warp: TMA bulk copies into the ring ----------------
    if ((threadIdx.x & 31) == 0) {
      const uint64_t pol = l2_evict_first_policy();
      uint32_t it = 0;
      for (uint64_t ch = c0; ch < c1; ++ch, ++it) {
        const uint32_t st = it % kStages;
        if (it >= kStages) mbar_wait(empty + st, ((it / kStages) & 1u) ^ 1u);
        const uint64_t rem = args.nbody - ch * kChunk;
        const uint32_t bytes = (uint32_t)((rem < (uint64_t)kChunk ? rem : (uint64_t)kChunk) * 8);
        mbar_arrive_expect_tx(full + st, bytes);
        tma_load_1d(ring + (size_t)st * kChunk, args.rec + ch * kChunk, bytes, full + st, pol);
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  Ctx c;
  c.va_lo = args.va_lo;
  c.va_hi = args.va_hi;
  c.s = args.page_shift;
  c.A = A;
  c.B = kBig ? args.bounds : sB;
  Out o;
  o.page_counts = args.page_counts;
  o.alloc_counts = args.alloc_counts;
  o.totals = args.totals;
  o.kac = args.kac;
  o.kstats = args.kstats;
  o.kpb = args.kpb;
  o.ids = args.ids;
  o.max_ids = args.max_ids;
  o.words = args.words;
  o.own_cnt = own_cnt;
  o.oow = oow;

  Lane L;
  L.olo = 1;
  L.ospan = 0;  // forces a search on the first lookup
  L.cnt = 0;
  L.kbit = kOOW;
  lookup<kBig>(L, 0ull, c);

  const uint32_t K = args.n_kernels;
  uint32_t k = 0;
  uint64_t kend = ~0ull;
  if (kRows && K > 1 && c0 < c1) {
    k = kernel_of(args.koffs, K, args.gidx0 + c0 * kChunk);
    kend = (k + 1 < K) ? __ldg(args.koffs + k + 1) : ~0ull;
  }

  const uint32_t lane = threadIdx.x & 31;
  const uint32_t base = threadIdx.x * kRPT;         // chunk position of my first record
  const uint32_t rsh = lane / (8 / kVec);           // LDS.128 rotation (bank-conflict free)

  uint32_t it = 0;
  for (uint64_t ch = c0; ch < c1; ++ch, ++it) {
    const uint32_t st = it % kStages;
    mbar_wait(full + st, (it / kStages) & 1u);
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(ring + (size_t)st * kChunk + base);
    uint64_t a[kRPT];
#pragma unroll
    for (int i = 0; i < kVec; ++i) {
      const ulonglong2 v = src[(i + rsh) % kVec];
      a[2 * i] = v.x;
      a[2 * i + 1] = v.y;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);

    const uint64_t g0 = args.gidx0 + ch * kChunk;
    const uint64_t remc = args.nbody - ch * kChunk;
    const uint32_t valid = (uint32_t)(remc < (uint64_t)kChunk ? remc : (uint64_t)kChunk);
    uint32_t r0 = 0;
    for (;;) {
      if (kRows && g0 + r0 >= kend) {
        segment_flush<kBig, kRows, kPages>(L, o, A, k);
        while (k + 1 < K && __ldg(args.koffs + k + 1) <= g0 + r0) ++k;
        kend = (k + 1 < K) ? __ldg(args.koffs + k + 1) : ~0ull;
      }
      uint32_t r1 = valid;
      if (kRows && kend - g0 < (uint64_t)r1) r1 = (uint32_t)(kend - g0);
      if (r0 == 0 && r1 == (uint32_t)kChunk)
        process<false, kBig, kRows, kPages>(a, base, rsh, r0, r1, L, c, o, k);
      else
        process<true, kBig, kRows, kPages>(a, base, rsh, r0, r1, L, c, o, k);
      r0 = r1;
      if (r0 >= valid) break;
    }
  }
  segment_flush<kBig, kRows, kPages>(L, o, A, k);
}

// The <= 2 records outside the aligned even body (unaligned head, odd tail): one
// warp, direct global atomics, same definitions.
__global__ void scan_extras_kernel(const ExtraArgs ea) {
  const ScanArgs& s = ea.s;
  const int lane = threadIdx.x;
  if (lane == 0 && s.add_records) red_add_u64(s.totals + 0, s.add_records);
  if (lane >= ea.n_ex) return;
  const uint64_t a = *ea.ex_ptr[lane];
  const uint64_t g = ea.ex_gidx[lane];
  uint32_t k = 0;
  const bool rows = s.kac != nullptr;
  if (rows && s.n_kernels > 1) k = kernel_of(s.koffs, s.n_kernels, g);
  Ctx c;
  c.va_lo = s.va_lo;
  c.va_hi = s.va_hi;
  c.s = s.page_shift;
  c.A = s.A;
  c.B = s.bounds;
  Lane L;
  L.olo = 1;
  L.ospan = 0;
  lookup<true>(L, a, c);
  Out o{};
  o.alloc_counts = s.alloc_counts;
  o.totals = s.totals;
  o.kac = s.kac;
  o.kstats = s.kstats;
  o.ids = s.ids;
  o.max_ids = s.max_ids;
  if (rows) owner_to_global<true>(o, L.own, s.A, 1, k);
  else owner_to_global<false>(o, L.own, s.A, 1, k);
  if (L.page == kOOW) {
    red_add_u64(s.totals + 2, 1);
  } else {
    red_add_u64(s.page_counts + L.page, 1);
    if (s.kpb) red_or_u64(s.kpb + (uint64_t)k * s.words + (L.page >> 6), 1ull << (L.page & 63));
  }
}

template <bool kBig, bool kRows, bool kPages>
cudaError_t launch_variant(const ScanArgs& a, int grid, cudaStream_t st) {
  const int smem = scan_smem_bytes(a.A, kBig);
  auto fn = scan_kernel<kBig, kRows, kPages>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool scan_table_fits_smem(uint32_t A) {
  return (size_t)kRingBytes + kMiscBytes + 16ull * A + 4ull * (A + 1) + 64 <= (size_t)kSmemLimit;
}

int scan_smem_bytes(uint32_t A, bool big_table) {
  if (big_table) return kRingBytes + kMiscBytes;
  return (int)(kRingBytes + kMiscBytes + 16ull * A + 4ull * (A + 1));
}

cudaError_t launch_scan(const ScanArgs& a, int grid, cudaStream_t st) {
  const bool big = !scan_table_fits_smem(a.A);
  const bool rows = a.kac != nullptr;
  const bool pages = a.kpb != nullptr;
  if (big) {
    if (!rows) return launch_variant<true, false, false>(a, grid, st);
    if (!pages) return launch_variant<true, true, false>(a, grid, st);
    return launch_variant<true, true, true>(a, grid, st);
  }
  if (!rows) return launch_variant<false, false, false>(a, grid, st);
  if (!pages) return launch_variant<false, true, false>(a, grid, st);
  return launch_variant<false, true, true>(a, grid, st);
}

cudaError_t launch_scan_extras(const ExtraArgs& a, cudaStream_t st) {
  scan_extras_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}

int scan_chunk_records() { return kChunk; }

}  // namespace pasta
