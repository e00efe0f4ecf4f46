// scan.cu -- the fused trace scan: S1 range lookup + S2 histograms + S3 per-kernel
// page bits in ONE pass over the records.
//
// Paper: "the profiling library records the instruction into a device buffer. A
// helper device function then processes many of these events concurrently"
// (P:322-323); "a profiling device function increments access count for each
// associated memory object upon each access". The paper's lookup / counting
// method is unstated; this is our sm_100a design:
//
//  * persistent grid, one CTA per SM; each CTA owns a contiguous run of 32 KiB
//    chunks; one producer warp streams them global -> shared with 1-D TMA bulk copies
//    (cp.async.bulk + mbarrier complete_tx, L2 evict_first) into a 4-stage ring;
//  * 16 consumer warps; warp w takes the 256-record slice [256w, 256w+256) of each
//    chunk with four conflict-free LDS.128 per lane (lane l holds slice positions
//    64i + 2l + {0,1}, i = 0..3, in position order);
//  * every address resolves to exactly one *interval* = (live range or gap between
//    ranges) intersected with (page or out-of-window region); the owner part comes
//    from a binary search over the sorted boundary array B = [base_0, end_0, ...]
//    in shared memory (count c of boundaries <= a: odd => range (c-1)/2, even =>
//    gap), cached per lane; the page part is arithmetic;
//  * tier W (warp-uniform): A = interval of the slice's first record, B = interval
//    of its last; if A == B or B starts right after A, and every lane's 8 records are
//    non-decreasing with a_0 >= A.lo and a_7 <= B.last, then every record is in
//    A u B and the A-count is #{a <= A.last}: one __reduce_add_sync per slice;
//  * tier L (per lane): A = interval of the lane's first record, B = interval of its
//    first record outside A, membership counts; the (page, owner, count) pairs of
//    the warp are merged by a leader loop (ballot / shfl / __reduce_add_sync);
//  * tier F (per lane, rare): records in neither A nor B are looked up one by one;
//  * counts accumulate in warp-uniform registers (current page, current owner) and
//    are flushed by one lane with red.global.add.u64 when the page / owner changes,
//    at kernel-segment boundaries (per warp, no CTA barrier) and at the end; the
//    per-kernel page bit is set with atom.or at the page flush.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace pasta {
namespace {

using namespace dev;

constexpr int kConsWarps = 16;
constexpr int kCons = kConsWarps * 32;  // consumer threads
constexpr int kThreads = kCons + 32;    // + one producer warp
constexpr int kSlice = 256;             // records per warp per chunk (8 per lane)
constexpr int kChunk = kConsWarps * kSlice;  // 4096 records = 32 KiB
constexpr int kStages = 4;
constexpr uint32_t kChunkBytes = kChunk * 8;
constexpr int kRingBytes = kStages * kChunkBytes;
constexpr int kMiscBytes = 2 * kStages * 8 + 16;
constexpr int kSmemLimit = 227 * 1024;

struct Ctx {
  uint64_t va_lo, va_hi, wbytes;  // window, wbytes = va_hi - va_lo
  uint32_t s;
  uint32_t A;
  const uint64_t* B;  // boundary array (shared or global)
};

struct Ival {           // one interval: [lo, lo + span]
  uint64_t lo, span;
  uint32_t page;        // page index or kOOW
  uint32_t own;         // live-range index, A = unattributed
};

struct OwnCache {       // last owner interval (range or gap) seen by this lane
  uint64_t olo, ospan;
  uint32_t own;
};

__device__ __forceinline__ bool inside(uint64_t a, const Ival& I) { return a - I.lo <= I.span; }

// #{ i < m : B[i] <= a } by bisection.
template <bool kGlobal>
__device__ __forceinline__ uint32_t count_le(const uint64_t* __restrict__ B, uint32_t m, uint64_t a) {
  uint32_t lo = 0, len = m;
  while (len > 0) {
    const uint32_t half = len >> 1;
    const uint64_t v = kGlobal ? __ldg(B + lo + half) : B[lo + half];
    if (v <= a) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return lo;
}

template <bool kBig>
__device__ __forceinline__ Ival lookup(OwnCache& oc, uint64_t a, const Ctx& c) {
  if (a - oc.olo > oc.ospan) {
    const uint32_t m = 2 * c.A;
    const uint32_t cc = count_le<kBig>(c.B, m, a);
    const uint64_t olo = cc ? (kBig ? __ldg(c.B + cc - 1) : c.B[cc - 1]) : 0ull;
    const uint64_t olast = (cc == m) ? ~0ull : (kBig ? __ldg(c.B + cc) : c.B[cc]) - 1;
    oc.olo = olo;
    oc.ospan = olast - olo;
    oc.own = (cc & 1u) ? (cc >> 1) : c.A;
  }
  uint64_t plo, plast;
  uint32_t page;
  const uint64_t d = a - c.va_lo;
  if (d < c.wbytes) {
    const uint64_t p = d >> c.s;
    page = static_cast<uint32_t>(p);
    plo = c.va_lo + (p << c.s);
    plast = plo + ((1ull << c.s) - 1);
  } else if (a < c.va_lo) {
    plo = 0;
    plast = c.va_lo - 1;
    page = kOOW;
  } else {
    plo = c.va_hi;
    plast = ~0ull;
    page = kOOW;
  }
  const uint64_t olast = oc.olo + oc.ospan;
  Ival I;
  I.lo = oc.olo > plo ? oc.olo : plo;
  const uint64_t last = olast < plast ? olast : plast;
  I.span = last - I.lo;
  I.page = page;
  I.own = oc.own;
  return I;
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
  uint32_t A;
};

// Owner count `v` of kernel k to global (one thread).
template <bool kRows>
__device__ __forceinline__ void owner_to_global(const Out& o, uint32_t own, uint64_t v, uint32_t k) {
  if (v == 0) return;
  if (own < o.A) {
    const uint32_t id = __ldg(o.ids + own);
    red_add_u64(o.alloc_counts + id, v);
    if (kRows) {
      red_add_u64(o.kac + (uint64_t)k * o.max_ids + id, v);
      if (o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 0, v);
    }
  } else {
    red_add_u64(o.totals + 1, v);
    if (kRows && o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 1, v);
  }
}

// Page count `v` of kernel k to global (one thread).
template <bool kPages>
__device__ __forceinline__ void page_to_global(const Out& o, uint32_t page, uint64_t v, uint32_t k) {
  if (v == 0) return;
  if (page == kOOW) {
    red_add_u64(o.totals + 2, v);
  } else {
    red_add_u64(o.page_counts + page, v);
    if (kPages) red_or_u64(o.kpb + (uint64_t)k * o.words + (page >> 6), 1ull << (page & 63));
  }
}

// Warp-uniform accumulators (every lane holds the same values).
struct WarpAcc {
  uint32_t page, own;
  uint32_t pcnt, ocnt;
};

template <bool kRows, bool kPages>
__device__ __forceinline__ void wadd(WarpAcc& w, const Out& o, uint32_t page, uint32_t own, uint32_t c, uint32_t k,
                                     uint32_t lane) {
  if (page != w.page) {
    if (lane == 0) page_to_global<kPages>(o, w.page, w.pcnt, k);
    w.page = page;
    w.pcnt = 0;
  }
  w.pcnt += c;
  if (own != w.own) {
    if (lane == 0) owner_to_global<kRows>(o, w.own, w.ocnt, k);
    w.own = own;
    w.ocnt = 0;
  }
  w.ocnt += c;
}

// Per-lane fallback accumulators (tier F).
struct LaneAcc {
  uint32_t own, ocnt;
  uint32_t kbit;  // last page whose kernel bit this lane set
};

// Tier F: one record, looked up alone; page count straight to L2, owner accumulated.
template <bool kBig, bool kRows, bool kPages>
__device__ __forceinline__ void fallback_record(uint64_t x, OwnCache& oc, LaneAcc& la, const Ctx& c, const Out& o,
                                             uint32_t k) {
  const Ival I = lookup<kBig>(oc, x, c);
  if (I.page == kOOW) {
    red_add_u64(o.totals + 2, 1);
  } else {
    red_add_u64(o.page_counts + I.page, 1);
    if (kPages && la.kbit != I.page) {
      red_or_u64(o.kpb + (uint64_t)k * o.words + (I.page >> 6), 1ull << (I.page & 63));
      la.kbit = I.page;
    }
  }
  if (I.own != la.own) {
    owner_to_global<kRows>(o, la.own, la.ocnt, k);
    la.own = I.own;
    la.ocnt = 0;
  }
  la.ocnt += 1;
}

// Warp-collective: merge every lane's up to two (page, owner, count) entries into the
// warp accumulators (leader loop; one __reduce_add_sync per distinct key).
template <bool kRows, bool kPages>
__device__ __forceinline__ void merge_entries(WarpAcc& w, const Out& o, uint32_t k, uint32_t lane, bool pa,
                                              uint32_t pA, uint32_t oA, uint32_t cA, bool pb, uint32_t pB,
                                              uint32_t oB, uint32_t cB) {
  for (;;) {
    const unsigned m = __ballot_sync(kFull, pa || pb);
    if (m == 0) break;
    const int leader = __ffs(m) - 1;
    const uint32_t kp = __shfl_sync(kFull, pa ? pA : pB, leader);
    const uint32_t ko = __shfl_sync(kFull, pa ? oA : oB, leader);
    const bool mA = pa && pA == kp && oA == ko;
    const bool mB = pb && pB == kp && oB == ko;
    const uint32_t sum = __reduce_add_sync(kFull, (mA ? cA : 0u) + (mB ? cB : 0u));
    wadd<kRows, kPages>(w, o, kp, ko, sum, k, lane);
    pa = pa && !mA;
    pb = pb && !mB;
  }
}

// Tier L + F for this lane's records selected by `valid` (bit i <-> a[i]).
template <bool kBig, bool kRows, bool kPages>
__device__ __forceinline__ void process_lane(const uint64_t (&a)[8], uint32_t valid, OwnCache& oc, LaneAcc& la,
                                             WarpAcc& w, const Ctx& c, const Out& o, uint32_t k, uint32_t lane) {
  // seed A: first valid record
  uint64_t x = a[7];
#pragma unroll
  for (int i = 6; i >= 0; --i)
    if ((valid >> i) & 1u) x = a[i];
  Ival IA{};
  uint32_t cA = 0, inA = 0;
  if (valid) {
    IA = lookup<kBig>(oc, x, c);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (((valid >> i) & 1u) && inside(a[i], IA)) inA |= 1u << i;
    cA = __popc(inA);
  }
  uint32_t miss = valid & ~inA;
  Ival IB{};
  uint32_t cB = 0;
  if (__any_sync(kFull, miss != 0)) {
    if (miss) {
      uint64_t y = a[7];
#pragma unroll
      for (int i = 6; i >= 0; --i)
        if ((miss >> i) & 1u) y = a[i];
      IB = lookup<kBig>(oc, y, c);
      uint32_t inB = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (((miss >> i) & 1u) && inside(a[i], IB)) inB |= 1u << i;
      cB = __popc(inB);
      miss &= ~inB;
    }
    if (__any_sync(kFull, miss != 0)) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if ((miss >> i) & 1u) fallback_record<kBig, kRows, kPages>(a[i], oc, la, c, o, k);
    }
  }
  merge_entries<kRows, kPages>(w, o, k, lane, cA > 0, IA.page, IA.own, cA, cB > 0, IB.page, IB.own, cB);
}

// Full 256-record slice: tier W, else tier L/F.
template <bool kBig, bool kRows, bool kPages>
__device__ __forceinline__ void process_full(const uint64_t (&a)[8], OwnCache& oc, LaneAcc& la, WarpAcc& w,
                                             const Ctx& c, const Out& o, uint32_t k, uint32_t lane) {
  const uint64_t xf = __shfl_sync(kFull, a[0], 0);
  const uint64_t xl = __shfl_sync(kFull, a[7], 31);
  const Ival IA = lookup<kBig>(oc, xf, c);
  const bool same = inside(xl, IA);
  Ival IB = IA;
  if (!same) IB = lookup<kBig>(oc, xl, c);
  const uint64_t alast = IA.lo + IA.span;
  const bool ok = same || (IB.lo - 1 == alast);
  bool lane_ok = ok && a[0] >= IA.lo && a[7] <= IB.lo + IB.span;
#pragma unroll
  for (int i = 0; i < 7; ++i) lane_ok = lane_ok && (a[i] <= a[i + 1]);
  if (__all_sync(kFull, lane_ok)) {
    if (same) {
      wadd<kRows, kPages>(w, o, IA.page, IA.own, kSlice, k, lane);
    } else {
      uint32_t cA = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) cA += (a[i] <= alast) ? 1u : 0u;
      const uint32_t sA = __reduce_add_sync(kFull, cA);
      wadd<kRows, kPages>(w, o, IA.page, IA.own, sA, k, lane);
      wadd<kRows, kPages>(w, o, IB.page, IB.own, kSlice - sA, k, lane);
    }
    return;
  }
  process_lane<kBig, kRows, kPages>(a, 0xFFu, oc, la, w, c, o, k, lane);
}

// Warp-local flush of everything accumulated for kernel segment k.
template <bool kRows, bool kPages>
__device__ __forceinline__ void warp_flush(WarpAcc& w, LaneAcc& la, const Out& o, uint32_t k, uint32_t lane) {
  if (lane == 0) {
    page_to_global<kPages>(o, w.page, w.pcnt, k);
    owner_to_global<kRows>(o, w.own, w.ocnt, k);
  }
  w.pcnt = 0;
  w.ocnt = 0;
  w.page = kOOW - 1;  // no page: forces the next wadd to (re)set the kernel bit
  // lane fallback owner counts: warp-aggregate by owner
  bool pend = la.ocnt > 0;
  for (;;) {
    const unsigned m = __ballot_sync(kFull, pend);
    if (m == 0) break;
    const int leader = __ffs(m) - 1;
    const uint32_t key = __shfl_sync(kFull, la.own, leader);
    const bool mine = pend && la.own == key;
    const uint32_t sum = __reduce_add_sync(kFull, mine ? la.ocnt : 0u);
    if (lane == (uint32_t)leader) owner_to_global<kRows>(o, key, sum, k);
    pend = pend && !mine;
  }
  la.ocnt = 0;
  la.kbit = kOOW;
}

__device__ __forceinline__ uint32_t kernel_of(const uint64_t* __restrict__ koffs, uint32_t K, uint64_t g) {
  // largest k in [0, K-1] with koffs[k] <= g
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
  uint64_t* sB = reinterpret_cast<uint64_t*>(smem + kRingBytes + kMiscBytes);

  const uint32_t A = args.A;
  const uint64_t nchunks = (args.nbody + kChunk - 1) / kChunk;
  const uint64_t c0 = (uint64_t)blockIdx.x * nchunks / gridDim.x;
  const uint64_t c1 = (uint64_t)(blockIdx.x + 1) * nchunks / gridDim.x;
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsWarps);
    }
    fence_mbar_init();
    if (blockIdx.x == 0 && args.add_records) red_add_u64(args.totals + 0, args.add_records);
  }
  if (!kBig)
    for (uint32_t i = threadIdx.x; i < 2 * A; i += kThreads) sB[i] = args.bounds[i];
  __syncthreads();

  if (warp == kConsWarps) {
    // ---------------- producer warp: TMA bulk copies into the ring ----------------
    if (lane == 0) {
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
  c.wbytes = args.va_hi - args.va_lo;
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
  o.A = A;

  OwnCache oc;
  oc.olo = 1;
  oc.ospan = 0;  // forces a search on the first lookup
  oc.own = A;
  WarpAcc w;
  w.page = kOOW - 1;
  w.own = A;
  w.pcnt = 0;
  w.ocnt = 0;
  LaneAcc la;
  la.own = A;
  la.ocnt = 0;
  la.kbit = kOOW;

  const uint32_t K = args.n_kernels;
  uint32_t k = 0;
  uint64_t kend = ~0ull;
  if (kRows && K > 1 && c0 < c1) {
    k = kernel_of(args.koffs, K, args.gidx0 + c0 * kChunk + (uint64_t)warp * kSlice);
    kend = (k + 1 < K) ? __ldg(args.koffs + k + 1) : ~0ull;
  }

  uint32_t it = 0;
  for (uint64_t ch = c0; ch < c1; ++ch, ++it) {
    const uint32_t st = it % kStages;
    mbar_wait(full + st, (it / kStages) & 1u);
    const ulonglong2* src =
        reinterpret_cast<const ulonglong2*>(ring + (size_t)st * kChunk + (size_t)warp * kSlice) + lane;
    uint64_t a[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const ulonglong2 v = src[32 * i];
      a[2 * i] = v.x;
      a[2 * i + 1] = v.y;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);

    const uint64_t remc = args.nbody - ch * kChunk;
    const uint32_t valid = (uint32_t)(remc < (uint64_t)kChunk ? remc : (uint64_t)kChunk);
    const uint32_t wbase = (uint32_t)warp * kSlice;
    if (valid <= wbase) continue;
    const uint32_t wvalid = (valid - wbase) < (uint32_t)kSlice ? (valid - wbase) : (uint32_t)kSlice;
    const uint64_t gw = args.gidx0 + ch * kChunk + wbase;
    uint32_t r0 = 0;
    for (;;) {
      if (kRows && gw + r0 >= kend) {
        warp_flush<kRows, kPages>(w, la, o, k, lane);
        while (k + 1 < K && __ldg(args.koffs + k + 1) <= gw + r0) ++k;
        kend = (k + 1 < K) ? __ldg(args.koffs + k + 1) : ~0ull;
      }
      uint32_t r1 = wvalid;
      if (kRows && kend - gw < (uint64_t)r1) r1 = (uint32_t)(kend - gw);
      if (r0 == 0 && r1 == (uint32_t)kSlice) {
        process_full<kBig, kRows, kPages>(a, oc, la, w, c, o, k, lane);
      } else {
        // positions of a[2i+h] in the slice: 64i + 2*lane + h
        uint32_t vm = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t pos = 64u * (i >> 1) + 2u * lane + (i & 1);
          if (pos >= r0 && pos < r1) vm |= 1u << i;
        }
        process_lane<kBig, kRows, kPages>(a, vm, oc, la, w, c, o, k, lane);
      }
      r0 = r1;
      if (r0 >= wvalid) break;
    }
  }
  warp_flush<kRows, kPages>(w, la, o, k, lane);
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
  c.wbytes = s.va_hi - s.va_lo;
  c.s = s.page_shift;
  c.A = s.A;
  c.B = s.bounds;
  OwnCache oc;
  oc.olo = 1;
  oc.ospan = 0;
  oc.own = s.A;
  const Ival I = lookup<true>(oc, a, c);
  Out o{};
  o.page_counts = s.page_counts;
  o.alloc_counts = s.alloc_counts;
  o.totals = s.totals;
  o.kac = s.kac;
  o.kstats = s.kstats;
  o.kpb = s.kpb;
  o.ids = s.ids;
  o.max_ids = s.max_ids;
  o.words = s.words;
  o.A = s.A;
  if (rows) owner_to_global<true>(o, I.own, 1, k);
  else owner_to_global<false>(o, I.own, 1, k);
  if (s.kpb) page_to_global<true>(o, I.page, 1, k);
  else page_to_global<false>(o, I.page, 1, k);
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
  return (size_t)kRingBytes + kMiscBytes + 16ull * A + 64 <= (size_t)kSmemLimit;
}

int scan_smem_bytes(uint32_t A, bool big_table) {
  if (big_table) return kRingBytes + kMiscBytes;
  return (int)(kRingBytes + kMiscBytes + 16ull * A);
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

}  // namespace pasta
