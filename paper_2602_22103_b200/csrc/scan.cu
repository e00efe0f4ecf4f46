// scan.cu -- the fused trace scan: S1 range lookup + S2 histograms + S3 per-kernel
// page bits in ONE pass over the records.
//
// Paper: "the profiling library records the instruction into a device buffer. A
// helper device function then processes many of these events concurrently"
// (P:322-323); "a profiling device function increments access count for each
// associated memory object upon each access". The paper's lookup / counting
// method is unstated; this is our sm_100a design:
//
//  * persistent grid, one CTA of 16 warps per SM; the records are cut into 2 KiB
//    slices (256 records) and every warp owns a contiguous run of slices; each warp
//    runs its own TMA pipeline: lane 0 keeps S-1 slices in flight with 1-D bulk
//    copies (cp.async.bulk + mbarrier complete_tx, L2 evict_first) into the warp's
//    S-slot shared-memory ring (S = 4, or 3 for 1,545-4,616 ranges), so warps never wait
//    on each other;
//  * a slice is read with four conflict-free LDS.128 per lane (lane l holds slice
//    positions 64i + 2l + {0,1}, i = 0..3, in position order);
//  * every address resolves to exactly one *interval* = (live range or gap between
//    ranges) intersected with (page or out-of-window region); the owner part comes
//    from a binary search over the sorted boundary array B = [base_0, end_0, ...]
//    in shared memory (count c of boundaries <= a: odd => range (c-1)/2, even =>
//    gap), cached per lane; the page part is arithmetic;
//  * tier W (warp-uniform): A = interval of the slice's first record (usually the
//    warp's cached interval), B = interval of its last; if A == B or B starts right
//    after A, and every lane's 8 records are non-decreasing with a_0 >= A.lo and
//    a_7 <= B.last, then every record is in A u B and the A-count is #{a <= A.last}:
//    one __reduce_add_sync per slice;
//  * tier W2 (warp-uniform): same A and B, per-record membership (tile jumps, row
//    switches: two intervals that are not adjacent);
//  * tier L (per lane): the slice is re-read lane-contiguously (8 consecutive
//    records per lane, rotated LDS.128 order); A = interval of the lane's first
//    record, B = interval of its first record outside A, membership counts; the
//    (page, owner, count) pairs of the warp are merged by a leader loop (ballot /
//    shfl / __reduce_add_sync);
//  * tier F (per lane, rare): records in neither A nor B are looked up one by one;
//  * counts accumulate in warp-uniform registers (current page, current owner) and
//    are flushed by one lane with red.global.add.u64 when the page / owner changes,
//    at kernel-segment boundaries (per warp, no CTA barrier) and at the end; the
//    per-kernel page bit is set with atom.or at the page flush.
#include <cstdint>
#include <cstddef>
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "pasta.h"

#ifndef PASTA_TRACE_TIMING
#define PASTA_TRACE_TIMING 0
#endif
#if PASTA_TRACE_TIMING
// debug: per-warp globaltimer stamps {start, first data, 1/4, end} (ns)
__device__ unsigned long long g_warp_times[148 * 64 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
#ifndef PASTA_SWPIPE
#define PASTA_SWPIPE 0
#endif
#ifndef PASTA_TREE
#define PASTA_TREE 0
#endif
#ifndef PASTA_FLAT_FLUSH
#define PASTA_FLAT_FLUSH 0
#endif
#ifndef PASTA_WADD2
#define PASTA_WADD2 1
#endif
#ifndef PASTA_XFL_LDS
#define PASTA_XFL_LDS 1
#endif

namespace pasta {
namespace {

using namespace dev;

#ifndef PASTA_WARPS
#define PASTA_WARPS 24
#endif
constexpr int kWarps = PASTA_WARPS;
#ifndef PASTA_PDL
#define PASTA_PDL 1  // programmatic dependent launch of consecutive scans
#endif
constexpr int kThreads = kWarps * 32;
constexpr int kSlice = 256;                 // records per slice (8 per lane)
#ifndef PASTA_TIER_S
#define PASTA_TIER_S 1  // tier S (one owner, scattered pages) before tier L
#endif
#ifndef PASTA_TMA_PAIR
#define PASTA_TMA_PAIR 1  // one 4 KiB bulk copy per two slices when the ring has an even depth
#endif
#ifndef PASTA_ISSUE2
#define PASTA_ISSUE2 0  // TMA refills in pairs
#endif
#ifndef PASTA_TIER_S_BATCH
#define PASTA_TIER_S_BATCH 1  // tier S (kPages == 0): page REDs issued back to back
#endif
#ifndef PASTA_IL
#define PASTA_IL 1  // interleaved chunk schedule for long launches (0 = always contiguous)
#endif
#ifndef PASTA_IL_LOG_CHUNK
#define PASTA_IL_LOG_CHUNK 6  // log2 slices per interleaved chunk
#endif
#ifndef PASTA_IL_DYNAMIC
#define PASTA_IL_DYNAMIC 1  // interleaved schedule: chunks after the first taken from a global counter
#endif
#ifndef PASTA_BIG_SAMPLES
#define PASTA_BIG_SAMPLES 1  // global range table: every 2^sh-th boundary sampled into shared memory
#endif
#ifndef PASTA_IL_PERMUTE_BELOW
#define PASTA_IL_PERMUTE_BELOW 128  // permuted hand-out when warps take fewer chunks than this
#endif
#ifndef PASTA_IL_LOG_CHUNK_MIN
#define PASTA_IL_LOG_CHUNK_MIN 6  // smallest chunk of the automatic interleaved schedule (>= 3)
#endif
#ifndef PASTA_IL_MIN_CHUNKS
#define PASTA_IL_MIN_CHUNKS 4  // interleave only when every warp gets this many chunks (dynamic: rn50 +2.7 %)
#endif
constexpr uint32_t kSliceBytes = kSlice * 8;  // 2 KiB
constexpr int kMaxStages = 8;
constexpr int kMinStages = 3;
constexpr int kBarBytes = kWarps * kMaxStages * 8;
#ifndef PASTA_LA_SMEM
#define PASTA_LA_SMEM 1
#endif
constexpr int kLaBytes = PASTA_LA_SMEM ? kThreads * 12 : 0;  // LaneAcc per thread
constexpr int kPfBytes = kWarps * 16;                        // per-warp chunk map slot
constexpr int kSmemLimit = 227 * 1024;

__host__ __device__ constexpr int ring_bytes(int stages) { return kWarps * stages * (int)kSliceBytes; }

struct Ctx {
  uint64_t va_lo, va_hi, wbytes;  // window, wbytes = va_hi - va_lo
  uint32_t s;
  uint32_t A;
  const uint64_t* B;  // boundary array (shared or global)
  // global table only: samples S[i] = B[i << sh] (i < nS) in shared memory narrow the
  // search to 2^sh entries of B (nS = 0: plain search of B)
  const uint64_t* S = nullptr;
  uint32_t nS = 0, sh = 0;
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

// v[i] for a runtime i, as masks: a select chain on a register array lets the compiler
// turn it into an indexed local-memory load (and spill the whole array every slice).
__device__ __forceinline__ uint64_t pick4(const uint64_t (&v)[4], int i) {
  uint64_t r = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) r |= v[q] & (0ull - (uint64_t)(i == q));
  return r;
}

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
__device__ __forceinline__ void own_lookup(OwnCache& oc, uint64_t a, const Ctx& c) {
  if (a - oc.olo > oc.ospan) {
    const uint32_t m = 2 * c.A;
    uint32_t cc;
    if (kBig && c.nS) {
      // B[(j - 1) << sh] <= a < B[j << sh]: the count lies in ((j - 1) << sh, j << sh]
      const uint32_t j = count_le<false>(c.S, c.nS, a);
      if (j == 0) {
        cc = 0;
      } else {
        const uint32_t lo = (j - 1) << c.sh, hi = min(j << c.sh, m);
        cc = lo + 1 + count_le<true>(c.B + lo + 1, hi - lo - 1, a);
      }
    } else {
      cc = count_le<kBig>(c.B, m, a);
    }
    const uint64_t olo = cc ? (kBig ? __ldg(c.B + cc - 1) : c.B[cc - 1]) : 0ull;
    const uint64_t olast = (cc == m) ? ~0ull : (kBig ? __ldg(c.B + cc) : c.B[cc]) - 1;
    oc.olo = olo;
    oc.ospan = olast - olo;
    oc.own = (cc & 1u) ? (cc >> 1) : c.A;
  }
}

// The interval holding address a: its owner interval (range or gap) cut to its page
// (or to the out-of-window region below / above the window).
template <bool kBig>
__device__ __forceinline__ Ival lookup(OwnCache& oc, uint64_t a, const Ctx& c) {
  own_lookup<kBig>(oc, a, c);
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
  uint64_t* hot;    // hotness matrix [windows x P] or nullptr (NEXT f1)
  uint64_t P;
  uint32_t wk;      // kernels per hotness window
  uint64_t wk_magic;  // ceil(2^64 / wk) (wk >= 2)
  const uint32_t* tids;  // tensor level (NEXT f3) or nullptr
  uint64_t* tcounts;
  uint64_t* ktc;
  uint64_t max_tids;
  uint32_t cache;   // 1: the page-count cache (2^kCacheBits slots at dynamic smem offset 0) is on
};

// Shared-memory page-count cache (modes without per-kernel page bits / hotness, whose
// page counts do not depend on the kernel): scattered page increments of the per-lane
// tiers go to a CTA-wide open-addressing table of (page << 32 | count) u64 slots instead
// of one L2 RED each. Insert = 64-bit shared CAS on one of 4 probe slots (count added to
// the page's slot, or an empty slot claimed); when all 4 hold other pages, the first is
// evicted with one exchange and its count written back with one RED (a write-back cache:
// a (page, count) pair is only ever in the table or already added to L2, never both, and
// the exchange takes it out atomically). The CTA writes the table back at its end.
// Off by default: measured slower on every config (A/B: s_perm 12.3 ->
// 30.8 ms, llama 13.4 -> 25.6 ms with 2^12 slots): shared 64-bit CAS retries when lanes
// hit one slot and evictions when a tensor spans more pages than the table cost more
// than the one L2 RED per scattered page run they replace.
#ifndef PASTA_PCACHE_BITS
#define PASTA_PCACHE_BITS 0
#endif
#ifndef PASTA_PCACHE_F
#define PASTA_PCACHE_F 0  // tier-F records through the cache (on: +spills in the interleaved row variants)
#endif
#ifndef PASTA_PCACHE_L
#define PASTA_PCACHE_L 1  // tier-L lane entries through the cache
#endif
constexpr int kCacheBits = PASTA_PCACHE_BITS;  // 0: no cache
constexpr uint32_t kCacheSlots = kCacheBits ? (1u << kCacheBits) : 0u;
constexpr int kCacheBytes = 8 * (int)kCacheSlots;
constexpr uint32_t kCacheEmpty = 0xFFFFFFFFu;  // key of an empty slot (== kOOW, never cached)
constexpr uint64_t kCacheEmptySlot = (uint64_t)kCacheEmpty << 32;

__device__ __forceinline__ uint32_t cache_base() {
  extern __shared__ __align__(128) unsigned char smem[];
  return smem_u32(smem);
}

__device__ __forceinline__ void cache_add(const Out& o, uint32_t page, uint32_t v) {
  const uint32_t h = (page * 0x9E3779B1u) >> (kCacheBits ? 32 - kCacheBits : 0);
  const uint32_t base = cache_base();
#pragma unroll 1
  for (uint32_t i = 0; i < 4; ++i) {
    const uint32_t addr = base + 8u * ((h + i) & (kCacheSlots - 1u));
    uint64_t cur = lds64(addr);
    for (;;) {
      const uint32_t key = (uint32_t)(cur >> 32), cnt = (uint32_t)cur;
      uint64_t nv;
      if (key == page && cnt < (1u << 31)) nv = cur + v;
      else if (key == kCacheEmpty) nv = ((uint64_t)page << 32) | v;
      else break;
      const uint64_t old = atoms_cas_u64(addr, cur, nv);
      if (old == cur) return;
      cur = old;
    }
  }
  const uint64_t old = atoms_exch_u64(base + 8u * (h & (kCacheSlots - 1u)), ((uint64_t)page << 32) | v);
  if ((uint32_t)(old >> 32) != kCacheEmpty && (uint32_t)old != 0u)
    red_add_u64(o.page_counts + (uint32_t)(old >> 32), (uint32_t)old);
}

// Time-windowed hotness: the page run's count also goes to row k / wk.
// Compiled in only for the hotness variants: kPages is a mode, bit 0 = per-kernel page
// bits, bit 1 = hotness.
template <int kMode>
__device__ __forceinline__ void hot_add(const Out& o, uint32_t page, uint64_t v, uint32_t k) {
  if ((kMode & 2) && page != kOOW) {
    // window k / wk by a multiply-high: wk_magic = ceil(2^64 / wk) is exact for k, wk < 2^32
    const uint64_t w = o.wk == 1 ? (uint64_t)k : __umul64hi((uint64_t)k, o.wk_magic);
    red_add_u64(o.hot + w * o.P + page, v);
  }
}

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
  // tensor level (R18): the table intervals refine objects by tensors, so the owner
  // interval also names the tensor (or none)
  if (o.tids != nullptr) {
    const uint32_t t = own < o.A ? __ldg(o.tids + own) : kNoTensor;
    if (t != kNoTensor) {
      red_add_u64(o.tcounts + t, v);
      if (kRows && o.ktc) red_add_u64(o.ktc + (uint64_t)k * o.max_tids + t, v);
    } else {
      red_add_u64(o.totals + kTotUntensored, v);
    }
  }
}

// Page count `v` of kernel k to global (one thread).
template <int kPages>
__device__ __forceinline__ void page_to_global(const Out& o, uint32_t page, uint64_t v, uint32_t k) {
  if (v == 0) return;
  if (page == kOOW) {
    red_add_u64(o.totals + 2, v);
  } else {
    red_add_u64(o.page_counts + page, v);
    if (kPages & 1) red_or_u64(o.kpb + (uint64_t)k * o.words + (page >> 6), 1ull << (page & 63));
    hot_add<kPages>(o, page, v, k);
  }
}

// A page count from a per-lane tier: through the shared cache when the launch has one.
template <int kPages>
__device__ __forceinline__ void page_scatter(const Out& o, uint32_t page, uint64_t v, uint32_t k) {
  if (kPages == 0 && kCacheBits && o.cache != 0u && page != kOOW && v != 0 && v < (1ull << 31)) {
    cache_add(o, page, (uint32_t)v);
    return;
  }
  page_to_global<kPages>(o, page, v, k);
}

// Warp-uniform accumulators (every lane holds the same values).
struct WarpAcc {
  uint32_t page, own;
  uint32_t pcnt, ocnt;
};

template <bool kRows, int kPages>
__device__ __forceinline__ void wadd(WarpAcc& w, const Out& o, uint32_t page, uint32_t own, uint32_t c, uint32_t k,
                                     uint32_t lane) {
  if (page != w.page) {
#if PASTA_FLAT_FLUSH
    // one predicated RED (no divergent branch): out-of-window counts go to totals[2]
    uint64_t* dst = (w.page == kOOW) ? o.totals + 2 : o.page_counts + w.page;
    if (lane == 0 && w.pcnt != 0) red_add_u64(dst, w.pcnt);
    if ((kPages & 1) && lane == 0 && w.pcnt != 0 && w.page != kOOW)
      red_or_u64(o.kpb + (uint64_t)k * o.words + (w.page >> 6), 1ull << (w.page & 63));
#else
    if (lane == 0) page_to_global<kPages>(o, w.page, w.pcnt, k);
#endif
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

// One predicated RED for a finished page run (out-of-window runs go to totals[2]).
template <int kPages>
__device__ __forceinline__ void flush_page_run(const Out& o, uint32_t page, uint32_t v, uint32_t k, uint32_t lane) {
  uint64_t* dst = (page == kOOW) ? o.totals + 2 : o.page_counts + page;
  if (lane == 0) red_add_u64(dst, v);
  if ((kPages & 1) && lane == 0 && page != kOOW)
    red_or_u64(o.kpb + (uint64_t)k * o.words + (page >> 6), 1ull << (page & 63));
  if ((kPages & 2) && lane == 0) hot_add<kPages>(o, page, v, k);
}

// Accumulate sA records of interval A then sB of interval B (sB may be 0). Fast path:
// A continues the warp's current page and owner and B has the same owner, so page A
// is complete: one RED, no owner flush.
template <bool kRows, int kPages>
__device__ __forceinline__ void wadd2(WarpAcc& w, const Out& o, const Ival& IA, uint32_t sA, const Ival& IB,
                                      uint32_t sB, uint32_t k, uint32_t lane) {
#if PASTA_WADD2
  if (IA.page == w.page && IA.own == w.own && (sB == 0 || (IB.own == IA.own && IB.page != IA.page))) {
    w.ocnt += sA + sB;
    if (sB == 0) {
      w.pcnt += sA;
    } else {
      flush_page_run<kPages>(o, IA.page, w.pcnt + sA, k, lane);
      w.page = IB.page;
      w.pcnt = sB;
    }
    return;
  }
#endif
  wadd<kRows, kPages>(w, o, IA.page, IA.own, sA, k, lane);
  if (sB) wadd<kRows, kPages>(w, o, IB.page, IB.own, sB, k, lane);
}

// Per-lane fallback accumulators (tier F).
struct LaneAcc {
  uint32_t own, ocnt;
  uint32_t kbit;  // last page whose kernel bit this lane set
};

// Tier F: one record, looked up alone; page count straight to L2, owner accumulated.
template <bool kBig, bool kRows, int kPages>
__device__ __forceinline__ void fallback_record(uint64_t x, OwnCache& oc, LaneAcc& la, const Ctx& c, const Out& o,
                                             uint32_t k) {
  const Ival I = lookup<kBig>(oc, x, c);
  if (I.page == kOOW) {
    red_add_u64(o.totals + 2, 1);
  } else if (kPages == 0 && kCacheBits && PASTA_PCACHE_F && o.cache != 0u) {
    cache_add(o, I.page, 1);
  } else {
    red_add_u64(o.page_counts + I.page, 1);
    hot_add<kPages>(o, I.page, 1, k);
    if ((kPages & 1) && la.kbit != I.page) {
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

// One lane's own (page, owner, count) entry straight to L2 (page) and to its LaneAcc
// (owner), as tier F does for a single record.
template <bool kRows, int kPages>
__device__ __forceinline__ void lane_entry(LaneAcc& la, const Out& o, uint32_t page, uint32_t own, uint32_t cnt,
                                           uint32_t k) {
#if PASTA_PCACHE_L
  page_scatter<kPages>(o, page, cnt, k);
#else
  page_to_global<kPages>(o, page, cnt, k);
#endif
  if (own != la.own) {
    owner_to_global<kRows>(o, la.own, la.ocnt, k);
    la.own = own;
    la.ocnt = 0;
  }
  la.ocnt += cnt;
}

// Warp-collective: merge every lane's up to two (page, owner, count) entries into the
// warp accumulators (leader loop; one __reduce_add_sync per distinct key). After
// PASTA_MERGE_ITERS distinct keys the entries are scattered (random pages): every lane
// then sends its remaining entries itself instead of serialising one key per step.
#ifndef PASTA_MERGE_ITERS
#define PASTA_MERGE_ITERS 2
#endif
template <bool kRows, int kPages>
__device__ __forceinline__ void merge_entries(WarpAcc& w, LaneAcc& la, const Out& o, uint32_t k, uint32_t lane,
                                              bool pa, uint32_t pA, uint32_t oA, uint32_t cA, bool pb, uint32_t pB,
                                              uint32_t oB, uint32_t cB) {
#pragma unroll 1
  for (int it = 0;; ++it) {
    const unsigned m = __ballot_sync(kFull, pa || pb);
    if (m == 0) return;
    if (it == PASTA_MERGE_ITERS) break;
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
  if (pa) lane_entry<kRows, kPages>(la, o, pA, oA, cA, k);
  if (pb) lane_entry<kRows, kPages>(la, o, pB, oB, cB, k);
}

// Tier L + F for this lane's records selected by `valid` (bit i <-> a[i]).
template <bool kBig, bool kRows, int kPages>
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
      // a rolled loop over the remaining records keeps the compiler from hoisting the
      // per-record address arithmetic of the rare path into every slice
#pragma unroll 1
      while (miss) {
        const int i = __ffs(miss) - 1;
        miss &= miss - 1;
        uint64_t z = a[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) z = (i == j) ? a[j] : z;
        fallback_record<kBig, kRows, kPages>(z, oc, la, c, o, k);
      }
    }
  }
  merge_entries<kRows, kPages>(w, la, o, k, lane, cA > 0, IA.page, IA.own, cA, cB > 0, IB.page, IB.own, cB);
}

__device__ __forceinline__ uint32_t lo32(uint64_t x) { return static_cast<uint32_t>(x); }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return static_cast<uint32_t>(x >> 32); }

// #{ i : v[i] <= t } for non-decreasing v[0..7] (three probes + the top element).
__device__ __forceinline__ uint32_t count_sorted8(const uint32_t (&v)[8], uint32_t t) {
  uint32_t c = (v[3] <= t) ? 4u : 0u;
  const uint32_t x = c ? v[5] : v[1];
  c += (x <= t) ? 2u : 0u;
  const uint32_t y = (c & 4u) ? ((c & 2u) ? v[6] : v[4]) : ((c & 2u) ? v[2] : v[0]);
  c += (y <= t) ? 1u : 0u;
  return (v[7] <= t) ? 8u : c;
}

// Full 256-record slice. `a` holds the strided view (lane l: positions 64i + 2l + h);
// `slot` is the slice's shared-memory address (for the lane-contiguous re-read).
template <bool kBig, bool kRows, int kPages>
__device__ __forceinline__ void process_full(const uint64_t (&a)[8], uint32_t slot, Ival& cur, OwnCache& oc,
                                             LaneAcc& la, WarpAcc& w, const Ctx& c, const Out& o, uint32_t k,
                                             uint32_t lane) {
#if PASTA_XFL_LDS
  const uint64_t xf = lds64(slot);
  const uint64_t xl = lds64(slot + 8u * (kSlice - 1));
#else
  const uint64_t xf = __shfl_sync(kFull, a[0], 0);
  const uint64_t xl = __shfl_sync(kFull, a[7], 31);
#endif
  Ival IA = cur;
  if (!inside(xf, IA)) IA = lookup<kBig>(oc, xf, c);
  const bool same = inside(xl, IA);
  Ival IB = IA;
  if (!same) IB = lookup<kBig>(oc, xl, c);
  cur = IB;
  const uint64_t alast = IA.lo + IA.span;
  const uint64_t blast = IB.lo + IB.span;
  const uint32_t H = hi32(IA.lo);
  // ---- tier W: A u B is one 32-bit-addressable range and every lane is sorted ----
  if ((same || IB.lo - 1 == alast) && hi32(blast) == H) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = lo32(a[i]);
#if PASTA_TREE
    // independent predicates combined by a balanced tree (short dependency chains)
    const bool h01 = (hi32(a[0]) == H) & (hi32(a[1]) == H), h23 = (hi32(a[2]) == H) & (hi32(a[3]) == H);
    const bool h45 = (hi32(a[4]) == H) & (hi32(a[5]) == H), h67 = (hi32(a[6]) == H) & (hi32(a[7]) == H);
    const bool m03 = (v[0] <= v[1]) & (v[1] <= v[2]) & (v[2] <= v[3]);
    const bool m37 = (v[3] <= v[4]) & (v[4] <= v[5]) & (v[5] <= v[6]) & (v[6] <= v[7]);
    const bool ends = (v[0] >= lo32(IA.lo)) & (v[7] <= lo32(blast));
    const bool ok = ((h01 & h23) & (h45 & h67)) & (m03 & m37) & ends;
#else
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 8; ++i) ok = ok && hi32(a[i]) == H;
    ok = ok && v[0] >= lo32(IA.lo) && v[7] <= lo32(blast);
#pragma unroll
    for (int i = 0; i < 7; ++i) ok = ok && v[i] <= v[i + 1];
#endif
    if (__all_sync(kFull, ok)) {
      const uint32_t sA = same ? (uint32_t)kSlice : __reduce_add_sync(kFull, count_sorted8(v, lo32(alast)));
      wadd2<kRows, kPages>(w, o, IA, sA, IB, kSlice - sA, k, lane);
      return;
    }
  }
  // ---- tier W2: every record in A or B, any order ----
  {
    uint32_t cA = 0;
    bool ok = true;
    if (hi32(alast) == H && hi32(IB.lo) == hi32(blast)) {
      const uint32_t HB = hi32(IB.lo), LA = lo32(IA.lo), LB = lo32(IB.lo);
      const uint32_t SA = lo32(IA.span), SB = lo32(IB.span);
#if PASTA_TREE
      uint32_t mA = 0, mB = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        mA |= ((hi32(a[i]) == H) & (lo32(a[i]) - LA <= SA)) ? (1u << i) : 0u;
        mB |= ((hi32(a[i]) == HB) & (lo32(a[i]) - LB <= SB)) ? (1u << i) : 0u;
      }
      cA = __popc(mA);
      ok = (mA | mB) == 0xFFu;
#else
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool inA = hi32(a[i]) == H && lo32(a[i]) - LA <= SA;
        const bool inB = hi32(a[i]) == HB && lo32(a[i]) - LB <= SB;
        cA += inA ? 1u : 0u;
        ok = ok && (inA || inB);
      }
#endif
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool inA = inside(a[i], IA);
        cA += inA ? 1u : 0u;
        ok = ok && (inA || inside(a[i], IB));
      }
    }
    if (__all_sync(kFull, ok)) {
      const uint32_t sA = __reduce_add_sync(kFull, cA);
      wadd2<kRows, kPages>(w, o, IA, sA, IB, kSlice - sA, k, lane);
      return;
    }
  }
#if PASTA_TIER_S
  // ---- tier S: every record in one owner interval and in the window, pages scattered
  // (random or strided access inside one allocation): owner count warp-uniform, each
  // lane sends its own page runs, no per-record lookup ----
  {
    own_lookup<kBig>(oc, xf, c);  // xf's owner interval: the same in every lane
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 8; ++i) ok = ok && (a[i] - oc.olo <= oc.ospan) && (a[i] - c.va_lo < c.wbytes);
    if (__all_sync(kFull, ok)) {
      if (oc.own != w.own) {
        if (lane == 0) owner_to_global<kRows>(o, w.own, w.ocnt, k);
        w.own = oc.own;
        w.ocnt = 0;
      }
      w.ocnt += kSlice;
#if PASTA_TIER_S_BATCH
      if (kPages == 0 && !(kCacheBits && o.cache)) {
        // every page and run end first, then the REDs back to back: each RED has its own
        // address / value registers, so no RED waits for the previous one's operands to
        // drain (the loop below stalled on that write-after-read at every RED)
        uint32_t q[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) q[i] = (uint32_t)((a[i] - c.va_lo) >> c.s);
        uint32_t start = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i == 7 || q[i + 1 < 8 ? i + 1 : 7] != q[i]) {
            red_add_u64(o.page_counts + q[i], (uint64_t)(i + 1 - start));
            start = i + 1;
          }
        }
        return;
      }
#endif
      uint32_t pp = (uint32_t)((a[0] - c.va_lo) >> c.s), n = 1;
#pragma unroll
      for (int i = 1; i < 8; ++i) {
        const uint32_t p = (uint32_t)((a[i] - c.va_lo) >> c.s);
        if (p != pp) {
          page_scatter<kPages>(o, pp, n, k);
          pp = p;
          n = 0;
        }
        ++n;
      }
      page_scatter<kPages>(o, pp, n, k);
      return;
    }
  }
#endif
  // ---- tier L: lane-contiguous re-read (8 consecutive records, rotated order) ----
  uint64_t b[8];
  const uint32_t rsh = (lane >> 1) & 3u;
  const uint32_t base = slot + 64u * lane;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const ulonglong2 x = lds128(base + 16u * ((i + rsh) & 3u));
    b[2 * i] = x.x;
    b[2 * i + 1] = x.y;
  }
  process_lane<kBig, kRows, kPages>(b, 0xFFu, oc, la, w, c, o, k, lane);
}

// Warp-local flush of everything accumulated for kernel segment k.
template <bool kRows, int kPages>
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

template <bool kBig, bool kRows, int kPages, bool kIL, bool kPair>
__global__ void __launch_bounds__(kThreads, 1) scan_kernel(const ScanArgs args, const int stages, const int cache_on) {
  // Programmatic dependent launch: the next analyze call's scan may start its prologue
  // (barrier init, range table into shared memory) on free SMs while this one runs. A
  // chained scan (early == 2) triggers at entry: its predecessor is a scan that already
  // passed its own grid-dependency wait. Any other scan triggers only after its wait, so
  // a chained successor (which never waits before its REDs) cannot start before the
  // chain's first call has seen every earlier kernel (e.g. the outputs' zeroing) complete.
  if (args.early == 2) grid_dep_launch_dependents();
  extern __shared__ __align__(128) unsigned char smem[];
  // dynamic shared memory: [page-count cache (kPages == 0, cache_on) | ring | barriers |
  // lane accumulators | chunk map slots | range table]
  unsigned char* sm = smem + ((kPages == 0 && kCacheBits && cache_on) ? kCacheBytes : 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + ring_bytes(stages));
  uint64_t* sB = reinterpret_cast<uint64_t*>(sm + ring_bytes(stages) + kBarBytes + kLaBytes + kPfBytes);

  const uint32_t A = args.A;
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nsl = (args.nbody + kSlice - 1) / kSlice;
  const uint32_t gwarp = blockIdx.x * kWarps + warp;
  const uint32_t nwarp = gridDim.x * kWarps;
  // the last slice of the trace may be partial
  const uint32_t tail_valid = (uint32_t)(args.nbody - (nsl - 1) * kSlice);
  // Relative slice j of this warp -> global slice gsl(j).
  //  * contiguous schedule: slices [s0, s1) (short launches, where every warp holds few
  //    slices and a straggler costs little);
  //  * interleaved schedule (kIL): chunks of 2^lc slices, warp gw takes chunks gw,
  //    gw + W, ..., so every warp samples the whole trace (cheap sweeps, tiled jumps and
  //    scattered records alike) and no warp straggles behind an expensive region.
  //  * dynamic interleaved (kIL, PASTA_IL_DYNAMIC): the warp's first chunk is gw, every
  //    later one comes from a global counter (lane 0, one atomic per chunk, taken when the
  //    previous chunk starts), so warps that drew cheap chunks take more and all warps end
  //    within about one chunk of each other (static interleaving: the last warp ended
  //    5-8 % after the median one, scripts/warp_times.py).
  uint32_t lc = 0, icm = 0, nmy;
  uint64_t s0 = 0;
  bool tail_mine;
  uint32_t nch = 0;
  const uint32_t ring_u32 = smem_u32(sm) + (uint32_t)(warp * stages) * kSliceBytes;
  const uint32_t bar_u32 = smem_u32(bars + warp * kMaxStages);
  // the ids of this warp's m-th chunk live in its spare barrier slots 6 and 7 (stages <= 6):
  // cid(m) = slot 6 + (m & 1)
  const uint32_t cid_u32 = bar_u32 + 8u * 6u;
  auto clen = [&](uint32_t q) -> uint32_t { return q + 1 == nch ? (uint32_t)(nsl - ((uint64_t)q << lc)) : icm + 1u; };
  if constexpr (kIL) {
    lc = args.log_ic;
    icm = (1u << lc) - 1u;
    nch = (uint32_t)((nsl + icm) >> lc);
#if PASTA_IL_DYNAMIC
    // until chunk 0 starts (and takes chunk 1's id) the warp knows only its first chunk
    tail_mine = gwarp + 1 == nch;
    nmy = gwarp < nch ? clen(gwarp) : 0u;
    if (lane == 0) sts32_o(cid_u32, gwarp);
    __syncwarp();
#else
    const uint64_t nct = gwarp < nch ? (nch - gwarp + nwarp - 1) / nwarp : 0;  // my chunks
    tail_mine = nct > 0 && (gwarp + (nct - 1) * nwarp == nch - 1);            // I own the last chunk
    nmy = (uint32_t)((nct << lc) - (tail_mine ? ((uint64_t)nch << lc) - nsl : 0));
#endif
  } else {
    s0 = (uint64_t)gwarp * nsl / nwarp;
    const uint64_t s1 = (uint64_t)(gwarp + 1) * nsl / nwarp;
    nmy = (uint32_t)(s1 - s0);
    tail_mine = s1 == nsl;
  }
  auto gsl = [&](uint32_t j) -> uint64_t {
    // chunk index < 2^32 (a launch holds < 2^32 slices)
    if constexpr (kIL) {
#if PASTA_IL_DYNAMIC
      return ((uint64_t)lds32_o(cid_u32 + 4u * ((j >> lc) & 1u)) << lc) + (j & icm);
#else
      return ((uint64_t)((j >> lc) * nwarp + gwarp) << lc) + (j & icm);
#endif
    } else {
      return s0 + j;
    }
  };
  uint32_t nfull = (tail_mine && nmy > 0 && tail_valid != (uint32_t)kSlice) ? nmy - 1 : nmy;

  if (lane == 0) {
    for (int j = 0; j < stages; ++j) mbar_init(bars + warp * kMaxStages + j, 1);
    fence_mbar_init();
  }
  // the range table is only ever written by stream-ordered copies, never by a kernel
  if (!kBig)
    for (uint32_t i = threadIdx.x; i < 2 * A; i += kThreads) sB[i] = args.bounds[i];
  else  // the global table's shared-memory samples (where the table would otherwise sit)
    for (uint32_t i = threadIdx.x; i < args.samp_n; i += kThreads) sB[i] = args.bounds[(uint64_t)i << args.samp_sh];
  const bool cache = kPages == 0 && kCacheBits && cache_on;
  if (cache)
    for (uint32_t i = threadIdx.x; i + 1 <= kCacheSlots; i += kThreads) sts64(cache_base() + 8u * i, kCacheEmptySlot);
  __syncthreads();
  // Everything the stream's previous kernel wrote (the records, a chunk map, zeroed or
  // partial outputs) is visible after grid_dep_wait; nothing before it touches that
  // data, except the first record loads when the caller declared the records stable
  // (PASTA_REC_STABLE: not written by the stream's previous kernel).
  if (!args.early) {
    grid_dep_wait();
    grid_dep_launch_dependents();
  }
#if PASTA_TRACE_TIMING
  const uint32_t tslot = (blockIdx.x * kWarps + warp) * 4;
  if (lane == 0) g_warp_times[tslot] = gtimer();
#endif

  const uint64_t pol = l2_evict_first_policy();
  // TMA for relative slice j into ring slot `slot` (lane 0 only)
  auto issue = [&](uint32_t j, uint32_t slot) {
    const uint32_t bytes = j < nfull ? kSliceBytes : tail_valid * 8u;
    PASTA_DCHECK(slot < (uint32_t)stages && j < nmy && gsl(j) * kSlice * 8 + bytes <= args.nbody * 8);
    mbar_arrive_expect_tx_u32(bar_u32 + 8u * slot, bytes);
    tma_load_1d_u32(ring_u32 + slot * kSliceBytes, args.rec + gsl(j) * kSlice, bytes, bar_u32 + 8u * slot, pol);
  };
  // kPair: double slots, relative slices 2p, 2p + 1 in one 4 KiB copy (contiguous in both
  // schedules: interleaved chunks hold an even number of slices, the partial tail is the
  // trace's last slice). Half as many bulk copies in flight for the same bytes: llama
  // 13.55 -> 13.22 ms (B200 A/B; the read microbenchmark scripts/micro/read_bw.cu shows
  // fewer, larger copies per SM reaching more of HBM). Used when the ring depth is even.
  const uint32_t S2 = (uint32_t)stages / 2u;
  auto issue_pair = [&](uint32_t p, uint32_t s2) {
    const uint32_t j = 2u * p;
    uint32_t bytes = j < nfull ? kSliceBytes : tail_valid * 8u;
    if (j + 1 < nmy) bytes += j + 1 < nfull ? kSliceBytes : tail_valid * 8u;
    PASTA_DCHECK(s2 < S2 && j < nmy && gsl(j) * kSlice * 8 + bytes <= args.nbody * 8 &&
                 (j + 1 >= nmy || gsl(j + 1) == gsl(j) + 1));
    mbar_arrive_expect_tx_u32(bar_u32 + 8u * s2, bytes);
    tma_load_1d_u32(ring_u32 + s2 * 2u * kSliceBytes, args.rec + gsl(j) * kSlice, bytes, bar_u32 + 8u * s2, pol);
  };
  if (lane == 0) {
    if constexpr (kPair) {
      for (uint32_t p = 0; p < S2 && 2u * p < nmy; ++p) issue_pair(p, p);
    } else {
      for (uint32_t j = 0; j < (uint32_t)stages && j < nmy; ++j) issue(j, j);
    }
  }
  if (args.early == 1) {
    grid_dep_wait();
    grid_dep_launch_dependents();
  }
  if (lane == 0 && blockIdx.x == 0 && warp == 0 && args.add_records) red_add_u64(args.totals + 0, args.add_records);

  Ctx c;
  c.va_lo = args.va_lo;
  c.va_hi = args.va_hi;
  c.wbytes = args.va_hi - args.va_lo;
  c.s = args.page_shift;
  c.A = A;
  c.B = kBig ? args.bounds : sB;
  if (kBig) {
    c.S = sB;
    c.nS = args.samp_n;
    c.sh = args.samp_sh;
  }
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
  o.hot = args.hot;
  o.P = args.P;
  o.wk = args.window_kernels;
  o.wk_magic = args.wk_magic;
  o.tids = args.tids;
  o.tcounts = args.tensor_counts;
  o.ktc = args.ktc;
  o.max_tids = args.max_tids;
  o.cache = cache ? 1u : 0u;

  OwnCache oc;
  oc.olo = 1;
  oc.ospan = 0;  // forces a search on the first lookup
  oc.own = A;
  Ival cur = lookup<kBig>(oc, 0ull, c);  // a valid interval (the one holding address 0)
  WarpAcc w;
  w.page = kOOW - 1;
  w.own = A;
  w.pcnt = 0;
  w.ocnt = 0;
#if PASTA_LA_SMEM
  // the rarely used tier-F accumulators live in shared memory (fewer live registers)
  LaneAcc& la = reinterpret_cast<LaneAcc*>(sm + ring_bytes(stages) + kBarBytes)[threadIdx.x];
#else
  LaneAcc la;
#endif
  la.own = A;
  la.ocnt = 0;
  la.kbit = kOOW;

  // Kernel segments: slice j holds global records gidx0 + 256 gsl(j) + position.
  const uint32_t K = args.n_kernels;
  uint32_t k = 0;
  uint64_t kend = ~0ull;  // global index where segment k ends
  // interleaved: chunk starts are events, the chunk's (k, kend) comes from the pre-pass
  // table, copied to this warp's shared slot one chunk ahead (cp.async), off the critical
  // path and out of the register file
  const uint32_t pf_u32 = smem_u32(sm) + ring_bytes(stages) + kBarBytes + kLaBytes + 16u * warp;
  auto prefetch_chunk = [&](uint32_t j) {
    if (kRows && K > 1 && j < nmy && lane == 0) cp_async_16(pf_u32, args.chunk_k + (gsl(j) >> lc));
  };
  auto enter_chunk = [&](uint32_t j) {
#if PASTA_IL_DYNAMIC
    if constexpr (kIL) {
      // take the chunk after this one (all lanes: nmy / nfull are warp-uniform)
      const uint32_t m = j >> lc;
      uint32_t qn = 0;
      if (lane == 0) {
        const uint64_t c = atomicAdd(args.chunk_ctr, 1ull);
        // chunk_perm != 0: the grab order is permuted over the dynamic chunks except the
        // trace's last one (always drawn last, so a warp's partial tail slice is its final
        // slice): the last grabs land anywhere in the trace instead of on its final region
        const uint64_t M1 = nch > nwarp + 1 ? (uint64_t)(nch - nwarp - 1) : 0;
        qn = nwarp + (uint32_t)(args.chunk_perm && c < M1 ? (c * args.chunk_perm) % M1 : c);
        sts32_o(cid_u32 + 4u * ((m + 1u) & 1u), qn);
      }
      __syncwarp();
      qn = __shfl_sync(kFull, qn, 0);
      const uint32_t qm = lds32_o(cid_u32 + 4u * (m & 1u));
      const bool more = qn < nch;
      PASTA_DCHECK(qm < nch && (j & icm) == 0 && lc >= 3);
      nmy = j + clen(qm) + (more ? clen(qn) : 0u);
      tail_mine = (more ? qn : qm) + 1 == nch;
      nfull = (tail_mine && tail_valid != (uint32_t)kSlice) ? nmy - 1 : nmy;
    }
#endif
    if (kRows && K > 1) {
      if (lane == 0) cp_async_wait_all();
      __syncwarp();
      const ulonglong2 pf = lds128(pf_u32);
      __syncwarp();
      const uint32_t nk = (uint32_t)pf.x;
      if (nk != k) {
        warp_flush<kRows, kPages>(w, la, o, k, lane);
        k = nk;
      }
      kend = pf.y;
      prefetch_chunk(j + icm + 1);
    }
  };
  // first relative slice after j that is not a plain full slice inside segment k: the
  // slice holding record kend, the partial tail slice, or (interleaved) the next chunk
  auto next_event_after = [&](uint32_t j) -> uint32_t {
    if constexpr (kIL) {
      const uint32_t jb = j & ~icm;
      // chunk starts are events (the chunk map; with the dynamic schedule also the next grab)
      uint64_t e = ((kRows && K > 1) || PASTA_IL_DYNAMIC) ? (uint64_t)jb + icm + 1 : nfull;
      if (nfull < e) e = nfull;
      if (kRows && kend != ~0ull) {
        const uint64_t gb = args.gidx0 + gsl(jb) * kSlice;
        if (kend >= gb) {
          const uint64_t kb = jb + (kend - gb) / kSlice;
          if (kb < e && kb > j) e = kb;
        }
      }
      return (uint32_t)e;
    } else {
      uint64_t e = nfull;
      if (kRows && kend != ~0ull) {
        const uint64_t kb = (kend - args.gidx0) / kSlice - s0;  // slice holding record kend (or starting at it)
        if (kb < e) e = kb;
      }
      return (uint32_t)e;
    }
  };
  uint32_t jev;
  if constexpr (kIL) {
    prefetch_chunk(0);
    if (nmy > 0) enter_chunk(0);  // (dynamic: takes chunk 1's id, extends nmy)
    jev = nmy > 0 ? next_event_after(0) : 0;
    if (kRows && K > 1 && nmy > 0) {
      // the first slice itself may hold a boundary
      const uint64_t gb = args.gidx0 + gsl(0) * kSlice;
      if (kend < gb + kSlice) jev = 0;
    }
    if (nfull == 0) jev = 0;
  } else {
    if (kRows && K > 1 && nmy > 0) {
      k = kernel_of(args.koffs, K, args.gidx0 + s0 * kSlice);
      kend = (k + 1 < K) ? __ldg(args.koffs + k + 1) : ~0ull;
    }
    jev = next_event_after(0);
  }

  uint32_t slot = 0, phase = 0;
  for (uint32_t j = 0; j < nmy; ++j) {
    const uint32_t sa = ring_u32 + slot * (kPair ? 2u : 1u) * kSliceBytes + (kPair ? (j & 1u) * kSliceBytes : 0u);
    if (!kPair || (j & 1u) == 0) mbar_wait_u32(bar_u32 + 8u * slot, phase);
#if PASTA_TRACE_TIMING
    if (lane == 0 && j == 0) g_warp_times[tslot + 1] = gtimer();
    if (lane == 0 && j == nmy / 4) g_warp_times[tslot + 2] = gtimer();
#endif
    uint64_t a[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const ulonglong2 v = lds128(sa + 16u * lane + 512u * i);
      a[2 * i] = v.x;
      a[2 * i + 1] = v.y;
    }
    if (j != jev) {
      process_full<kBig, kRows, kPages>(a, sa, cur, oc, la, w, c, o, k, lane);
    } else {
      // kernel boundary in or at this slice, or the partial tail slice (or, in the
      // interleaved schedule, the first slice of a chunk)
      if (kIL && (j & icm) == 0 && j > 0) enter_chunk(j);
      const uint32_t valid = j < nfull ? (uint32_t)kSlice : tail_valid;
      const uint64_t g0 = args.gidx0 + gsl(j) * kSlice;
      uint32_t r0 = 0;
      for (;;) {
        if (kRows && g0 + r0 >= kend) {
          warp_flush<kRows, kPages>(w, la, o, k, lane);
          while (k + 1 < K && __ldg(args.koffs + k + 1) <= g0 + r0) ++k;
          kend = (k + 1 < K) ? __ldg(args.koffs + k + 1) : ~0ull;
        }
        uint32_t r1 = valid;
        if (kRows && kend - g0 < (uint64_t)r1) r1 = (uint32_t)(kend - g0);
        if (r0 == 0 && r1 == (uint32_t)kSlice) {
          process_full<kBig, kRows, kPages>(a, sa, cur, oc, la, w, c, o, k, lane);
        } else {
          uint32_t vm = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t pos = 64u * (i >> 1) + 2u * lane + (i & 1);
            if (pos >= r0 && pos < r1) vm |= 1u << i;
          }
          process_lane<kBig, kRows, kPages>(a, vm, oc, la, w, c, o, k, lane);
        }
        r0 = r1;
        if (r0 >= valid) break;
      }
      jev = next_event_after(j);  // > j: kend now lies beyond every record of this slice
    }
    // the slot is free again (every lane has consumed its values): refill it with the
    // slice `stages` ahead
    __syncwarp();
    if constexpr (kPair) {
      if ((j & 1u) || j + 1 == nmy) {  // both slices of the double slot consumed
        if (lane == 0 && 2u * ((j >> 1) + S2) < nmy) issue_pair((j >> 1) + S2, slot);
        if (++slot == S2) {
          slot = 0;
          phase ^= 1u;
        }
      }
    } else {
#if PASTA_ISSUE2
    // refills in pairs (every odd slice, this slot and the previous one): the issue path
    // recomputes its shared-memory and source addresses (register pressure), and two
    // issues share that work
    if (lane == 0 && (j & 1u)) {
      const uint32_t prev = slot == 0 ? (uint32_t)stages - 1u : slot - 1u;
      if (j - 1 + stages < nmy) issue(j - 1 + stages, prev);
      if (j + stages < nmy) issue(j + stages, slot);
    }
#else
      if (lane == 0 && j + stages < nmy) issue(j + stages, slot);
#endif
      if (++slot == (uint32_t)stages) {
        slot = 0;
        phase ^= 1u;
      }
    }
  }
  warp_flush<kRows, kPages>(w, la, o, k, lane);
  if (cache) {  // write the page-count cache back
    __syncthreads();
    for (uint32_t i = threadIdx.x; i + 1 <= kCacheSlots; i += kThreads) {
      const uint64_t v = lds64(cache_base() + 8u * i);
      if ((uint32_t)(v >> 32) != kCacheEmpty && (uint32_t)v != 0u)
        red_add_u64(args.page_counts + (uint32_t)(v >> 32), (uint32_t)v);
    }
  }
  // PASTA_REC_CHAINED: the predecessor is a scan into the same outputs (its REDs commute
  // with ours), so the work above never waited for it; this grid still completes only
  // after it, which keeps completion in stream order for every later reader.
  if (args.early == 2) grid_dep_wait();
#if PASTA_TRACE_TIMING
  if (lane == 0) g_warp_times[tslot + 3] = gtimer();
#endif
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
  o.hot = s.hot;
  o.P = s.P;
  o.wk = s.window_kernels;
  o.wk_magic = s.wk_magic;
  o.tids = s.tids;
  o.tcounts = s.tensor_counts;
  o.ktc = s.ktc;
  o.max_tids = s.max_tids;
  if (rows) owner_to_global<true>(o, I.own, 1, k);
  else owner_to_global<false>(o, I.own, 1, k);
  const int mode = (s.kpb ? 1 : 0) | (s.hot ? 2 : 0);
  if (mode == 3) page_to_global<3>(o, I.page, 1, k);
  else if (mode == 2) page_to_global<2>(o, I.page, 1, k);
  else if (mode == 1) page_to_global<1>(o, I.page, 1, k);
  else page_to_global<0>(o, I.page, 1, k);
}

int stages_for(uint32_t A, bool big, long extra = 0) {
  const long table = big ? 0 : 16l * A;
  const long avail = (long)kSmemLimit - kBarBytes - kLaBytes - kPfBytes - table - extra;
  long st = avail / ring_bytes(1);
  if (st > 6) st = 6;  // barrier slots 6 and 7 of each warp hold the dynamic schedule's chunk ids
  return (int)st;
}

// The page-count cache is on when it leaves at least PASTA_PCACHE_MIN_STAGES ring stages.
#ifndef PASTA_PCACHE_MIN_STAGES
#define PASTA_PCACHE_MIN_STAGES 3
#endif
bool cache_fits(uint32_t A, bool big) { return kCacheBits && stages_for(A, big, kCacheBytes) >= PASTA_PCACHE_MIN_STAGES; }

// chunk_k[c] = (kernel segment k of interleaved chunk c's first record, koffs[k + 1])
// (fill: kernel rows with several kernels); thread 0 also resets the dynamic schedule's
// chunk counter. Runs before every interleaved scan.
__global__ void chunk_kernel_map(const __grid_constant__ ScanArgs a, ulonglong2* chunk_k, uint64_t nch, int fill) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && a.chunk_ctr) *a.chunk_ctr = 0;
  if (!fill || i >= nch) return;
  const uint32_t k = kernel_of(a.koffs, a.n_kernels, a.gidx0 + (i << a.log_ic) * kSlice);
  chunk_k[i] = make_ulonglong2(k, k + 1 < a.n_kernels ? a.koffs[k + 1] : ~0ull);
}

template <bool kBig, bool kRows, int kPages>
cudaError_t launch_variant(const ScanArgs& a, int grid, cudaStream_t st) {
  const int cache_on = (kPages == 0 && cache_fits(a.A, kBig)) ? 1 : 0;
  const int stages = stages_for(a.A, kBig, cache_on ? kCacheBytes : 0);
  ScanArgs b = a;
  b.samp_n = b.samp_sh = 0;
  if (kBig && PASTA_BIG_SAMPLES) {  // samples of the global table in the free shared memory
    const long base = (long)ring_bytes(stages) + kBarBytes + kLaBytes + kPfBytes + (cache_on ? kCacheBytes : 0);
    const uint64_t room = (uint64_t)((long)kSmemLimit - base) / 8, m = 2ull * a.A;
    uint32_t sh = 3;
    while (((m + (1ull << sh) - 1) >> sh) > room) ++sh;
    b.samp_sh = sh;
    b.samp_n = (uint32_t)((m + (1ull << sh) - 1) >> sh);
  }
  const int smem = ring_bytes(stages) + kBarBytes + kLaBytes + kPfBytes + (kBig ? 8 * (int)b.samp_n : (int)(16ull * a.A)) +
                   (cache_on ? kCacheBytes : 0);
  // paired 4 KiB copies need an even ring depth and (interleaved) chunks of >= 2 slices
  const bool pair = PASTA_TMA_PAIR && stages % 2 == 0 && a.log_ic != 0;
  // the dynamic interleaved schedule needs chunks of more than a ring depth of slices
  if (PASTA_IL_DYNAMIC && a.log_ic >= 0 && (1 << a.log_ic) < 2 * stages) return cudaErrorInvalidValue;
  auto fn = a.log_ic >= 0 ? (pair ? scan_kernel<kBig, kRows, kPages, true, true> : scan_kernel<kBig, kRows, kPages, true, false>)
                          : (pair ? scan_kernel<kBig, kRows, kPages, false, true>
                                  : scan_kernel<kBig, kRows, kPages, false, false>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // launched as a programmatic dependent of the stream's previous kernel (the kernel
  // waits for it with griddepcontrol.wait before touching any global data)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = PASTA_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, b, stages, cache_on);
}

// ------------------------------------------------------------------------------------
// Streaming ring consumer (NEXT f2). The paper's operating point is a
// device buffer ("4MB") that the instrumented program fills and the analysis
// drains. One launch per buffer costs a launch each (1.4 us graph-replayed
// for 0.64 us of HBM time); here ONE persistent cooperative launch consumes batch
// descriptors that the host publishes into a device ring of `slots` descriptors while it
// runs. The global slice sequence G = b * spb + s (batch b, slice s of spb slots per
// batch) is dealt round-robin to the W warps (warp w takes G = w, w + W, ...), so every
// batch is spread over the whole GPU and consecutive batches overlap; each warp keeps its
// own TMA ring S slices ahead exactly like the scan, waiting (lane 0, nanosleep) only
// when the batch it needs is not published yet. A slice is handled by the scan's own
// tiers with the batch's kernel segment (row k0 + local kernel). Progress for the
// producer: each warp exposes the lowest slice it has not read yet, warp 0 of each CTA
// publishes the CTA's minimum (in whole batches) and CTA 0 the global minimum into
// host-mapped memory, so the host reuses a ring slot (and the batch's records) only
// after every warp has read that batch.
// ------------------------------------------------------------------------------------
constexpr int kSlotInfoBytes = 64;  // per warp and ring stage: the slice in flight
// Data warps of the stream consumer; one more warp is the monitor. 23 + 1 = 24 warps keep
// 6 warps per SM sub-partition and so the scan's 80 registers per thread; 24 + 1 (7 on one
// sub-partition) capped them at 72 with spills (ncu: an LDL per slice).
#ifndef PASTA_STREAM_DATA_WARPS
#define PASTA_STREAM_DATA_WARPS (kWarps - 1)
#endif
constexpr int kStreamData = PASTA_STREAM_DATA_WARPS;
static_assert(kStreamData <= kWarps, "the slot, front and turn arrays hold kWarps warps");
constexpr int kStreamThreads = (kStreamData + 1) * 32;
#ifndef PASTA_STREAM_CHUNK
#define PASTA_STREAM_CHUNK 32  // consecutive slices of one batch per warp turn
#endif
constexpr uint32_t kStreamChunk = PASTA_STREAM_CHUNK;
#ifndef PASTA_STREAM_PROF
#define PASTA_STREAM_PROF 0  // per-warp clock64 counters (fill, TMA wait, total) into StreamArgs::prof
#endif
#ifndef PASTA_STREAM_MON_NS
#define PASTA_STREAM_MON_NS 1000  // the monitor warp's pause between progress reports
#endif
constexpr int kFrontBytes = ((kWarps + 1) * 8 + 15) / 16 * 16;  // data warps + monitor, 16-byte multiple

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Lane 0's chunk state of one warp (shared memory). The first 32 bytes are all the
// per-slice fast path reads: slices [cs, cf) of the current chunk are full and lie inside
// one kernel, so issuing one is two 16-byte loads, a tag store and the TMA copy.
struct __align__(16) StreamTurn {
  const uint64_t* rec;   // the current batch's records
  uint32_t cs, cf;       // next slice to issue; end of the fast run
  uint64_t G0;           // global slice index of the batch's slice 0 (b * spb)
  uint32_t krow, eidx;   // kernel row of slice cs (k0 + kl); the chunk's entry (see SlotTag)
  uint32_t ce, nk;       // end of the chunk (slices); kernels in the batch
  uint32_t kl, k0;       // batch-local kernel of slice cs, the batch's first row
  uint64_t kend;         // batch-relative record where kernel kl ends (~0: never)
  const uint64_t* koffs;
  uint64_t n;            // records of the batch
  uint64_t Q, known_tail;
  uint32_t opened, pad;  // chunks opened (entry ring index)
};
static_assert(offsetof(StreamTurn, cs) == 8 && offsetof(StreamTurn, G0) == 16 && offsetof(StreamTurn, krow) == 24 &&
                  offsetof(StreamTurn, eidx) == 28,
              "the fast issue path reads the turn state as two 16-byte words");
constexpr int kTurnBytes = kWarps * (int)sizeof(StreamTurn);
constexpr int kStreamHead = kWarps * kMaxStages * kSlotInfoBytes + kFrontBytes + kTurnBytes;  // see stream_kernel
static_assert(kStreamHead % 16 == 0, "the ring after the head stays 16-byte aligned");

// Per ring slot: what the processing side needs about the slice in it (one 16-byte store
// by lane 0 when it issues the copy, one broadcast load per slice when it is processed).
struct __align__(16) SlotTag {
  uint64_t G;      // global slice index
  uint32_t krow;   // kernel row of the slice's first record
  uint32_t meta;   // bit 3: fast (full, one kernel); bits 0-2: the chunk entry
};
constexpr uint32_t kTagFast = 8u;
// Per chunk the warp opened (ring of kMaxStages = 8 >= stages entries: the slices in
// flight belong to at most `stages` consecutive chunks): what a slow slice needs.
struct __align__(16) ChunkEntry {
  const uint64_t* koffs;
  uint64_t n;
  uint64_t G0;
  uint32_t nk, k0;
};
static_assert(sizeof(SlotTag) + sizeof(ChunkEntry) <= (size_t)kSlotInfoBytes, "tag + entry fit the slot info bytes");
static_assert(kMaxStages == 8, "the entry index takes 3 tag bits");

// The monitor warp of each CTA (all 32 lanes): this CTA's progress to the producer. A
// batch is read by the CTA once every data warp's lowest unread slice lies beyond it;
// the CTA's count of read batches (only published ones: a warp's next slice may lie far
// beyond them) goes to ctl->cta_done[cta]; the monitor of CTA 0 also folds every CTA's
// count into the global minimum and writes it to the producer's host-mapped counter.
// No per-batch atomics: one load per warp and per CTA per round.
__device__ __forceinline__ void stream_report(const StreamArgs& ra, const volatile uint64_t* front,
                                              unsigned long long& cta_last, unsigned long long& glob_last) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t mn = lane < (uint32_t)kWarps ? front[lane] : ~0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t x = __shfl_xor_sync(kFull, mn, o);
    mn = x < mn ? x : mn;
  }
  unsigned long long done = mn == ~0ull ? ld_acquire_u64(&ra.ctl->end) : mn / ra.spb;
  const unsigned long long tail = ld_acquire_u64(&ra.ctl->tail);
  if (done > tail) done = tail;
  if (done > cta_last) {
    cta_last = done;
    if (lane == 0) st_release_u64(&ra.ctl->cta_done[blockIdx.x], done);
  }
  if (blockIdx.x == 0) {
    unsigned long long g = ~0ull;
    for (uint32_t c = lane; c < gridDim.x; c += 32) {
      const unsigned long long v = ld_acquire_u64(&ra.ctl->cta_done[c]);
      g = v < g ? v : g;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(kFull, g, o);
      g = x < g ? x : g;
    }
    if (g > glob_last) {
      glob_last = g;
      if (lane == 0) st_release_sys_u64(ra.consumed, g);
    }
  }
}

template <bool kBig, bool kRows, int kPages>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_kernel(const __grid_constant__ StreamArgs ra,
                                                                     const int stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  const ScanArgs& args = ra.s;
  // dynamic shared memory: [slot infos | fronts | turn states] at fixed offsets (cheap
  // addresses), then [ring | barriers | lane accumulators | range table]
  volatile uint64_t* front = reinterpret_cast<volatile uint64_t*>(smem + kWarps * kMaxStages * kSlotInfoBytes);
  StreamTurn* turns = reinterpret_cast<StreamTurn*>(smem + kWarps * kMaxStages * kSlotInfoBytes + kFrontBytes);
  unsigned char* sm2 = smem + kStreamHead;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm2 + ring_bytes(stages));
  uint64_t* sB = reinterpret_cast<uint64_t*>(sm2 + ring_bytes(stages) + kBarBytes + kLaBytes);
  const uint32_t A = args.A;
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  SlotTag* tags = reinterpret_cast<SlotTag*>(smem) + warp * kMaxStages;
  ChunkEntry* ents = reinterpret_cast<ChunkEntry*>(smem + kWarps * kMaxStages * sizeof(SlotTag)) + warp * kMaxStages;
  const uint32_t ring_u32 = smem_u32(sm2) + (uint32_t)(warp * stages) * kSliceBytes;
  const uint32_t bar_u32 = smem_u32(bars + warp * kMaxStages);
  if (lane == 0 && warp < kStreamData) {
    for (int j = 0; j < stages; ++j) mbar_init(bars + warp * kMaxStages + j, 1);
    fence_mbar_init();
  }
  if (!kBig)
    for (uint32_t i = threadIdx.x; i < 2 * A; i += blockDim.x) sB[i] = args.bounds[i];
  const uint64_t W = (uint64_t)gridDim.x * kStreamData;
  const uint64_t gnext = (uint64_t)blockIdx.x * kStreamData + warp;  // the warp's first chunk
  const uint64_t cpb = ra.cpb;  // chunks per batch slot (a parameter: no division to rematerialise)
  if (lane == 0)
    front[warp] = warp < kStreamData ? (gnext / cpb) * ra.spb + (gnext % cpb) * kStreamChunk : ~0ull;
  __syncthreads();
  if (warp == kStreamData) {
    // the CTA's monitor warp (processes no slices): publishes the CTA's progress until
    // every data warp has read its last slice (CTA 0's: until every CTA has), so the
    // producer never waits on a warp that is busy reading records
    unsigned long long cta_last = 0, glob_last = 0;
    for (;;) {
      stream_report(ra, front, cta_last, glob_last);
      const unsigned long long end = ld_acquire_u64(&ra.ctl->end);
      if (cta_last == end && (blockIdx.x != 0 || glob_last == end)) break;
      __nanosleep(PASTA_STREAM_MON_NS);
    }
    return;
  }

  const uint64_t pol = l2_evict_first_policy();
  // lane 0: the warp's next non-empty slice into ring slot `slot`. Returns 1 when issued,
  // 0 when its batch is not published yet (only if !block; with block it waits, reporting
  // progress meanwhile if this is warp 0), 2 when the stream has ended before it.
  // Warp turns: chunk Q = gw, gw + W, ... of the global chunk sequence (batch Q / cpb,
  // slices [C (Q % cpb), C (Q % cpb + 1)) of it), so a warp reads one descriptor and
  // locates one kernel segment per C consecutive slices, and the W warps together cover
  // W / cpb batches at a time.
  // lane 0's turn state lives in shared memory (registers are at the 80-per-thread limit)
  StreamTurn& t = turns[warp];
  if (lane == 0) {
    t.Q = gnext;
    t.cs = t.cf = t.ce = 0;
    t.known_tail = 0;
    t.opened = 0;
  }
  // the lowest slice this warp has not issued yet (lane 0)
  auto next_G = [&]() -> uint64_t {
    return t.cs < t.ce ? t.G0 + t.cs : (t.Q / cpb) * ra.spb + (t.Q % cpb) * kStreamChunk;
  };
#if PASTA_STREAM_PROF
  unsigned long long p_fill = 0, p_wait = 0, p_n = 0, p_t0 = clock64(), p_turns = 0, p_sleeps = 0;
#endif
  // lane 0, any slice: open the next non-empty chunk if the current one is done, locate
  // the slice's kernel, tag it and issue its copy into ring slot `slot`. Returns 1 when
  // issued, 0 when its batch is not published yet (only if !block; with block it waits),
  // 2 when the stream has ended before it. The fast run [cs, cf) is set up for the
  // following slices. Warp turns: chunk Q = gw, gw + W, ... of the global chunk sequence
  // (batch Q / cpb, slices [C (Q % cpb), C (Q % cpb + 1)) of it).
  auto issue_slow = [&](uint32_t slot, bool block) -> int {
    while (t.cs == t.ce) {
      const uint64_t b = t.Q / cpb, c0 = (t.Q % cpb) * kStreamChunk;
      while (t.known_tail <= b) {
        t.known_tail = ld_acquire_u64(&ra.ctl->tail);  // orders the descriptor loads below
        if (t.known_tail > b) break;
        if (ld_acquire_u64(&ra.ctl->end) <= b) return 2;
        if (!block) return 0;
        front[warp] = b * ra.spb + c0;  // nothing in flight: the warp's lowest unread slice
        __nanosleep(200);
#if PASTA_STREAM_PROF
        ++p_sleeps;
#endif
      }
#if PASTA_STREAM_PROF
      ++p_turns;
#endif
      // the 32-byte descriptor in two independent 16-byte loads (L2: written by copies)
      const ulonglong2* d = reinterpret_cast<const ulonglong2*>(ra.ring + (b % ra.slots));
      const ulonglong2 d0 = __ldcg(d), d1 = __ldcg(d + 1);
      t.Q += W;
      const uint64_t nsl = (d0.y + kSlice - 1) / kSlice;
      if (c0 >= nsl) continue;  // past the end of a short batch
      if (c0 == 0 && d0.y) red_add_u64(args.totals + 0, d0.y);  // the batch's records, once
      t.G0 = b * ra.spb;
      t.cs = (uint32_t)c0;
      t.ce = (uint32_t)(c0 + kStreamChunk < nsl ? c0 + kStreamChunk : nsl);
      t.rec = reinterpret_cast<const uint64_t*>(d0.x);
      t.n = d0.y;
      t.koffs = reinterpret_cast<const uint64_t*>(d1.x);
      t.nk = (uint32_t)d1.y;
      t.k0 = (uint32_t)(d1.y >> 32);
      t.kl = 0;
      t.kend = ~0ull;
      if (kRows && t.koffs != nullptr && t.nk > 1) {
        t.kl = kernel_of(t.koffs, t.nk, (uint64_t)t.cs * kSlice);
        t.kend = t.kl + 1 < t.nk ? __ldg(t.koffs + t.kl + 1) : ~0ull;
      }
      const uint32_t e = t.opened++ & (kMaxStages - 1);
      t.eidx = e;
      ChunkEntry& ce = ents[e];
      ce.koffs = t.koffs;
      ce.n = t.n;
      ce.G0 = t.G0;
      ce.nk = t.nk;
      ce.k0 = t.k0;
    }
    const uint32_t sl = t.cs++;
    const uint64_t r_lo = (uint64_t)sl * kSlice;
    while (kRows && t.kend <= r_lo) {  // a kernel boundary since the last slice (rare)
      ++t.kl;
      t.kend = t.kl + 1 < t.nk ? __ldg(t.koffs + t.kl + 1) : ~0ull;
    }
    const uint64_t left = t.n - r_lo;
    const uint32_t valid = left < (uint64_t)kSlice ? (uint32_t)left : (uint32_t)kSlice;
    const bool fast = valid == (uint32_t)kSlice && (!kRows || t.kend - r_lo >= (uint64_t)kSlice);
    t.krow = t.k0 + t.kl;
    // the fast run after this slice: full slices inside kernel kl and inside the chunk
    {
      uint64_t f = t.ce;
      const uint64_t nfull = t.n / kSlice;
      if (nfull < f) f = nfull;
      if (kRows && t.kend != ~0ull && t.kend / kSlice < f) f = t.kend / kSlice;
      t.cf = f > t.cs ? (uint32_t)f : t.cs;
    }
    PASTA_DCHECK(slot < (uint32_t)stages && sl < t.ce && r_lo < t.n && t.eidx < 8u && t.kl < t.nk);
    SlotTag tg;
    tg.G = t.G0 + sl;
    tg.krow = t.krow;
    tg.meta = t.eidx | (fast ? kTagFast : 0u);
    tags[slot] = tg;
    mbar_arrive_expect_tx_u32(bar_u32 + 8u * slot, valid * 8u);
    tma_load_1d_u32(ring_u32 + slot * kSliceBytes, t.rec + r_lo, valid * 8u, bar_u32 + 8u * slot, pol);
    return 1;
  };
  // lane 0: the next slice into `slot`: the fast run (full slice, same kernel, same
  // chunk) or issue_slow
  // (shared-memory addresses as 32-bit offsets: no generic-to-shared conversion per slice)
  const uint32_t t_u32 = smem_u32(&t);
  const uint32_t tag_u32 = smem_u32(tags);
  auto issue = [&](uint32_t slot, bool block) -> int {
    const ulonglong2 h0 = lds128_o(t_u32);  // rec | cs, cf
    const uint32_t cs = (uint32_t)h0.y;
    if (cs < (uint32_t)(h0.y >> 32)) {
      PASTA_DCHECK(slot < (uint32_t)stages && cs < t.ce && (uint64_t)(cs + 1) * kSlice <= t.n && t.eidx < 8u);
      sts32_o(t_u32 + 8u, cs + 1);
      const ulonglong2 h1 = lds128_o(t_u32 + 16u);  // G0 | krow, eidx
      sts128_o(tag_u32 + 16u * slot, h1.x + cs, h1.y | ((uint64_t)kTagFast << 32));
      mbar_arrive_expect_tx_u32(bar_u32 + 8u * slot, kSliceBytes);
      tma_load_1d_u32(ring_u32 + slot * kSliceBytes, reinterpret_cast<const uint64_t*>(h0.x) + (uint64_t)cs * kSlice,
                      kSliceBytes, bar_u32 + 8u * slot, pol);
      return 1;
    }
    return issue_slow(slot, block);
  };

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
  o.hot = nullptr;
  o.P = args.P;
  o.wk = 1;
  o.wk_magic = 0;
  o.tids = nullptr;
  o.tcounts = nullptr;
  o.ktc = nullptr;
  o.max_tids = 0;
  o.cache = 0u;

  OwnCache oc;
  oc.olo = 1;
  oc.ospan = 0;
  oc.own = A;
  Ival cur = lookup<kBig>(oc, 0ull, c);
  WarpAcc w;
  w.page = kOOW - 1;
  w.own = A;
  w.pcnt = 0;
  w.ocnt = 0;
  LaneAcc& la = reinterpret_cast<LaneAcc*>(sm2 + ring_bytes(stages) + kBarBytes)[threadIdx.x];
  la.own = A;
  la.ocnt = 0;
  la.kbit = kOOW;
  uint32_t k = 0xFFFFFFFFu;  // kernel row of the warp's accumulators (none yet)

  // The warp's slots form a FIFO (filled at `tail`, consumed at `head`): it fills every
  // free slot whose batch is published without waiting, and waits for a publication only
  // when nothing is in flight -- a warp must never sit on a loaded slice while it waits
  // for a later batch (the producer may be waiting for that slice to be read).
  uint32_t head = 0, tail_slot = 0, inflight = 0, phases = 0;  // phases: bit i = parity of slot i
  uint32_t nit = 0;
  bool ended = false;

  for (;;) {
    int r = 1;
#if PASTA_STREAM_PROF
    const unsigned long long q0 = clock64();
#endif
    if (lane == 0) {
      while (!ended && inflight < (uint32_t)stages) {
        r = issue(tail_slot, inflight == 0);
        if (r != 1) break;
        tail_slot = tail_slot + 1 == (uint32_t)stages ? 0 : tail_slot + 1;
        ++inflight;
      }
      if (r == 2) ended = true;
      // the warp's lowest unread slice, for the monitor; refreshed every 8 slices (a stale,
      // lower value only delays the producer; a warp about to wait sets it in issue())
      if ((++nit & 7u) == 0 || inflight == 0)
        front[warp] = inflight ? lds128_o(tag_u32 + 16u * head).x : (ended ? ~0ull : next_G());
    }
    inflight = __shfl_sync(kFull, inflight, 0);
    __syncwarp();
    if (inflight == 0) break;  // the stream ended and everything this warp took is done
    const uint32_t slot = head;
    SlotTag tg;  // written by lane 0 before the __syncwarp above
    {
      const ulonglong2 v = lds128_o(tag_u32 + 16u * slot);
      tg.G = v.x;
      tg.krow = (uint32_t)v.y;
      tg.meta = (uint32_t)(v.y >> 32);
    }
#if PASTA_STREAM_PROF
    const unsigned long long q1 = clock64();
#endif
    mbar_wait_u32(bar_u32 + 8u * slot, (phases >> slot) & 1u);
    phases ^= 1u << slot;
#if PASTA_STREAM_PROF
    const unsigned long long q2 = clock64();
    p_fill += q1 - q0;
    p_wait += q2 - q1;
    ++p_n;
#endif
    uint64_t a[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const ulonglong2 v = lds128(ring_u32 + slot * kSliceBytes + 16u * lane + 512u * i);
      a[2 * i] = v.x;
      a[2 * i + 1] = v.y;
    }
    if (kRows && tg.krow != k) {  // the slice starts in another kernel row than the warp's run
      if (k != 0xFFFFFFFFu) warp_flush<kRows, kPages>(w, la, o, k, lane);
      k = tg.krow;
    }
    const uint32_t sa = ring_u32 + slot * kSliceBytes;
    if (tg.meta & kTagFast) {
      process_full<kBig, kRows, kPages>(a, sa, cur, oc, la, w, c, o, kRows ? k : 0u, lane);
    } else {
      // a partial slice or one holding a kernel boundary: segments as the scan does
      const ChunkEntry e = ents[tg.meta & 7u];
      const uint64_t r_lo = (tg.G - e.G0) * kSlice;
      PASTA_DCHECK(tg.G >= e.G0 && r_lo < e.n && tg.krow >= e.k0 && tg.krow - e.k0 < e.nk);
      const uint64_t left = e.n - r_lo;
      const uint32_t valid = left < (uint64_t)kSlice ? (uint32_t)left : (uint32_t)kSlice;
      uint32_t kl = tg.krow - e.k0;
      uint64_t kend = (kRows && kl + 1 < e.nk) ? __ldg(e.koffs + kl + 1) : ~0ull;
      uint32_t r0 = 0;
      for (;;) {
        uint32_t r1 = valid;
        if (kRows && kend - r_lo < (uint64_t)r1) r1 = (uint32_t)(kend - r_lo);
        uint32_t vm = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t pos = 64u * (i >> 1) + 2u * lane + (i & 1);
          if (pos >= r0 && pos < r1) vm |= 1u << i;
        }
        process_lane<kBig, kRows, kPages>(a, vm, oc, la, w, c, o, kRows ? k : 0u, lane);
        r0 = r1;
        if (r0 >= valid) break;
        // the next kernel of the batch starts inside this slice
        warp_flush<kRows, kPages>(w, la, o, k, lane);
        ++kl;
        while (kl + 1 < e.nk && __ldg(e.koffs + kl + 1) <= r_lo + r0) ++kl;
        kend = kl + 1 < e.nk ? __ldg(e.koffs + kl + 1) : ~0ull;
        k = e.k0 + kl;
      }
    }
    __syncwarp();
    head = head + 1 == (uint32_t)stages ? 0 : head + 1;
    --inflight;
  }
  if (k != 0xFFFFFFFFu || !kRows) warp_flush<kRows, kPages>(w, la, o, kRows ? k : 0u, lane);
  if (lane == 0) front[warp] = ~0ull;
#if PASTA_STREAM_PROF
  if (lane == 0 && ra.prof) {
    unsigned long long* pr = ra.prof + 8ull * (blockIdx.x * kStreamData + warp);
    pr[0] = p_fill;
    pr[1] = p_wait;
    pr[2] = clock64() - p_t0;
    pr[3] = p_n;
    pr[4] = p_turns;
    pr[5] = p_sleeps;
  }
#endif
}

int stream_smem_bytes(uint32_t A, bool big, int* stages_out) {
  const long extra = (long)kWarps * kMaxStages * kSlotInfoBytes + kFrontBytes + kTurnBytes - kPfBytes;
  int st = stages_for(A, big, extra);
  if (st > 4) st = 4;
  *stages_out = st;
  return kStreamHead + ring_bytes(st) + kBarBytes + kLaBytes + (big ? 0 : (int)(16ull * A));
}

template <bool kBig, bool kRows, int kPages>
cudaError_t launch_stream_variant(const StreamArgs& a0, cudaStream_t st, int* ctas) {
  StreamArgs a = a0;
  a.cpb = (a.spb + kStreamChunk - 1) / kStreamChunk;
  int stages = 0;
  const int smem = stream_smem_bytes(a.s.A, kBig, &stages);
  auto fn = stream_kernel<kBig, kRows, kPages>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, nb = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kStreamThreads, smem);
  if (e != cudaSuccess) return e;
  int grid = sms * (nb < 1 ? 1 : (nb > 1 ? 1 : nb));
  if (grid > kStreamMaxCtas) grid = kStreamMaxCtas;
  *ctas = grid;
  void* args[] = {(void*)&a, (void*)&stages};
  // cooperative: every CTA is resident (a CTA that never ran could never report progress)
  return cudaLaunchCooperativeKernel((void*)fn, dim3(grid), dim3(kStreamThreads), args, smem, st);
}


// ------------------------------------------------------------------------------------
// Rich 16-byte records (NEXT f4; R21-R24). Same per-warp TMA pipeline over
// 2 KiB slices (128 records; lane l reads records l, l+32, l+64, l+96 with LDS.128).
// A record is dropped (and counted) if its grid id is outside the window or it is a
// shared-space access; the rest are attributed like 8-byte records of kernel row
// grid_id - grid_lo, with write counts and byte weights. Tier RC takes a full slice
// whose records belong to at most two kernels, both in the window (one per slice in a
// serial trace, two where a concurrent kernel's records interleave): packed per-interval
// sums (count, writes, bytes in one u32) against A = interval of the first record and
// B = of the last, two to four warp reductions, warp-uniform run accumulators (page
// run: count, writes; owner run: count, writes, bytes, kernel-row share). Any other
// slice goes to a leader loop that takes one grid id at a time with the same A / B
// classification. Records outside A and B go straight to L2.
// ------------------------------------------------------------------------------------
constexpr int kRSlice = 128;
#ifndef PASTA_RICH_BRANCHLESS
#define PASTA_RICH_BRANCHLESS 0  // tier RC per-record classification with selects (A/B: slower, DESIGN 3.5)
#endif
#ifndef PASTA_RICH_WARPS
#define PASTA_RICH_WARPS 24  // warps per CTA of the rich scan (A/B: 12-24 warps, more is faster)
#endif
constexpr int kRWarps = PASTA_RICH_WARPS;
constexpr int kRThreads = kRWarps * 32;
constexpr int kRBarBytes = kRWarps * kMaxStages * 8;
constexpr int kRSlotBytes = kRWarps * 16;  // per-warp second-kernel row run {own, k, count, -}
__host__ __device__ constexpr int rich_ring_bytes(int stages) { return kRWarps * stages * (int)kSliceBytes; }
int rich_stages(uint32_t A, bool big) {
  const long table = big ? 0 : 16l * A;
  long st = ((long)kSmemLimit - kRBarBytes - kRSlotBytes - table) / rich_ring_bytes(1);
  return (int)(st > kMaxStages ? kMaxStages : st);
}

struct RichOut {
  uint64_t* page_counts;
  uint64_t* page_writes;
  uint64_t* alloc_counts;
  uint64_t* alloc_writes;
  uint64_t* alloc_bytes;
  uint64_t* totals;
  uint64_t* kac;
  uint64_t* kstats;
  const uint32_t* ids;
  uint64_t max_ids;
  uint32_t A;
};

__device__ __forceinline__ void rich_page(const RichOut& o, uint32_t page, uint64_t c, uint64_t w) {
  if (c == 0) return;
  if (page == kOOW) {
    red_add_u64(o.totals + 2, c);
  } else {
    red_add_u64(o.page_counts + page, c);
    if (w && o.page_writes) red_add_u64(o.page_writes + page, w);
  }
}

template <bool kRows>
__device__ __forceinline__ void rich_owner(const RichOut& o, uint32_t own, uint64_t c, uint64_t w, uint64_t b,
                                           uint32_t k) {
  if (c == 0) return;
  if (own < o.A) {
    const uint32_t id = __ldg(o.ids + own);
    red_add_u64(o.alloc_counts + id, c);
    if (w && o.alloc_writes) red_add_u64(o.alloc_writes + id, w);
    if (o.alloc_bytes) red_add_u64(o.alloc_bytes + id, b);
    if (kRows) {
      red_add_u64(o.kac + (uint64_t)k * o.max_ids + id, c);
      if (o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 0, c);
    }
  } else {
    red_add_u64(o.totals + 1, c);
    if (kRows && o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 1, c);
  }
}

// Owner run whose kernel-row share (kc of its c records, kernel k) differs from c:
// the alloc statistics take all c records, the kernel row only kc.
template <bool kRows>
__device__ __forceinline__ void rich_owner_split(const RichOut& o, uint32_t own, uint64_t c, uint64_t w, uint64_t b,
                                                 uint64_t kc, uint32_t k) {
  if (c == 0) return;
  if (own < o.A) {
    const uint32_t id = __ldg(o.ids + own);
    red_add_u64(o.alloc_counts + id, c);
    if (w && o.alloc_writes) red_add_u64(o.alloc_writes + id, w);
    if (o.alloc_bytes) red_add_u64(o.alloc_bytes + id, b);
    if (kRows && kc) {
      red_add_u64(o.kac + (uint64_t)k * o.max_ids + id, kc);
      if (o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 0, kc);
    }
  } else {
    red_add_u64(o.totals + 1, c);
    if (kRows && kc && o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 1, kc);
  }
}

// c records' kernel-row count only (their alloc statistics went with a run).
__device__ __forceinline__ void rich_rows(const RichOut& o, uint32_t own, uint64_t c, uint32_t k) {
  if (own < o.A) {
    red_add_u64(o.kac + (uint64_t)k * o.max_ids + __ldg(o.ids + own), c);
    if (o.kstats) red_add_u64(o.kstats + (uint64_t)k * 4 + 0, c);
  } else if (o.kstats) {
    red_add_u64(o.kstats + (uint64_t)k * 4 + 1, c);
  }
}

// Second-kernel row counts of tier RC (one lane): a run {own, k, count} in the warp's
// shared-memory slot, sent to L2 when the owner or the kernel changes (registers are
// at the 80-per-thread limit of 24 warps, so the run is not kept in registers).
__device__ __forceinline__ void rich_rows_run(const RichOut& o, uint4* slot, uint32_t own, uint32_t k, uint32_t c) {
  uint4 s = *slot;
  if (s.x == own && s.y == k) {
    s.z += c;
  } else {
    if (s.z) rich_rows(o, s.x, s.z, s.y);
    s = make_uint4(own, k, c, 0u);
  }
  *slot = s;
}

struct RichAcc {  // warp-uniform run accumulators
  uint32_t page, pcnt, pw;
  uint32_t own, ocnt, ow, okc;  // okc: records of the run counted in kernel row k
  uint64_t ob;
};

template <bool kRows>
__device__ __forceinline__ void rich_flush(RichAcc& r, const RichOut& o, uint32_t k, uint32_t lane) {
  if (lane == 0) {
    rich_page(o, r.page, r.pcnt, r.pw);
    rich_owner_split<kRows>(o, r.own, r.ocnt, r.ow, r.ob, r.okc, k);
  }
  r.pcnt = r.pw = r.ocnt = r.ow = r.okc = 0;
  r.ob = 0;
}

template <bool kRows>
__device__ __forceinline__ void rich_add(RichAcc& r, const RichOut& o, const Ival& I, uint32_t c, uint32_t w,
                                         uint32_t b, uint32_t kc, uint32_t k, uint32_t lane) {
  if (I.page != r.page) {
    if (lane == 0) rich_page(o, r.page, r.pcnt, r.pw);
    r.page = I.page;
    r.pcnt = r.pw = 0;
  }
  r.pcnt += c;
  r.pw += w;
  if (I.own != r.own) {
    if (lane == 0) rich_owner_split<kRows>(o, r.own, r.ocnt, r.ow, r.ob, r.okc, k);
    r.own = I.own;
    r.ocnt = r.ow = r.okc = 0;
    r.ob = 0;
  }
  r.ocnt += c;
  r.ow += w;
  r.ob += b;
  r.okc += kc;
}

template <bool kBig, bool kRows>
__global__ void __launch_bounds__(kRThreads, 1) rich_kernel(const RichArgs args, const int stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + rich_ring_bytes(stages));
  uint4* slot2 = reinterpret_cast<uint4*>(smem + rich_ring_bytes(stages) + kRBarBytes) + (threadIdx.x >> 5);
  uint64_t* sB = reinterpret_cast<uint64_t*>(smem + rich_ring_bytes(stages) + kRBarBytes + kRSlotBytes);
  const uint32_t A = args.A;
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nsl = (args.n + kRSlice - 1) / kRSlice;
  const uint32_t gwarp = blockIdx.x * kRWarps + warp;
  const uint32_t nwarp = gridDim.x * kRWarps;
  const uint64_t s0 = (uint64_t)gwarp * nsl / nwarp, s1 = (uint64_t)(gwarp + 1) * nsl / nwarp;
  const uint32_t nmy = (uint32_t)(s1 - s0);
  const uint32_t tail_valid = (uint32_t)(args.n - (nsl - 1) * kRSlice);
  const uint32_t ring_u32 = smem_u32(smem) + (uint32_t)(warp * stages) * kSliceBytes;
  const uint32_t bar_u32 = smem_u32(bars + warp * kMaxStages);
  if (lane == 0) {
    for (int j = 0; j < stages; ++j) mbar_init(bars + warp * kMaxStages + j, 1);
    fence_mbar_init();
    *slot2 = make_uint4(A, 0u, 0u, 0u);
  }
  if (!kBig)
    for (uint32_t i = threadIdx.x; i < 2 * A; i += kRThreads) sB[i] = args.bounds[i];
  __syncthreads();
  grid_dep_wait();  // the previous kernel's writes (records, outputs) are visible from here
  grid_dep_launch_dependents();  // as scan_kernel (after the wait): the next call's prologue may start
  const uint64_t pol = l2_evict_first_policy();
  // only the trace's last slice may be partial: the warp that owns it sees it at j = tail_j
  const uint32_t tail_j = (s1 == nsl && nmy) ? nmy - 1u : 0xFFFFFFFFu;
  auto slice_valid = [&](uint32_t j) -> uint32_t { return j == tail_j ? tail_valid : (uint32_t)kRSlice; };
  auto issue = [&](uint32_t j, uint32_t slot) {
    const uint32_t bytes = slice_valid(j) * 16u;
    mbar_arrive_expect_tx_u32(bar_u32 + 8u * slot, bytes);
    tma_load_1d_u32(ring_u32 + slot * kSliceBytes, args.rec + 2 * (s0 + j) * kRSlice, bytes, bar_u32 + 8u * slot,
                    pol);
  };
  if (lane == 0)
    for (uint32_t j = 0; j < (uint32_t)stages && j < nmy; ++j) issue(j, j);

  Ctx c;
  c.va_lo = args.va_lo;
  c.va_hi = args.va_hi;
  c.wbytes = args.va_hi - args.va_lo;
  c.s = args.page_shift;
  c.A = A;
  c.B = kBig ? args.bounds : sB;
  RichOut o;
  o.page_counts = args.page_counts;
  o.page_writes = args.page_writes;
  o.alloc_counts = args.alloc_counts;
  o.alloc_writes = args.alloc_writes;
  o.alloc_bytes = args.alloc_bytes;
  o.totals = args.totals;
  o.kac = args.kac;
  o.kstats = args.kstats;
  o.ids = args.ids;
  o.max_ids = args.max_ids;
  o.A = A;
  OwnCache oc;
  oc.olo = 1;
  oc.ospan = 0;
  oc.own = A;
  Ival cur = lookup<kBig>(oc, 0ull, c);
  RichAcc r;
  r.page = kOOW - 1;
  r.own = A;
  r.pcnt = r.pw = r.ocnt = r.ow = r.okc = 0;
  r.ob = 0;
  uint32_t k = 0;
  // per-lane totals: dropped by the grid window, dropped as shared, analyzed, writes, bytes
  uint32_t n_filt = 0, n_shared = 0, n_an = 0, n_wr = 0;
  uint64_t n_bytes = 0;
  uint32_t u_an = 0, u_wr = 0, u_sh = 0;  // warp-uniform totals of tier-RC slices
  uint64_t u_bytes = 0;

  uint32_t slot = 0, phase = 0;
  for (uint32_t j = 0; j < nmy; ++j) {
    const uint32_t sa = ring_u32 + slot * kSliceBytes;
    mbar_wait_u32(bar_u32 + 8u * slot, phase);
    const uint32_t valid = slice_valid(j);
    uint64_t a[4], m[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const ulonglong2 v = lds128(sa + 16u * (32u * i + lane));
      a[i] = v.x;
      m[i] = v.y;
    }
    __syncwarp();
    if (lane == 0 && j + stages < nmy) issue(j + stages, slot);
    if (++slot == (uint32_t)stages) {
      slot = 0;
      phase ^= 1u;
    }
    const uint64_t m0 = __shfl_sync(kFull, m[0], 0);
    const uint32_t g = (uint32_t)m0;
    const uint32_t kg = g - args.grid_lo;
    // Tier RC: all 128 records valid, of lane 0's kernel g or (concurrent kernels, with
    // kernel rows) of one other kernel g2, both inside the grid window; shared-space
    // records (dropped, R22) may be among them. Per analyzed record h = size_bytes |
    // is_write << 16 | 1 << 24: a warp sum holds up to 128 * 128 bytes in bits 0-15, 128
    // writes in bits 16-23 and 128 records in bits 24-31. Two warp reductions (interval
    // A and all), a third when some record is in neither A nor B = the interval of the
    // slice's last record, a fourth for g2's kernel-row counts in A (bits 0-7) and B
    // (bits 8-15). Page and alloc statistics do not depend on the kernel.
    auto tier_rc = [&](auto two_t, const uint32_t mis, const uint32_t km, const uint32_t k2) {
      constexpr bool kTwo = decltype(two_t)::value;
      if (kRows && km != k) {
        rich_flush<kRows>(r, o, k, lane);
        k = km;
      }
      const uint64_t a0 = __shfl_sync(kFull, a[0], 0);
      const uint64_t b0 = __shfl_sync(kFull, a[3], 31);
      Ival IA = cur;
      if (!inside(a0, IA)) IA = lookup<kBig>(oc, a0, c);
      Ival IB = IA;
      if (!inside(b0, IA)) IB = lookup<kBig>(oc, b0, c);
      cur = IB;
      uint32_t hA = 0, hT = 0, hR = 0, rest = 0, mAB = 0;
#if PASTA_RICH_BRANCHLESS
      // branch-free classification (selects, no per-record reconvergence blocks)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t hi = (uint32_t)(m[i] >> 32);
        const bool an = !(hi & 0x20000u);
        const uint32_t h = an ? (hi & 0x1FFFFu) + (1u << 24) : 0u;
        const bool inA = inside(a[i], IA);
        const bool inB = inside(a[i], IB);
        const bool rs = an & !inA & !inB;
        hT += h;
        hA += inA ? h : 0u;
        hR += rs ? h : 0u;
        rest |= (rs ? 1u : 0u) << i;
        if (kTwo && kRows) {
          const uint32_t mi = an ? (mis >> i) & 1u : 0u;
          mAB += inA ? mi : ((inB ? mi : 0u) << 8);
        }
      }
#else
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t hi = (uint32_t)(m[i] >> 32);
        if (!(hi & 0x20000u)) {
          const uint32_t h = (hi & 0x1FFFFu) + (1u << 24);
          hT += h;
          if (inside(a[i], IA)) {
            hA += h;
            if (kTwo && kRows) mAB += (mis >> i) & 1u;
          } else if (!inside(a[i], IB)) {
            rest |= 1u << i;
            hR += h;
          } else if (kTwo && kRows) {
            mAB += ((mis >> i) & 1u) << 8;
          }
        }
      }
#endif
      const bool any_rest = __any_sync(kFull, rest != 0);
      hA = __reduce_add_sync(kFull, hA);
      hT = __reduce_add_sync(kFull, hT);
      hR = any_rest ? __reduce_add_sync(kFull, hR) : 0u;
      if (kTwo && kRows) mAB = __reduce_add_sync(kFull, mAB);
      const uint32_t cA = hA >> 24, cT = hT >> 24, cB = cT - cA - (hR >> 24);
      const uint32_t bA = hA & 0xFFFFu, wA = (hA >> 16) & 0xFFu;
      const uint32_t bT = hT & 0xFFFFu, wT = (hT >> 16) & 0xFFu;
      if (cA) rich_add<kRows>(r, o, IA, cA, wA, bA, cA - (mAB & 0xFFu), km, lane);
      if (cB)
        rich_add<kRows>(r, o, IB, cB, wT - wA - ((hR >> 16) & 0xFFu), bT - bA - (hR & 0xFFFFu), cB - (mAB >> 8),
                        km, lane);
      if (kTwo && kRows) {
        if (lane == 0) {
          if (IA.own == IB.own) {
            if (mAB) rich_rows_run(o, slot2, IA.own, k2, (mAB & 0xFFu) + (mAB >> 8));
          } else {
            if (mAB & 0xFFu) rich_rows_run(o, slot2, IA.own, k2, mAB & 0xFFu);
            if (mAB >> 8) rich_rows_run(o, slot2, IB.own, k2, mAB >> 8);
          }
        }
      }
      if (any_rest) {
#pragma unroll 1
        while (rest) {
          const int i = __ffs(rest) - 1;
          rest &= rest - 1;
          const uint64_t x = pick4(a, i), mm = pick4(m, i);
          const Ival I = lookup<kBig>(oc, x, c);
          const uint64_t w = (mm >> 48) & 1u;
          rich_page(o, I.page, 1, w);
          rich_owner<kRows>(o, I.own, 1, w, (mm >> 32) & 0xFFFFu, (uint32_t)mm - args.grid_lo);
        }
      }
      u_an += cT;
      u_sh += (uint32_t)kRSlice - cT;
      u_wr += wT;
      u_bytes += bT;
    };
    if (valid == (uint32_t)kRSlice && kg <= args.grid_last) {
      uint32_t mis = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) mis |= ((uint32_t)m[i] != g ? 1u : 0u) << i;
      const unsigned mis_lanes = __ballot_sync(kFull, mis != 0);
      if (mis_lanes == 0) {
        tier_rc(std::false_type{}, 0u, kg, 0u);
        continue;
      }
      // the other kernel: the largest grid id among the records that are not g's (any
      // third id makes `bad` below)
      uint32_t gl = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) gl = max(gl, ((mis >> i) & 1u) ? (uint32_t)m[i] : 0u);
      const uint32_t g2 = __reduce_max_sync(kFull, gl);
      uint32_t bad = g2 - args.grid_lo > args.grid_last ? 1u : 0u;
#pragma unroll
      for (int i = 0; i < 4; ++i) bad |= (((mis >> i) & 1u) && (uint32_t)m[i] != g2) ? 1u : 0u;
      if (!__any_sync(kFull, bad != 0)) {
        // the run accumulators keep the current kernel when it is the other one here
        const uint32_t k2 = g2 - args.grid_lo;
        const bool sw = kRows && kg != k && k2 == k;
        tier_rc(std::true_type{}, sw ? ~mis & 0xFu : mis, sw ? k2 : kg, sw ? kg : k2);
        continue;
      }
    }
    uint32_t pend = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (32u * i + lane < valid) {
        const uint32_t g = (uint32_t)m[i];
        const bool inwin = g - args.grid_lo <= args.grid_last;
        const bool shared = (m[i] >> 49) & 1u;
        n_filt += inwin ? 0u : 1u;
        n_shared += (inwin && shared) ? 1u : 0u;
        if (inwin && !shared) {
          pend |= 1u << i;
          ++n_an;
          n_wr += (uint32_t)(m[i] >> 48) & 1u;
          n_bytes += (m[i] >> 32) & 0xFFFFu;
        }
      }
    }
    for (;;) {
      const unsigned any = __ballot_sync(kFull, pend != 0);
      if (any == 0) break;
      const int leader = __ffs(any) - 1;
      const int li = pend ? __ffs(pend) - 1 : 0;
      const uint64_t al = pick4(a, li), ml = pick4(m, li);
      const uint32_t g = (uint32_t)__shfl_sync(kFull, ml, leader);
      const uint64_t a0 = __shfl_sync(kFull, al, leader);
      uint32_t sel = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (((pend >> i) & 1u) && (uint32_t)m[i] == g) sel |= 1u << i;
      // the group's last record (highest slice position)
      const uint32_t mypos = sel ? 32u * (31u - __clz(sel)) + lane + 1u : 0u;
      const uint32_t last = __reduce_max_sync(kFull, mypos) - 1u;
      const uint64_t b0 = __shfl_sync(kFull, pick4(a, (int)(last >> 5)), last & 31u);
      const uint32_t kg = g - args.grid_lo;
      if (kRows && kg != k) {
        rich_flush<kRows>(r, o, k, lane);
        k = kg;
      }
      Ival IA = cur;
      if (!inside(a0, IA)) IA = lookup<kBig>(oc, a0, c);
      Ival IB = IA;
      if (!inside(b0, IA)) IB = lookup<kBig>(oc, b0, c);
      cur = IB;
      uint32_t cA = 0, wA = 0, bA = 0, cB = 0, wB = 0, bB = 0, rest = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if ((sel >> i) & 1u) {
          const uint32_t w = (uint32_t)(m[i] >> 48) & 1u, sz = (uint32_t)(m[i] >> 32) & 0xFFFFu;
          if (inside(a[i], IA)) {
            ++cA;
            wA += w;
            bA += sz;
          } else if (inside(a[i], IB)) {
            ++cB;
            wB += w;
            bB += sz;
          } else {
            rest |= 1u << i;
          }
        }
      }
      cA = __reduce_add_sync(kFull, cA);
      wA = __reduce_add_sync(kFull, wA);
      bA = __reduce_add_sync(kFull, bA);
      cB = __reduce_add_sync(kFull, cB);
      wB = __reduce_add_sync(kFull, wB);
      bB = __reduce_add_sync(kFull, bB);
      if (cA) rich_add<kRows>(r, o, IA, cA, wA, bA, cA, kg, lane);
      if (cB) rich_add<kRows>(r, o, IB, cB, wB, bB, cB, kg, lane);
      // records outside A and B: looked up one by one, straight to L2
#pragma unroll 1
      while (rest) {
        const int i = __ffs(rest) - 1;
        rest &= rest - 1;
        const uint64_t x = pick4(a, i), mm = pick4(m, i);
        const Ival I = lookup<kBig>(oc, x, c);
        const uint64_t w = (mm >> 48) & 1u;
        rich_page(o, I.page, 1, w);
        rich_owner<kRows>(o, I.own, 1, w, (mm >> 32) & 0xFFFFu, kg);
      }
      pend &= ~sel;
    }
  }
  rich_flush<kRows>(r, o, k, lane);
  if (kRows && lane == 0) {
    const uint4 s = *slot2;
    if (s.z) rich_rows(o, s.x, s.z, s.y);
  }
  // per-warp totals
  const uint32_t f = __reduce_add_sync(kFull, n_filt), sh = __reduce_add_sync(kFull, n_shared);
  const uint32_t an = __reduce_add_sync(kFull, n_an), wr = __reduce_add_sync(kFull, n_wr);
  const uint64_t by = warp_sum_u64(n_bytes);
  if (lane == 0) {
    if (f) red_add_u64(args.rich_totals + 0, f);
    if (sh + u_sh) red_add_u64(args.rich_totals + 1, (uint64_t)sh + u_sh);
    if (wr + u_wr) red_add_u64(args.rich_totals + 2, (uint64_t)wr + u_wr);
    if (by + u_bytes) red_add_u64(args.rich_totals + 3, by + u_bytes);
    if (an + u_an) red_add_u64(args.totals + 0, (uint64_t)an + u_an);
  }
}

template <bool kBig, bool kRows>
cudaError_t launch_rich_variant(const RichArgs& a, int grid, cudaStream_t st) {
  const int stages = rich_stages(a.A, kBig);
  const int smem = rich_ring_bytes(stages) + kRBarBytes + kRSlotBytes + (kBig ? 0 : (int)(16ull * a.A));
  auto fn = rich_kernel<kBig, kRows>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kRThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = PASTA_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, a, stages);
}

}  // namespace

int scan_warps() { return kWarps; }
int scan_permute_below() { return PASTA_IL_PERMUTE_BELOW; }

int scan_schedule(uint64_t nbody, int grid, uint32_t force, uint32_t A) {
  const uint64_t nsl = (nbody + kSlice - 1) / kSlice;
  const uint64_t nwarp = (uint64_t)grid * kWarps;
  if (force == PASTA_SCHED_CONTIGUOUS) return -1;
  if (force == PASTA_SCHED_INTERLEAVED) {
    // the largest chunk (<= PASTA_IL_LOG_CHUNK) that still gives every warp one; the
    // dynamic schedule needs chunks of >= 8 slices (a warp's refills run up to a ring
    // depth, <= 6 slices, ahead, and only the next chunk's id is known in advance)
    int lc = PASTA_IL_DYNAMIC ? 3 : 0;
    while (lc < PASTA_IL_LOG_CHUNK && (nsl >> (lc + 1)) >= nwarp) ++lc;
    return lc;
  }
  // a global-memory range table keeps its lookups cheap through each warp's locality:
  // medium launches stay contiguous there (S-manyranges: 0.78 contiguous vs 1.01 ms)
  const uint64_t min_chunks = scan_table_fits_smem(A) ? PASTA_IL_MIN_CHUNKS : 16;
  if (!PASTA_IL || (nsl >> PASTA_IL_LOG_CHUNK) < nwarp * min_chunks) return -1;
  // medium launches: smaller chunks (down to 2^PASTA_IL_LOG_CHUNK_MIN slices) so that every
  // warp still takes about 16, and the dynamic schedule's end spread (one chunk) shrinks
  int lc = PASTA_IL_LOG_CHUNK;
  while (lc > PASTA_IL_LOG_CHUNK_MIN && (nsl >> lc) < nwarp * 16) --lc;
  return lc;
}

// [chunk map: 16 B per chunk | 256 B: the dynamic schedule's chunk counter at offset 0]
size_t scan_scratch_bytes(uint64_t nbody, int log_ic) {
  if (log_ic < 0) return 256;
  const uint64_t nsl = (nbody + kSlice - 1) / kSlice;
  const uint64_t nch = (nsl + (1ull << log_ic) - 1) >> log_ic;
  return 16 * nch + 256;
}

extern "C" int pasta_debug_warp_times(unsigned long long* out, int n) {
#if PASTA_TRACE_TIMING
  return cudaMemcpyFromSymbol(out, g_warp_times, sizeof(unsigned long long) * n) == cudaSuccess ? n : -1;
#else
  (void)out;
  (void)n;
  return 0;
#endif
}

bool scan_table_fits_smem(uint32_t A) { return stages_for(A, false) >= kMinStages; }

int scan_smem_bytes(uint32_t A, bool big_table) {
  return ring_bytes(stages_for(A, big_table)) + kBarBytes + kLaBytes + kPfBytes + (big_table ? 0 : (int)(16ull * A));
}

cudaError_t launch_scan(const ScanArgs& a, int grid, cudaStream_t st, int* launches) {
  const bool big = !scan_table_fits_smem(a.A);
  const bool rows = a.kac != nullptr;  // per-kernel outputs all require kernel rows
  const bool fill = a.log_ic >= 0 && rows && a.n_kernels > 1 && a.nbody > 0;
  if (fill || (PASTA_IL_DYNAMIC && a.log_ic >= 0 && a.nbody > 0)) {
    const uint64_t nsl = (a.nbody + kSlice - 1) / kSlice;
    const uint64_t nch = (nsl + (1ull << a.log_ic) - 1) >> a.log_ic;
    chunk_kernel_map<<<fill ? (unsigned)((nch + 255) / 256) : 1u, 256, 0, st>>>(
        a, const_cast<ulonglong2*>(a.chunk_k), nch, fill ? 1 : 0);
    const cudaError_t e0 = cudaGetLastError();
    if (e0 != cudaSuccess) return e0;
    ++*launches;
  }
  ++*launches;
  const int mode = (a.kpb != nullptr ? 1 : 0) | (a.hot != nullptr ? 2 : 0);
  if (big) {
    if (!rows) return launch_variant<true, false, 0>(a, grid, st);
    switch (mode) {
      case 0: return launch_variant<true, true, 0>(a, grid, st);
      case 1: return launch_variant<true, true, 1>(a, grid, st);
      case 2: return launch_variant<true, true, 2>(a, grid, st);
      default: return launch_variant<true, true, 3>(a, grid, st);
    }
  }
  if (!rows) return launch_variant<false, false, 0>(a, grid, st);
  switch (mode) {
    case 0: return launch_variant<false, true, 0>(a, grid, st);
    case 1: return launch_variant<false, true, 1>(a, grid, st);
    case 2: return launch_variant<false, true, 2>(a, grid, st);
    default: return launch_variant<false, true, 3>(a, grid, st);
  }
}

cudaError_t launch_rich(const RichArgs& a, int grid, cudaStream_t st) {
  const bool big = !scan_table_fits_smem(a.A);
  const bool rows = a.kac != nullptr;
  if (big) return rows ? launch_rich_variant<true, true>(a, grid, st) : launch_rich_variant<true, false>(a, grid, st);
  return rows ? launch_rich_variant<false, true>(a, grid, st) : launch_rich_variant<false, false>(a, grid, st);
}

int rich_slice_records() { return kRSlice; }
int rich_warps() { return kRWarps; }

cudaError_t launch_stream_consumer(const StreamArgs& a, cudaStream_t st, int* ctas) {
  const bool big = !scan_table_fits_smem(a.s.A);
  const bool rows = a.s.kac != nullptr;
  const bool pages = a.s.kpb != nullptr;
  if (big) {
    if (!rows) return launch_stream_variant<true, false, 0>(a, st, ctas);
    return pages ? launch_stream_variant<true, true, 1>(a, st, ctas) : launch_stream_variant<true, true, 0>(a, st, ctas);
  }
  if (!rows) return launch_stream_variant<false, false, 0>(a, st, ctas);
  return pages ? launch_stream_variant<false, true, 1>(a, st, ctas) : launch_stream_variant<false, true, 0>(a, st, ctas);
}

cudaError_t launch_scan_extras(const ExtraArgs& a, cudaStream_t st) {
  scan_extras_kernel<<<1, 32, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace pasta
