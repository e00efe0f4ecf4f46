/* pasta.h -- C ABI of the B200-native PASTA trace-analysis hot path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, arxiv 2602.22103):
 *   "When a kernel is launched, a map from memory object to access count is
 *    transferred to the GPU. During execution, a profiling device function
 *    increments access count for each associated memory object upon each access.
 *    When the kernel completes, the access count map is copied back to the CPU,
 *    where objects with non-zero access counts are identified as part of the
 *    kernel's working set."
 *   working set = "the maximum memory footprint of any single kernel execution"
 *
 *   hotness "in the unit of 2MB virtual memory blocks"; hot blocks are prefetch /
 *   cudaMemAdvise candidates
 * Here the collected records sit in a device buffer ("the profiling library
 * records the instruction into a device buffer. A helper device function then
 * processes many of these events concurrently") and are reduced on the
 * device into: per-page, per-allocation and per-kernel histograms, the unique-page
 * bitmap with popcount, per-kernel footprints / working set, and the top-K hot
 * pages. The readings R1-R14 that fix what the paper leaves open are listed in
 * DESIGN.md ("Readings"); they are cited below as (Rn).
 *
 * Conventions for every call:
 *   - returns an int status: PASTA_OK (0) or a negative PASTA_E* code; never
 *     aborts, never throws, never prints;
 *   - argument validation is synchronous and happens before anything is enqueued;
 *     a failed call leaves the handle and every output unchanged;
 *   - device work is asynchronous on the handle's stream (pasta_open_params.stream);
 *     PASTA_ECUDA reports a launch or copy failure; asynchronous device faults
 *     surface at the next call or at pasta_sync;
 *   - "device pointer" = memory the handle's device can dereference (cudaMalloc /
 *     torch CUDA tensors; pinned host memory also qualifies). The caller owns
 *     records and outputs; the handle owns its range table and scratch.
 *   - a handle is not thread-safe; several handles per device are fine.
 *
 * Entry points (in this file's order): handle (pasta_trace_open / pasta_close /
 * pasta_strerror / pasta_sync), registration (pasta_register_alloc / _free,
 * pasta_register_tensor / _free, pasta_report_memory_usage), analysis (pasta_analyze
 * and pasta_analyze_batches for 8-byte records, pasta_analyze_rich for 16-byte records, pasta_finalize,
 * pasta_topk), multi-GPU merge (pasta_peer_reduce + pasta_enable_peer over peer
 * memory; pasta_bitmap_or + pasta_topk_merge after NCCL collectives), prefetch plans
 * (pasta_prefetch_plan) and timing (pasta_set_timing / pasta_get_timing /
 * pasta_reset_timing). Readings R15-R25 (tensor level, rich records, grid-id window,
 * signed sizes) are in DESIGN.md as well.
 */
#ifndef PASTA_H
#define PASTA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PASTA_OK = 0,
  PASTA_EINVAL = -1,    /* bad argument (null, zero size, misaligned window, ...) */
  PASTA_EOVERLAP = -2,  /* register_alloc intersects a live range (R4) */
  PASTA_ENOENT = -3,    /* register_free of a base that is not live */
  PASTA_ECAPACITY = -4, /* more than max_live live ranges or max_ids ids issued */
  PASTA_ECUDA = -5,     /* CUDA runtime error (launch, copy, allocation, async fault) */
  PASTA_ESTATE = -6,    /* call not valid in the handle's current state */
  PASTA_ENOMEM = -7     /* host allocation failed */
};

/* Indices into the totals[PASTA_TOTALS] output array (u64 each). */
enum {
  PASTA_T_RECORDS = 0,       /* += n per analyze call                                   */
  PASTA_T_UNATTRIBUTED = 1,  /* += records owned by no live range (R5)                  */
  PASTA_T_OUT_OF_WINDOW = 2, /* += records outside [va_lo, va_hi) (R8)                  */
  PASTA_T_UNIQUE_PAGES = 3,  /* = popcount(bitmap) (overwritten by finalize)            */
  PASTA_T_WS_OBJ = 4,        /* = max_k footprint[k] in bytes (overwritten; R11) */
  PASTA_T_UNTENSORED = 5,    /* += records in no live tensor (needs tensor_counts; R18) */
  PASTA_T_WS_TENSOR = 6,     /* = max_k tensor footprint[k] (overwritten; needs kernel_tensor_footprint) */
  PASTA_T_MAX_KERNEL = 7,    /* = MAX_MEM_REFERENCED_KERNEL (R24): kernel_row0 + the
                                kernel row with the most analyzed records, ties to the lowest
                                (overwritten by finalize when kernel_stats is given)      */
  PASTA_T_MAX_KERNEL_RECORDS = 8, /* = the analyzed records of that kernel (overwritten with
                                it). Slots 7-8 form one (index, records) pair: shards merge
                                it with pasta_peer_reduce(PASTA_PEER_ARGMAX), not by sum */
  PASTA_TOTALS = 9
};

/* Per-kernel stats row: kernel_stats[k * PASTA_KSTATS + i]. */
enum {
  PASTA_K_ATTRIBUTED = 0,   /* += records of kernel k owned by some live range          */
  PASTA_K_UNATTRIBUTED = 1, /* += records of kernel k owned by none                     */
  PASTA_K_FOOTPRINT = 2,    /* = sum of registered sizes of ids with count > 0  */
  PASTA_K_UNIQUE_PAGES = 3, /* = popcount of kernel k's page-bitmap row, 0 if absent    */
  PASTA_KSTATS = 4
};

typedef struct pasta_trace pasta_trace; /* opaque; one per (process, device, window) */

typedef struct {
  int32_t device;     /* CUDA device ordinal the handle binds to                        */
  uint32_t max_live;  /* range-table capacity (simultaneously live ranges), >= 1        */
  uint32_t max_ids;   /* ids ever issued by this handle (= bins of alloc_counts), >= 1  */
  uint32_t flags;     /* 0, or one PASTA_SCHED_* schedule override (tuning / testing)   */
  uint64_t va_lo;     /* page window [va_lo, va_hi): multiples of 4 KiB, va_lo < va_hi  */
  uint64_t va_hi;
  uintptr_t stream;   /* cudaStream_t for all device work (0 = legacy default stream)   */
  uint64_t host_chunk_bytes; /* staging chunk for PASTA_REC_HOST (0 = 256 MiB)          */
  uint32_t max_live_tensors; /* tensor level (NEXT f3, R18): live tensors, 0 = no tensor level */
  uint32_t max_tensor_ids;   /* tensor ids ever issued (= bins of tensor_counts)            */
} pasta_open_params;

/* Scan schedule (pasta_open_params.flags). By default a launch over few records per
 * warp gives each warp one contiguous range of 2 KiB slices, and a longer launch
 * (>= ~0.23e9 records on 148 SMs; >= ~0.9e9 when the range table is too large for shared
 * memory) hands out chunks of 64 slices dynamically: each warp's first chunk is fixed,
 * later ones come from a device counter, so no warp straggles behind an expensive region
 * of the trace. Results are identical under every schedule; the flags force one (for
 * tests and tuning; forced interleaving uses chunks of 8-64 slices). */
enum { PASTA_SCHED_CONTIGUOUS = 1u, PASTA_SCHED_INTERLEAVED = 2u };

/* Input records. By default both arrays are DEVICE memory, read-only, never copied
 * to the host. With PASTA_REC_HOST they are HOST memory (pinned for full speed):
 * the library streams them to the device in chunks on an internal copy stream
 * overlapped with the scan (the end-to-end path); the raw trace still never comes
 * back. Record j is the 8-byte address of one access (R1, R2); segment k of the
 * CSR offsets is kernel launch k (R12). */
typedef struct {
  const uint64_t* addr;           /* [n] records, 8-byte aligned                        */
  const uint64_t* kernel_offsets; /* [n_kernels+1], o[0]=0, o[n_kernels]=n, non-decreasing;
                                     NULL => one kernel. Device memory is not checked
                                     (bad offsets mis-attribute, never write out of
                                     bounds); host offsets are checked (EINVAL).       */
  uint32_t n_kernels;
  uint32_t flags;                 /* PASTA_REC_HOST | PASTA_REC_STABLE */
} pasta_records;

/* PASTA_REC_STABLE (device records only): the records and kernel offsets were complete
 * before the previous kernel on the handle's stream started (that kernel does not
 * write them), so the scan may begin loading them while that kernel is still running.
 * Consecutive pasta_analyze scans on a stream are programmatic dependent launches:
 * each one waits for its predecessor's completion (griddepcontrol.wait) before it
 * writes any output, and with this flag only after issuing its first record loads —
 * the streaming mode's per-call latency (NEXT f2). Without the flag every access to
 * global data follows the wait. The scan triggers its dependents right after that wait
 * (a chained scan, below, at entry), so a caller's own kernel launched as a
 * programmatic dependent right after it must griddepcontrol.wait
 * (cudaGridDependencySynchronize) before reading the outputs; ordinary launches, copies
 * and events after the call are ordered as usual. */
/* PASTA_REC_CHAINED (device records; implies PASTA_REC_STABLE): in addition, the
 * previous kernel on the handle's stream is a pasta_analyze scan of this handle into
 * the same outputs, with no other work in between. Its REDs commute with this call's,
 * so this scan does not wait for it at all before working; it waits only before it
 * exits, which keeps completion in stream order (a reader enqueued after the last call
 * of a chain sees every call's counts). The first call of a chain (e.g. after zeroing
 * the outputs) must not carry the flag: it waits for the zeroing before it lets any
 * chained successor launch. */
enum { PASTA_REC_HOST = 1u, PASTA_REC_STABLE = 2u, PASTA_REC_CHAINED = 4u };

/* Outputs: caller-owned DEVICE memory (e.g. torch int64 tensors viewed as u64).
 * Counts ACCUMULATE (+=) across calls, so a long trace can be analyzed in batches
 * and shards can be merged by summation. P = (va_hi-va_lo) >> s,
 * W = ceil(P/64). */
typedef struct {
  uint64_t* page_counts;         /* [P]           required  += (R7, R8)                */
  uint64_t* alloc_counts;        /* [max_ids]     required  +=, indexed by alloc id   */
  uint64_t* totals;              /* [PASTA_TOTALS] required (see PASTA_T_*)                    */
  uint64_t* page_bitmap;         /* [W] optional, overwritten: bit p%64 of word p/64 = count>0 (R14) */
  uint64_t* kernel_alloc_counts; /* [n_kernels*max_ids] optional, row-major +=   */
  uint64_t* kernel_stats;        /* [n_kernels*PASTA_KSTATS] optional; needs kernel_alloc_counts */
  uint64_t* kernel_page_bitmap;  /* [n_kernels*W] optional, OR-accumulated; needs kernel_alloc_counts */
  uint32_t flags;                /* PASTA_NO_FINALIZE */
  uint32_t window_kernels;       /* kernels per hotness window (>= 1 when hotness != NULL) */
  uint64_t* hotness;             /* [ceil(n_kernels/window_kernels) * P] optional +=, needs
                                    kernel_alloc_counts: time-windowed page hotness, row
                                    w = kernel k / window_kernels (NEXT f1)   */
  /* Tensor level (NEXT f3, R18; handles opened with max_tensor_ids > 0). A record
   * counts for its object (above) and for the live tensor holding it, else in
   * totals[UNTENSORED]. */
  uint64_t* tensor_counts;           /* [max_tensor_ids] optional +=, indexed by tensor id  */
  uint64_t* kernel_tensor_counts;    /* [n_kernels*max_tensor_ids] optional +=; needs
                                        tensor_counts and kernel_alloc_counts               */
  uint64_t* kernel_tensor_footprint; /* [n_kernels] optional, overwritten by finalize: sum
                                        of registered tensor sizes with a count in kernel k;
                                        totals[WS_TENSOR] = max; needs kernel_tensor_counts */
  uint64_t kernel_row0;              /* global index of kernel row 0 of these outputs (a
                                        shard's first kernel; 0 for a whole trace): finalize
                                        reports totals[MAX_KERNEL] as kernel_row0 + row, so
                                        shards' (index, records) pairs merge by ARGMAX    */
} pasta_histograms;

/* Skip the finalize step in pasta_analyze (bitmap, unique pages, footprints, WS);
 * call pasta_finalize once at the end instead (streaming and multi-GPU merge). */
enum { PASTA_NO_FINALIZE = 1u };

/* Open a handle: binds to params->device, allocates the device range table for
 * max_live ranges and max_ids ids. *out is set only on success. */
int pasta_trace_open(const pasta_open_params* params, pasta_trace** out);

/* Register a live allocation [base, base+size) (R3: half-open). size > 0 and
 * base + size <= 2^64 - 1, else EINVAL; intersecting a live range => EOVERLAP
 * (adjacent ranges are legal); ids are issued 0, 1, 2, ... and never reused; more
 * than max_live live ranges or max_ids ids => ECAPACITY. Takes effect for the
 * pasta_analyze calls enqueued after it (snapshot semantics, R13: "When a kernel is
 * launched, a map ... is transferred to the GPU"). */
int pasta_register_alloc(pasta_trace* h, uint64_t base, uint64_t size, uint32_t* out_id);

/* Remove the live range whose base is exactly `base` (ENOENT otherwise). Its id's
 * counts stay addressable; the id is never reissued. */
int pasta_register_free(pasta_trace* h, uint64_t base);

/* Tensor level (NEXT f3; R18, R19). Register a live tensor [base, base+size)
 * inside a live object ("[address, address+size) lies within the containing
 * object"): size > 0, the range inside one live object, else EINVAL (also when the
 * handle has no tensor level); intersecting a live tensor => EOVERLAP (adjacent is
 * legal); tensor ids 0, 1, 2, ... never reused; more than max_live_tensors live or
 * max_tensor_ids issued => ECAPACITY. Snapshot semantics as pasta_register_alloc.
 * pasta_register_free of an object also ends every live tensor inside it (R19). */
int pasta_register_tensor(pasta_trace* h, uint64_t base, uint64_t size, uint32_t* out_tid);

/* Remove the live tensor whose base is exactly `base` (ENOENT otherwise). */
int pasta_register_tensor_free(pasta_trace* h, uint64_t base);

/* Signed-size registration in the convention of PyTorch's allocator callback
 * c10::reportMemoryUsage ("function hooks and callbacks (e.g.
 * c10::reportMemoryUsage ...)"; SPEC S:121-124 RawEventRMX: "a single signed size
 * (negative = release)", normalized to positive sizes). The event goes to the
 * tensor level if the handle has one (max_tensor_ids > 0, R18), else to the object
 * level (R6). delta > 0: register [ptr, ptr + delta) exactly as pasta_register_tensor /
 * pasta_register_alloc (same errors), *out_id (may be NULL) = the new id. delta < 0:
 * release the live range whose base is ptr, which must have size -delta (EINVAL
 * otherwise, nothing released; ENOENT if no live range starts at ptr); *out_id = its
 * id. delta == 0 or INT64_MIN: EINVAL. */
int pasta_report_memory_usage(pasta_trace* h, uint64_t ptr, int64_t delta, uint32_t* out_id);

/* Analyze n records at page granularity 2^page_shift (12 <= page_shift <= 30;
 * va_lo and va_hi must be multiples of 2^page_shift and P < 2^32). Steps, all on the
 * device in one scan of the records (S1-S3 of DESIGN.md section 1):
 *   owner(a) = the live range holding a, else unattributed          (R2-R5)
 *   page_counts[(a - va_lo) >> s] += 1 if va_lo <= a < va_hi, else out_of_window
 *   alloc_counts[id(owner)] += 1; kernel rows / stats per segment
 *   kernel_page_bitmap[k] |= bit(page)
 * then, unless PASTA_NO_FINALIZE, pasta_finalize. n = 0 is legal (finalize only). */
int pasta_analyze(pasta_trace* h, const pasta_records* trace, uint64_t n, uint32_t page_shift,
                  pasta_histograms* out);

/* Streaming submission (NEXT f2; "a device buffer"): `count` batches, each
 * analyzed exactly as pasta_analyze(h, &b[i].trace, b[i].n, page_shift, &b[i].out), in
 * order, with the host-side per-call overhead of one C loop instead of one foreign call
 * per batch. A batch's outputs usually point into one shared set of histograms (per-
 * kernel rows offset to the batch's first kernel, PASTA_NO_FINALIZE), with
 * PASTA_REC_STABLE on the first batch and PASTA_REC_STABLE | PASTA_REC_CHAINED on the
 * rest. Stops at the first failing batch and returns its status; batches before it
 * stay enqueued. */
typedef struct {
  pasta_records trace;
  uint64_t n;
  pasta_histograms out;
} pasta_batch;
int pasta_analyze_batches(pasta_trace* h, const pasta_batch* batches, uint32_t count, uint32_t page_shift);

/* Rich 16-byte records (NEXT f4; R21-R23; SPEC S:39-42 MemAccessInfo):
 * little endian u64 address, u32 grid_id, u16 size_bytes (1..128), u8 flags
 * (PASTA_ACC_WRITE | PASTA_ACC_SHARED), u8 zero. */
typedef struct {
  uint64_t addr;
  uint32_t grid_id;
  uint16_t size_bytes;
  uint8_t flags;
  uint8_t reserved;
} pasta_rich_record;
enum { PASTA_ACC_WRITE = 1u, PASTA_ACC_SHARED = 2u };

typedef struct {
  const pasta_rich_record* records; /* [n] DEVICE memory, 16-byte aligned, read-only     */
  uint32_t grid_lo, grid_hi;        /* inclusive grid-id window (P:424 START_GRID_ID /
                                       END_GRID_ID); kernel row k = grid_id - grid_lo,
                                       n_kernels = grid_hi - grid_lo + 1               */
} pasta_rich_records;

/* Extra outputs of the rich analysis (caller-owned DEVICE memory, += like counts). */
enum { PASTA_RT_FILTERED = 0, PASTA_RT_SHARED = 1, PASTA_RT_WRITES = 2, PASTA_RT_BYTES = 3, PASTA_RICH_TOTALS = 4 };
typedef struct {
  uint64_t* rich_totals;        /* [PASTA_RICH_TOTALS] required: records outside the window,
                                   shared-space records (both dropped, R22-R23), writes and
                                   bytes (size_bytes) of the analyzed records            */
  uint64_t* page_write_counts;  /* [P] optional: analyzed writes per page                */
  uint64_t* alloc_write_counts; /* [max_ids] optional: analyzed writes per alloc id      */
  uint64_t* alloc_bytes;        /* [max_ids] optional: sum of size_bytes per alloc id (R21) */
} pasta_rich_outputs;

/* Analyze n rich records: every record whose grid_id lies in [grid_lo, grid_hi] and
 * that is not a shared-space access is analyzed exactly as pasta_analyze analyzes an
 * 8-byte record of kernel row grid_id - grid_lo (records of different kernels may be
 * interleaved); totals[RECORDS] counts the analyzed records. `out` may not ask for
 * kernel_page_bitmap, hotness or the tensor level (EINVAL). Then, unless
 * PASTA_NO_FINALIZE, pasta_finalize with n_kernels = grid_hi - grid_lo + 1. */
int pasta_analyze_rich(pasta_trace* h, const pasta_rich_records* trace, uint64_t n, uint32_t page_shift,
                       pasta_histograms* out, pasta_rich_outputs* rich);

/* Recompute the derived outputs from the accumulated counts in `out`:
 * page_bitmap (if non-NULL) and totals[UNIQUE_PAGES] from page_counts; for
 * n_kernels rows (if kernel_alloc_counts and kernel_stats are non-NULL)
 * footprint[k] = sum of registered sizes of ids with a non-zero count (P:797-799,
 * P:844), totals[WS_OBJ] = max_k footprint[k], and unique pages per kernel
 * from kernel_page_bitmap (if non-NULL); totals[MAX_KERNEL] from kernel_stats (R24); tensor
 * footprints and totals[WS_TENSOR] (if kernel_tensor_footprint is non-NULL). */
int pasta_finalize(pasta_trace* h, uint32_t page_shift, uint32_t n_kernels, pasta_histograms* out);

/* Top-K hot pages: the first min(k, nnz) pages with a non-zero count,
 * ordered by count descending then page index ascending (R10). out_page[k],
 * out_count[k] receive them; slots [found, k) get (UINT64_MAX, 0); *out_found =
 * min(k, nnz). All three are device pointers (pinned host memory works for
 * out_found). Radix select on the device; no host synchronization. k >= 1. */
int pasta_topk(pasta_trace* h, const uint64_t* page_counts, uint64_t P, uint32_t k, uint64_t* out_page,
               uint64_t* out_count, uint64_t* out_found);

/* Several top-K lists of the same counts (e.g. a config's top-16 and top-1024) with ONE
 * selection: for every j < n_k, out_page[j], out_count[j], out_found[j] receive exactly
 * what pasta_topk(h, page_counts, P, ks[j], ...) writes. R10's order (count desc, page
 * asc) is total, so a top-k list is the first k entries of the top-k_max list
 * (k_max = max_j ks[j]): the selection runs once for k_max into that entry's outputs and
 * one launch copies the prefixes into the others (pasta_topk_prefix). ks, out_page,
 * out_count, out_found are HOST arrays of n_k (1..16) entries; the pointers they hold are
 * device pointers as in pasta_topk; outputs of different entries must not overlap.
 * Every ks[j] >= 1. Asynchronous; PASTA_EINVAL on a bad argument. */
int pasta_topk_many(pasta_trace* h, const uint64_t* page_counts, uint64_t P, uint32_t n_k, const uint32_t* ks,
                    uint64_t* const* out_page, uint64_t* const* out_count, uint64_t* const* out_found);

/* The prefix step on its own (e.g. after pasta_topk_merge of the largest k in a
 * multi-GPU merge): src_* is a top-k_src list as pasta_topk / pasta_topk_merge write it
 * (device pointers); entry j (HOST arrays of n_k <= 16 entries) gets its first ks[j]
 * entries and *out_found[j] = min(ks[j], *src_found). 1 <= ks[j] <= k_src, else
 * PASTA_EINVAL. One launch, asynchronous on the handle's stream. */
int pasta_topk_prefix(pasta_trace* h, const uint64_t* src_page, const uint64_t* src_count, const uint64_t* src_found,
                      uint32_t k_src, uint32_t n_k, const uint32_t* ks, uint64_t* const* out_page,
                      uint64_t* const* out_count, uint64_t* const* out_found);

/* Multi-GPU merge helper (OR of bitmaps): out_bitmap[w] =
 * OR over r < g of gathered[r*words + w]; *out_popcount (device u64, may be NULL)
 * = number of set bits. NCCL has no bitwise-OR reduction, so shards all_gather their
 * bitmaps and OR them here. out_bitmap may alias gathered (r = 0 row). */
int pasta_bitmap_or(pasta_trace* h, const uint64_t* gathered, uint32_t g, uint64_t words, uint64_t* out_bitmap,
                    uint64_t* out_popcount);

/* Multi-GPU merge over peer memory (every count
 * is a pointwise sum over a partition of the records; working sets merge by MAX, R11).
 * src[r] (a HOST array of g <= 16 pointers) are DEVICE pointers readable from this
 * handle's device: local memory, or other ranks' buffers mapped with CUDA IPC (peer
 * access over NVLink / NVSwitch; see pasta_enable_peer). op PASTA_PEER_SUM:
 * out[i] = sum_r src[r][lo + i] (u64, wrapping) for i < n; if out_bitmap or
 * out_popcount is non-NULL, lo and n must be multiples of 64 (else EINVAL) and the same
 * pass writes out_bitmap[i / 64] bit i % 64 = (out[i] != 0) and adds the number of
 * non-zero out[i] to *out_popcount (device u64). op PASTA_PEER_MAX: out[i] = max_r
 * src[r][lo + i] (no bitmap). op PASTA_PEER_ARGMAX (n must be 2): each source holds an
 * (index, value) pair at src[r][lo], src[r][lo + 1] -- the totals[MAX_KERNEL,
 * MAX_KERNEL_RECORDS] pair of kernel-aligned shards (R24); out[0..1] = the pair with the
 * largest value, ties to the smallest index ("the kernel with the most memory
 * references"). out must not overlap any source range. The sources must
 * be complete (producers synchronized, e.g. a barrier after their analyze) and stay
 * unchanged until this call's stream work is done. */
enum { PASTA_PEER_SUM = 0u, PASTA_PEER_MAX = 1u, PASTA_PEER_ARGMAX = 2u };
int pasta_peer_reduce(pasta_trace* h, const uint64_t* const* src, uint32_t g, uint64_t lo, uint64_t n, uint32_t op,
                      uint64_t* out, uint64_t* out_bitmap, uint64_t* out_popcount);

/* Enable this handle's device to access memory of CUDA device `peer_device` (for
 * pasta_peer_reduce sources that live on another GPU). Idempotent; EINVAL for an
 * invalid device, ECUDA if the pair has no peer access. */
int pasta_enable_peer(pasta_trace* h, int peer_device);

/* Merge over peer memory without host round trips.
 *
 * pasta_peer_reduce_small: the small result part [alloc_counts | totals | tensor counts]
 * of g shards (src as in pasta_peer_reduce) in ONE launch: out[i] = sum_r src[r][lo + i]
 * (u64, wrapping) for i < n, except the listed slots: PASTA_PEER_MAX -> max_r;
 * PASTA_PEER_ARGMAX -> the (index, value) pair at i, i + 1 with the largest value, ties
 * to the smallest index (as pasta_peer_reduce's ARGMAX; R24); PASTA_PEER_ZERO -> 0 (a slot
 * another step recomputes, e.g. unique pages from the merged bitmap). slots: HOST array
 * of n_slots <= 16 entries with index < n (an ARGMAX entry needs index + 1 < n). SUM over
 * a partition is SPEC S:291-299, MAX for working sets R11. out must not overlap a source.
 * EINVAL on bad arguments. */
enum { PASTA_PEER_ZERO = 3u };
typedef struct {
  uint32_t index;  /* element index in [0, n) */
  uint32_t op;     /* PASTA_PEER_MAX, PASTA_PEER_ARGMAX or PASTA_PEER_ZERO */
} pasta_peer_slot;
int pasta_peer_reduce_small(pasta_trace* h, const uint64_t* const* src, uint32_t g, uint64_t lo, uint64_t n,
                            const pasta_peer_slot* slots, uint32_t n_slots, uint64_t* out);

/* pasta_peer_gather: up to 120 copies in ONE launch on the handle's stream (the second
 * merge phase: peers' bitmap words, unique-page counts and top-k candidates).
 * table: HOST array of count entries; entry e reads n u64 words at src (device memory
 * readable from this device: local, peer-enabled or IPC-mapped) and writes them to dst
 * (op PASTA_COPY) or adds them to dst with device atomics (PASTA_COPY_ADD: several
 * entries may add into one word). Entries with op COPY must not overlap each other or
 * any source. EINVAL for count == 0 or > 120, a NULL pointer with n > 0, or a bad op. */
enum { PASTA_COPY = 0u, PASTA_COPY_ADD = 1u };
typedef struct {
  const uint64_t* src;
  uint64_t* dst;
  uint64_t n;   /* u64 words */
  uint32_t op;  /* PASTA_COPY or PASTA_COPY_ADD */
  uint32_t pad;
} pasta_peer_copy;
int pasta_peer_gather(pasta_trace* h, const pasta_peer_copy* table, uint32_t count);

/* Streaming consumer (NEXT f2). The paper's profiler "records the
 * instruction into a device buffer" that the analysis drains, the program stalling
 * while the buffer is full, "e.g., 4MB" of it. pasta_stream_open launches
 * ONE persistent consumer on the handle's stream; the producer then publishes batches
 * (each a device buffer of records, e.g. 524,288 = 4 MB) with pasta_stream_push while it
 * runs, and the consumer accumulates them into `out` exactly as pasta_analyze calls with
 * PASTA_NO_FINALIZE would (counts are sums over any partition of the records, S:291-299;
 * kernel rows at kernel_row0 + local kernel, so a kernel cut between batches accumulates
 * into one row). At most `slots` batches are published and not yet read: push waits
 * (host spin, up to ~30 s, then PASTA_ESTATE) until the consumer has read the batch
 * `slots` places back, after which that batch's records and kernel offsets may be reused
 * by the producer (pasta_stream_consumed tells how many batches have been read; a pushed
 * batch's buffers must stay valid until then). pasta_stream_close publishes the end
 * (asynchronous: later work on the handle's stream, e.g. pasta_finalize / pasta_topk, is
 * ordered after the consumer drains); pasta_stream_destroy waits for the consumer and
 * frees (pasta_close does both for streams still open on the handle). The range table
 * is the one current at open (snapshot, R13). out: page_counts,
 * alloc_counts, totals required; kernel_alloc_counts / kernel_stats / kernel_page_bitmap
 * optional (rows for every kernel_row0 + local kernel pushed); no hotness, no tensor level
 * (EINVAL); out->flags ignored (never finalizes). Batches: addr 16-byte aligned, n even and
 * <= max_batch (n = 0 is skipped), kernel_offsets NULL (one kernel) or [n_kernels + 1]
 * batch-relative offsets with [0] = 0 and [n_kernels] = n (not checked: device memory).
 * While a stream is open the handle's stream is busy with it: do not enqueue other calls
 * of this handle until close. */
typedef struct pasta_stream pasta_stream;
typedef struct {
  uint32_t page_shift;
  uint32_t slots;      /* ring depth in batches, 2 .. 4096 */
  uint64_t max_batch;  /* records per batch at most (even, >= 256) */
} pasta_stream_params;
typedef struct {
  const uint64_t* addr;            /* device records */
  uint64_t n;
  const uint64_t* kernel_offsets;  /* device, batch-relative, or NULL */
  uint32_t n_kernels;
  uint32_t kernel_row0;
} pasta_stream_batch;
int pasta_stream_open(pasta_trace* h, const pasta_stream_params* p, const pasta_histograms* out, pasta_stream** s);
int pasta_stream_push(pasta_stream* s, const pasta_stream_batch* batches, uint32_t count);
int pasta_stream_consumed(pasta_stream* s, uint64_t* out_batches);
int pasta_stream_close(pasta_stream* s);
int pasta_stream_destroy(pasta_stream* s);

/* CUDA IPC of device buffers between the ranks of one node, opened in the HANDLE's device
 * context (cudaIpcMemLazyEnablePeerAccess: NVLink / NVSwitch loads once mapped).
 * pasta_ipc_export: a handle for the device allocation holding ptr (any address inside a
 * cudaMalloc'd block, e.g. a PyTorch caching-allocator tensor; the offset inside the
 * block is recorded). pasta_ipc_open (another process): *out_ptr = the same address in
 * this process, valid until pasta_ipc_close(out_ptr) or pasta_close; a block opened
 * twice is mapped once (reference counted). The exporting process must keep the block
 * alive while peers use it. Handles are plain bytes (send them over any channel).
 * ECUDA if the driver refuses (e.g. opening a handle in the exporting process). */
typedef struct {
  unsigned char handle[64];  /* cudaIpcMemHandle_t */
  uint64_t offset;           /* ptr - block base */
  uint64_t block_bytes;      /* size of the block */
  int32_t device;            /* CUDA ordinal of the exporting process's device */
  int32_t pad;
} pasta_ipc_handle;
int pasta_ipc_export(pasta_trace* h, const void* ptr, pasta_ipc_handle* out);
int pasta_ipc_open(pasta_trace* h, const pasta_ipc_handle* in, void** out_ptr);
int pasta_ipc_close(pasta_trace* h, void* ptr);

/* Multi-GPU top-K merge: g shard-local top-k lists, rank-major
 * (cand_page[r*k + i], cand_count[r*k + i], device pointers; pages relative to shard r,
 * empty slots have count 0), shard r covering global pages [r*shard_pages,
 * (r+1)*shard_pages). Writes the global top-k by (count desc, page asc) with global page
 * ids, (UINT64_MAX, 0) in slots [found, k), and *out_found = min(k, non-empty
 * candidates). Exact: a page in the global top-k is in its own shard's top-k. */
int pasta_topk_merge(pasta_trace* h, const uint64_t* cand_page, const uint64_t* cand_count, uint32_t g, uint32_t k,
                     uint64_t shard_pages, uint64_t* out_page, uint64_t* out_count, uint64_t* out_found);

/* Prefetch-plan builder (NEXT f3; S:488-514 build_prefetch_plan; R20). For
 * each kernel row k of `rows` (device, [n_kernels * n_ids] counts: kernel_alloc_counts
 * with level PASTA_LEVEL_OBJECT and n_ids = max_ids, or kernel_tensor_counts with
 * PASTA_LEVEL_TENSOR and n_ids = max_tensor_ids), the ranges to stage before kernel k:
 * the sorted disjoint union of [base, base + size) of the ids with a non-zero count
 * (registered ranges, even if freed since), touching intervals merged. Output (device):
 * plan_offsets[n_kernels + 1] (CSR, plan_offsets[0] = 0) and plan_ranges[2 * cap] as
 * (start, end) pairs, row k in [plan_offsets[k], plan_offsets[k+1]). *out_total (host)
 * = the number of intervals; if it exceeds cap nothing is written to plan_ranges and
 * the call returns ECAPACITY (plan_offsets is valid: size the buffer and call again).
 * Synchronizes the handle's stream (the total crosses to the host). */
enum { PASTA_LEVEL_OBJECT = 0u, PASTA_LEVEL_TENSOR = 1u };
int pasta_prefetch_plan(pasta_trace* h, const uint64_t* rows, uint32_t n_kernels, uint32_t level,
                        uint64_t* plan_offsets, uint64_t* plan_ranges, uint64_t cap, uint64_t* out_total);

/* Block until the handle's stream is idle; reports asynchronous faults (ECUDA). */
int pasta_sync(pasta_trace* h);

/* Release the handle's device and host resources (synchronizes its stream first).
 * pasta_close(NULL) is a no-op returning PASTA_OK. */
int pasta_close(pasta_trace* h);

/* Static string for a status code. */
const char* pasta_strerror(int status);

/* Instrumentation. With timing enabled every kernel the library launches is
 * bracketed by CUDA events on the launching stream. pasta_get_timing synchronizes
 * those events and returns accumulated milliseconds per phase
 * (out_ms[PASTA_PHASES]) and the number of kernels launched since open (always
 * counted). pasta_reset_timing zeroes both. */
enum { PASTA_PH_SCAN = 0, PASTA_PH_FINALIZE = 1, PASTA_PH_TOPK = 2, PASTA_PH_MERGE = 3, PASTA_PH_COPY = 4,
       PASTA_PH_PLAN = 5, PASTA_PHASES = 6 };
int pasta_set_timing(pasta_trace* h, int enable);
int pasta_get_timing(pasta_trace* h, double* out_ms, uint64_t* out_launches);
int pasta_reset_timing(pasta_trace* h);

#ifdef __cplusplus
}
#endif
#endif /* PASTA_H */
