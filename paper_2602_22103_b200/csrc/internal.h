// internal.h -- structures shared by the host library (pasta.cpp) and the kernel
// launchers (*.cu). Not part of the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pasta {

constexpr uint32_t kOOW = 0xFFFFFFFFu;       // page index sentinel: outside the window
constexpr uint32_t kNoTensor = 0xFFFFFFFFu;  // table interval in no live tensor
constexpr int kTotUntensored = 5;            // totals[PASTA_T_UNTENSORED]

// Everything the fused scan needs.
struct ScanArgs {
  const uint64_t* rec;       // body records (16-byte aligned), rec[0] has global index gidx0
  uint64_t nbody;            // even count of body records
  uint64_t gidx0;            // global record index of rec[0] (for kernel offsets)
  const uint64_t* bounds;    // [2A] sorted boundary array of the live ranges
  uint32_t samp_n, samp_sh;  // global-memory table: samp_n samples bounds[i << samp_sh] in shared memory (0: none)
  const uint32_t* ids;       // [A] alloc id of live range r
  uint32_t A;                // live ranges
  uint32_t n_kernels;        // >= 1
  const uint64_t* koffs;     // [n_kernels+1] or nullptr (one kernel)
  uint64_t va_lo, va_hi;
  uint32_t page_shift;
  uint32_t words;            // ceil(P/64) (kernel page bitmap row length)
  uint64_t max_ids;
  uint64_t* page_counts;
  uint64_t* alloc_counts;
  uint64_t* totals;
  uint64_t* kac;             // kernel_alloc_counts or nullptr
  uint64_t* kstats;          // kernel_stats or nullptr
  uint64_t* kpb;             // kernel_page_bitmap or nullptr
  uint64_t add_records;      // added to totals[RECORDS] by block 0
  uint64_t* hot;             // hotness [windows x P] or nullptr
  uint64_t P;                // pages in the window
  uint32_t window_kernels;   // kernels per hotness window (>= 1)
  uint64_t wk_magic;         // ceil(2^64 / window_kernels) for window_kernels >= 2
  const ulonglong2* chunk_k; // [chunks] (k, koffs[k+1]) of each interleaved chunk's first record (scratch)
  int32_t log_ic;            // log2 slices per interleaved chunk, -1 = contiguous (scan_schedule)
  unsigned long long* chunk_ctr;  // interleaved: the dynamic schedule's chunk counter (scratch, reset by the pre-pass)
  uint64_t chunk_perm;            // 0, or a multiplier coprime with (dynamic chunks - 1): permuted hand-out
  // tensor level (NEXT f3): all nullptr when off
  const uint32_t* tids;      // [A] tensor id of table interval r, kNoTensor = none
  uint64_t* tensor_counts;   // [max_tids]
  uint64_t* ktc;             // kernel_tensor_counts [n_kernels x max_tids] or nullptr
  uint64_t max_tids;
  uint32_t early;            // 1 PASTA_REC_STABLE: first loads before the grid-dependency wait; 2 CHAINED: wait at the end
};

// Streaming ring consumer (NEXT f2): one persistent launch consumes
// batch descriptors that the host publishes into a device ring while it runs.
struct StreamDesc {          // one batch (32 B, a device ring slot)
  const uint64_t* rec;       // [n] records, 16-byte aligned, n even
  uint64_t n;                // <= the stream's max batch
  const uint64_t* koffs;     // [nk + 1] batch-relative kernel offsets (device) or nullptr (one kernel)
  uint32_t nk;               // kernels in the batch (>= 1)
  uint32_t k0;               // kernel row of the batch's first kernel
};
constexpr int kStreamMaxCtas = 256;
struct StreamCtl {                              // device
  unsigned long long tail;                      // batches published (stream-ordered host copies)
  unsigned long long end;                       // total batches once closed, else ~0
  unsigned long long cta_done[kStreamMaxCtas];  // per CTA: batches all its warps have read
};
struct StreamArgs {
  ScanArgs s;                   // table, window, outputs (rec / nbody / koffs unused)
  const StreamDesc* ring;       // [slots]
  uint32_t slots;
  StreamCtl* ctl;
  uint64_t spb;                 // slices (256 records) per batch slot
  uint64_t cpb;                 // chunks (warp turns) per batch slot, set by the launcher
  unsigned long long* consumed; // host-mapped: batches every CTA has read (flow control)
  unsigned long long* prof;     // PASTA_STREAM_PROF builds: [ctas x warps x 5] counters, else unused
};
cudaError_t launch_stream_consumer(const StreamArgs& a, cudaStream_t st, int* ctas);

// Rich 16-byte records (NEXT f4; R21-R24).
struct RichArgs {
  const uint64_t* rec;       // [2n] u64 words: record i = (rec[2i], rec[2i+1]), 16-byte aligned
  uint64_t n;
  uint32_t grid_lo, grid_last;  // grid-id window [grid_lo, grid_lo + grid_last] (inclusive)
  const uint64_t* bounds;
  const uint32_t* ids;
  uint32_t A;
  uint64_t va_lo, va_hi;
  uint32_t page_shift;
  uint64_t max_ids;
  uint64_t* page_counts;
  uint64_t* page_writes;     // optional
  uint64_t* alloc_counts;
  uint64_t* alloc_writes;    // optional
  uint64_t* alloc_bytes;     // optional
  uint64_t* totals;          // [0] analyzed records, [1] unattributed, [2] out of window
  uint64_t* rich_totals;     // [4] filtered, shared, writes, bytes
  uint64_t* kac;             // [grid_n x max_ids] or nullptr
  uint64_t* kstats;          // [grid_n x 4] or nullptr
};
cudaError_t launch_rich(const RichArgs& a, int grid, cudaStream_t st);
int rich_slice_records();
int rich_warps();

// MAX_MEM_REFERENCED_KERNEL (R24): *out = argmax_k kstats[4k] + kstats[4k+1], ties low.
cudaError_t launch_max_kernel(const uint64_t* kstats, uint32_t n_kernels, uint64_t row0, uint64_t* out,
                              cudaStream_t st);

// Extra records that are not part of the 16-byte aligned even body (<= 2).
struct ExtraArgs {
  ScanArgs s;
  const uint64_t* ex_ptr[2];
  uint64_t ex_gidx[2];
  int n_ex;
};

int scan_smem_bytes(uint32_t A, bool big_table);
// Enqueues the scan of a (the chunk map pre-pass first when it is needed); adds the
// number of kernels launched to *launches.
cudaError_t launch_scan(const ScanArgs& a, int grid, cudaStream_t st, int* launches);
cudaError_t launch_scan_extras(const ExtraArgs& a, cudaStream_t st);
bool scan_table_fits_smem(uint32_t A);
int scan_warps();
// Scan schedule of a launch over nbody records on `grid` CTAs: log2 slices per
// interleaved chunk, or -1 for contiguous per-warp ranges; and the chunk map scratch.
// force: 0 = automatic, else PASTA_SCHED_CONTIGUOUS / PASTA_SCHED_INTERLEAVED.
int scan_schedule(uint64_t nbody, int grid, uint32_t force, uint32_t A);
int scan_permute_below();  // chunks per warp under which the dynamic hand-out is permuted
size_t scan_scratch_bytes(uint64_t nbody, int log_ic);

cudaError_t launch_finalize_bitmap(const uint64_t* page_counts, uint64_t P, uint64_t* bitmap, uint64_t* unique_out,
                                   int grid, cudaStream_t st);
// footprint[k] = sum of id_size[i] over ids with kac[k][i] > 0 -> fp_out[k * fp_stride],
// unique pages of row k of kpb (if non-null) -> up_out[k * up_stride] (if non-null),
// *ws_out = max_k footprint[k].
cudaError_t launch_footprint(const uint64_t* kac, uint32_t n_kernels, uint64_t max_ids, const uint64_t* id_size,
                             const uint64_t* kpb, uint32_t words, uint64_t* fp_out, uint32_t fp_stride,
                             uint64_t* up_out, uint32_t up_stride, uint64_t* ws_out, int grid, cudaStream_t st);

// Prefetch plans (NEXT f3, plan.cu): for each of n_kernels rows of `rows` ([n_kernels x
// n_ids]), the union of [base[i], base[i] + size[i]) over the ids with a non-zero
// count, visiting ids in `order` (ids sorted by base, n_order entries). Pass 1 writes
// per-row interval counts into offsets[1..n_kernels] and their exclusive scan (offsets[0]
// = 0); pass 2 (ranges != nullptr) writes the (start, end) pairs.
cudaError_t launch_plan_count(const uint64_t* rows, uint32_t n_kernels, uint64_t n_ids, const uint32_t* order,
                              uint32_t n_order, const uint64_t* base, const uint64_t* size, uint64_t* offsets,
                              cudaStream_t st, int* launches);
cudaError_t launch_plan_write(const uint64_t* rows, uint32_t n_kernels, uint64_t n_ids, const uint32_t* order,
                              uint32_t n_order, const uint64_t* base, const uint64_t* size, const uint64_t* offsets,
                              uint64_t* ranges, cudaStream_t st);
cudaError_t launch_bitmap_or(const uint64_t* gathered, uint32_t g, uint64_t words, uint64_t* out,
                             uint64_t* popcount, int grid, cudaStream_t st);

// Peer-memory merge (peer.cu): sources are device pointers readable from this device
// (local, peer-enabled or CUDA-IPC-mapped allocations of other ranks).
constexpr int kMaxPeers = 16;
struct PeerSrc {
  const uint64_t* p[kMaxPeers];
};
// op 0: out[i] = sum_r src[r][lo + i], and with out_bitmap / out_popcount (n and lo
// multiples of 64) the bitmap words of out and their popcount (+=); op 1: MAX.
cudaError_t launch_peer_reduce(const PeerSrc& src, uint32_t g, uint64_t lo, uint64_t n, uint32_t op, uint64_t* out,
                               uint64_t* out_bitmap, uint64_t* out_popcount, int grid, cudaStream_t st);

// pasta_peer_reduce_small: slot exceptions of the SUM (op 1 MAX, 2 ARGMAX pair, 3 ZERO).
struct PeerSlots {
  uint32_t idx[16];
  uint32_t op[16];
  uint32_t n;
};
cudaError_t launch_peer_small(const PeerSrc& src, uint32_t g, uint64_t lo, uint64_t n, const PeerSlots& sl,
                              uint64_t* out, int grid, cudaStream_t st);
// pasta_peer_gather: copies (op 0) / atomic adds (op 1) of n u64 words, one launch.
constexpr uint32_t kMaxCopies = 120;
struct PeerCopy {
  const uint64_t* src;
  uint64_t* dst;
  uint64_t n;
  uint32_t op;
  uint32_t pad;
};
struct PeerCopyTable {
  PeerCopy e[kMaxCopies];
  uint32_t count;
};
cudaError_t launch_peer_gather(const PeerCopyTable& t, int grid, cudaStream_t st);

// Top-K scratch (device): run_topk needs topk_scratch_bytes(k, P, max_ctas) (max_ctas =
// its CTA limit), run_topk_merge topk_merge_scratch_bytes(g * k, grid).
size_t topk_scratch_bytes(uint64_t k, uint64_t P, int max_ctas);
size_t topk_merge_scratch_bytes(uint64_t n, int grid);
// Enqueues the whole radix-select + gather + sort pipeline; `launch` is called once
// per kernel launch with the phase's cudaError_t (for counting / timing hooks).
typedef void (*launch_hook)(void* ctx, int begin);
// *head_state: 0 = unknown (the scratch is fresh or pasta_topk_merge used it), 1 / 2 =
// head 0 / head 1 is zero; run_topk updates it (the caller keeps it per scratch buffer).
cudaError_t run_topk(const uint64_t* page_counts, uint64_t P, uint32_t k, uint64_t* out_page, uint64_t* out_count,
                     uint64_t* out_found, void* scratch, int max_ctas, cudaStream_t st, int* n_launches,
                     int* head_state);

// Prefix copies of one top-k_max list into several top-k outputs (pasta_topk_many /
// pasta_topk_prefix): entry j gets the first k_j entries and found_j = min(k_j, found).
constexpr uint32_t kMaxTopkPrefix = 16;
struct TopkPrefix {
  uint64_t* dst_page;
  uint64_t* dst_count;
  uint64_t* dst_found;
  uint64_t k;
};
struct TopkPrefixTable {
  const uint64_t* src_page;
  const uint64_t* src_count;
  const uint64_t* src_found;
  TopkPrefix e[kMaxTopkPrefix];
  uint32_t count;
};
cudaError_t launch_topk_prefix(const TopkPrefixTable& t, int grid, cudaStream_t st);

cudaError_t run_topk_merge(const uint64_t* cand_page, const uint64_t* cand_count, uint32_t g, uint32_t k,
                           uint64_t shard_pages, uint64_t* out_page, uint64_t* out_count, uint64_t* out_found,
                           void* scratch, int grid, cudaStream_t st, int* n_launches);

}  // namespace pasta
