// pasta.cpp -- host side of the C ABI (include/pasta.h): handle, range table,
// argument validation, stream-ordered table upload, kernel launches, the host-record
// (end-to-end) streaming path and instrumentation.
//
// The range table is the paper's "map from memory object to access count ...
// transferred to the GPU" when a kernel is launched: registrations edit a
// host std::map; the next pasta_analyze uploads the sorted boundary array
// B = [base_0, end_0, base_1, end_1, ...] and the range -> id map on the handle's
// stream (snapshot semantics, R13), so every enqueued call sees the table as it was
// when it was enqueued.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "internal.h"
#include "pasta.h"

using namespace pasta;

struct TimedLaunch {
  int phase;
  cudaEvent_t a, b;
};

struct pasta_trace {
  int device = 0;
  uint32_t sched = 0;  // PASTA_SCHED_* override, 0 = automatic
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;
  uint64_t va_lo = 0, va_hi = 0;
  uint32_t max_live = 0, max_ids = 0;
  int sm_count = 148;

  // host registration state
  std::map<uint64_t, std::pair<uint64_t, uint32_t>> live;  // base -> (size, id)
  std::vector<uint64_t> id_size;                           // id -> registered size
  std::vector<uint64_t> id_base;                           // id -> registered base (plans)
  bool dirty = true;

  // tensor level (NEXT f3, R18): tensors inside live objects
  uint32_t max_live_tensors = 0, max_tids = 0;
  std::map<uint64_t, std::pair<uint64_t, uint32_t>> tlive;  // base -> (size, tid)
  std::vector<uint64_t> tid_size, tid_base;
  uint32_t* d_tids = nullptr;      // [table capacity] tensor id of each table interval
  uint64_t* d_tid_size = nullptr;  // [max_tids]

  // prefetch-plan scratch: base[n], size[n], order[n]
  unsigned char* d_plan = nullptr;
  size_t plan_bytes = 0;
  uint64_t* h_total = nullptr;  // pinned: the plan's interval count

  // device table (capacity max_live / max_ids)
  uint64_t* d_bounds = nullptr;  // [2*max_live]
  uint32_t* d_ids = nullptr;     // [max_live]
  uint64_t* d_id_size = nullptr; // [max_ids]
  uint32_t A_dev = 0;            // live ranges in the most recently enqueued table
  unsigned char* h_stage = nullptr;  // pinned staging for table uploads
  size_t h_stage_bytes = 0;
  cudaEvent_t upload_done = nullptr;
  bool upload_pending = false;

  // top-K scratch
  void* d_topk = nullptr;
  size_t topk_bytes = 0;
  int topk_heads = 0;  // run_topk's head state for d_topk (0 = unknown)

  // streaming consumers opened on this handle and not destroyed yet (pasta_close ends them)
  std::vector<pasta_stream*> streams;

  // CUDA IPC blocks opened in this handle's context: handle bytes -> (base, refs); and
  // every pointer handed out -> its block's handle bytes
  std::map<std::string, std::pair<void*, int>> ipc_blocks;
  std::map<void*, std::pair<std::string, int>> ipc_ptrs;  // pointer -> (block key, opens)

  // scan scratch (interleaved schedule: chunk -> kernel map)
  unsigned char* d_scan = nullptr;
  size_t scan_bytes = 0;

  // host-record streaming path
  uint64_t host_chunk_bytes = 256ull << 20;
  uint64_t* d_stage[2] = {nullptr, nullptr};
  uint64_t* d_koffs = nullptr;
  size_t d_koffs_cap = 0;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_consumed[2] = {nullptr, nullptr};

  // instrumentation
  bool timing = false;
  std::vector<TimedLaunch> pending;
  std::vector<cudaEvent_t> free_events;
  double ms[PASTA_PHASES] = {};
  uint64_t launches = 0;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

cudaEvent_t take_event(pasta_trace* h) {
  if (!h->free_events.empty()) {
    cudaEvent_t e = h->free_events.back();
    h->free_events.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Brackets device work of one phase with events when timing is on.
struct Timed {
  pasta_trace* h;
  int phase;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Timed(pasta_trace* h_, int ph, cudaStream_t s) : h(h_), phase(ph), st(s) {
    if (h->timing) {
      a = take_event(h);
      cudaEventRecord(a, st);
    }
  }
  ~Timed() {
    if (h->timing && a) {
      cudaEvent_t b = take_event(h);
      cudaEventRecord(b, st);
      h->pending.push_back({phase, a, b});
    }
  }
};

int cuda_status(cudaError_t e) { return e == cudaSuccess ? PASTA_OK : PASTA_ECUDA; }

// Table capacity in intervals: objects, each tensor splitting its object at most twice.
uint64_t table_capacity(const pasta_trace* h) { return (uint64_t)h->max_live + 2ull * h->max_live_tensors; }

// Upload the current registration table if it changed (stream-ordered). The device
// table is a partition of the registered space into intervals: each live object, cut
// at its live tensors' bounds (R18), so one lookup names the object and the tensor.
int upload_table(pasta_trace* h) {
  if (!h->dirty) return PASTA_OK;
  const bool tens = h->max_tids > 0;
  uint64_t I = h->live.size();
  if (tens) I += 2ull * h->tlive.size();  // upper bound
  const size_t nid = h->id_size.size(), ntid = h->tid_size.size();
  const size_t need = 16ull * I + 8ull * I + 8ull * nid + 8ull * ntid + 64;
  if (h->upload_pending) {
    // the previous upload must have left the staging buffer before we overwrite it
    if (cudaEventSynchronize(h->upload_done) != cudaSuccess) return PASTA_ECUDA;
    h->upload_pending = false;
  }
  if (need > h->h_stage_bytes) {
    if (h->h_stage) cudaFreeHost(h->h_stage);
    h->h_stage = nullptr;
    size_t cap = std::max<size_t>(need, 4096);
    if (cudaMallocHost(&h->h_stage, cap) != cudaSuccess) {
      h->h_stage_bytes = 0;
      return PASTA_ECUDA;
    }
    h->h_stage_bytes = cap;
  }
  uint64_t* hb = reinterpret_cast<uint64_t*>(h->h_stage);
  uint64_t* hs = hb + 2ull * I;
  uint64_t* hts = hs + nid;
  uint32_t* hi = reinterpret_cast<uint32_t*>(hts + ntid);
  uint32_t* ht = hi + I;
  uint32_t r = 0;
  auto emit = [&](uint64_t lo, uint64_t hi_, uint32_t id, uint32_t tid) {
    hb[2 * r] = lo;
    hb[2 * r + 1] = hi_;
    hi[r] = id;
    ht[r] = tid;
    ++r;
  };
  for (const auto& kv : h->live) {  // std::map iterates in ascending base order
    const uint64_t ob = kv.first, oe = kv.first + kv.second.first;
    const uint32_t id = kv.second.second;
    if (!tens) {
      emit(ob, oe, id, kNoTensor);
      continue;
    }
    uint64_t cur = ob;
    for (auto t = h->tlive.lower_bound(ob); t != h->tlive.end() && t->first < oe; ++t) {
      if (t->first > cur) emit(cur, t->first, id, kNoTensor);
      emit(t->first, t->first + t->second.first, id, t->second.second);
      cur = t->first + t->second.first;
    }
    if (cur < oe) emit(cur, oe, id, kNoTensor);
  }
  for (size_t i = 0; i < nid; ++i) hs[i] = h->id_size[i];
  for (size_t i = 0; i < ntid; ++i) hts[i] = h->tid_size[i];
  cudaError_t e = cudaSuccess;
  if (r) e = cudaMemcpyAsync(h->d_bounds, hb, 16ull * r, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess && r) e = cudaMemcpyAsync(h->d_ids, hi, 4ull * r, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess && r && tens) e = cudaMemcpyAsync(h->d_tids, ht, 4ull * r, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess && nid) e = cudaMemcpyAsync(h->d_id_size, hs, 8ull * nid, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess && ntid)
    e = cudaMemcpyAsync(h->d_tid_size, hts, 8ull * ntid, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaEventRecord(h->upload_done, h->stream);
  if (e != cudaSuccess) return PASTA_ECUDA;
  h->upload_pending = true;
  h->A_dev = r;
  h->dirty = false;
  return PASTA_OK;
}

bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }

// Launch the scan over records [j0, j0 + n) that live at `rec` (device), with global
// record indices starting at g0 (for kernel offsets). add_records is added once.
constexpr uint32_t kChainSlicesPerWarp = 16;

int scan_range(pasta_trace* h, const uint64_t* rec, uint64_t n, uint64_t g0, ScanArgs base, cudaStream_t st,
               uint64_t add_records) {
  ExtraArgs ex{};
  ex.s = base;
  ex.n_ex = 0;
  const uint64_t* body = rec;
  uint64_t gb = g0;
  uint64_t nb = n;
  if (nb > 0 && (reinterpret_cast<uintptr_t>(body) & 15u) != 0) {  // 8-aligned, not 16: head record
    ex.ex_ptr[ex.n_ex] = body;
    ex.ex_gidx[ex.n_ex] = gb;
    ++ex.n_ex;
    ++body;
    ++gb;
    --nb;
  }
  if (nb & 1) {  // odd tail record
    ex.ex_ptr[ex.n_ex] = body + nb - 1;
    ex.ex_gidx[ex.n_ex] = gb + nb - 1;
    ++ex.n_ex;
    --nb;
  }
  // Per-CTA shared counters are u32: bound the records one launch gives a CTA.
  const uint64_t per_launch_max = (uint64_t)h->sm_count * (1ull << 31);
  bool added = false;
  for (uint64_t off = 0; off < nb; off += per_launch_max) {
    const uint64_t cnt = std::min<uint64_t>(per_launch_max, nb - off);
    ScanArgs a = base;
    a.rec = body + off;
    a.nbody = cnt;
    a.gidx0 = gb + off;
    a.add_records = added ? 0 : add_records;
    added = true;
    const uint64_t slices = (cnt + 255) / 256;  // 2 KiB slices, scan_warps() warps per CTA
    // A chained call overlaps its predecessors instead of waiting for them, so it takes
    // at least kChainSlicesPerWarp slices per warp: fewer CTAs per call, more calls in
    // flight (4 MB calls: 1.43 us each at 16 vs 4.06 us at 1 slice per warp). Other
    // calls spread over every SM (lowest latency for one call).
    const uint64_t wpc = (uint64_t)scan_warps() * (a.early == 2 ? kChainSlicesPerWarp : 1u);
    const int grid = (int)std::min<uint64_t>((uint64_t)h->sm_count, std::max<uint64_t>(1, (slices + wpc - 1) / wpc));
    a.log_ic = scan_schedule(cnt, grid, h->sched, a.A);
    if (a.log_ic >= 0 && a.early == 2) a.early = 1;  // the chunk-map pre-pass is this scan's predecessor
    const size_t sneed = scan_scratch_bytes(cnt, a.log_ic);
    if (sneed > h->scan_bytes) {
      if (h->d_scan) {
        cudaStreamSynchronize(st);
        cudaFree(h->d_scan);
      }
      h->d_scan = nullptr;
      h->scan_bytes = 0;
      if (cudaMalloc(&h->d_scan, sneed) != cudaSuccess) return PASTA_ECUDA;
      h->scan_bytes = sneed;
    }
    a.chunk_k = reinterpret_cast<const ulonglong2*>(h->d_scan);
    a.chunk_ctr = nullptr;
    if (a.log_ic >= 0) {  // the counter follows the chunk map (scan_scratch_bytes)
      const uint64_t nch = ((cnt + 255) / 256 + (1ull << a.log_ic) - 1) >> a.log_ic;
      a.chunk_ctr = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(h->d_scan) + 16 * nch);
      // a multiplier near 0.618 (M - 1) coprime with M - 1, M = the dynamically handed-out chunks
      const uint64_t nwarp = (uint64_t)grid * scan_warps();
      const uint64_t m1 = nch > nwarp + 1 ? nch - nwarp - 1 : 1;
      uint64_t mul = m1 * 618 / 1000 | 1;
      auto gcd = [](uint64_t x, uint64_t y) { while (y) { const uint64_t t = x % y; x = y; y = t; } return x; };
      while (m1 > 1 && gcd(mul, m1) != 1) ++mul;
      // permuted only when warps take few chunks (measured: gpt2m +1.7 %, uvm +1 %, rn50
      // +0.8 %; llama, 184 chunks per warp, -0.4 %): there the last grabs decide the end
      a.chunk_perm = (m1 > 1 && nch < nwarp * (uint64_t)scan_permute_below()) ? mul : 0;
    }
    Timed t(h, PASTA_PH_SCAN, st);
    int nl = 0;
    cudaError_t e = launch_scan(a, grid, st, &nl);
    h->launches += nl;
    if (e != cudaSuccess) return PASTA_ECUDA;
  }
  if (ex.n_ex > 0 || !added) {
    ex.s.add_records = added ? 0 : add_records;
    if (ex.n_ex > 0 || ex.s.add_records) {
      Timed t(h, PASTA_PH_SCAN, st);
      cudaError_t e = launch_scan_extras(ex, st);
      ++h->launches;
      if (e != cudaSuccess) return PASTA_ECUDA;
    }
  }
  return PASTA_OK;
}

int finalize_impl(pasta_trace* h, uint32_t page_shift, uint32_t n_kernels, pasta_histograms* out) {
  const uint64_t P = (h->va_hi - h->va_lo) >> page_shift;
  const uint32_t words = (uint32_t)((P + 63) / 64);
  const int grid = h->sm_count * 8;
  {
    Timed t(h, PASTA_PH_FINALIZE, h->stream);
    cudaError_t e = launch_finalize_bitmap(out->page_counts, P, out->page_bitmap, out->totals + PASTA_T_UNIQUE_PAGES,
                                           grid, h->stream);
    ++h->launches;
    if (e != cudaSuccess) return PASTA_ECUDA;
  }
  if (out->kernel_alloc_counts && out->kernel_stats && n_kernels > 0) {
    Timed t(h, PASTA_PH_FINALIZE, h->stream);
    cudaError_t e = launch_footprint(out->kernel_alloc_counts, n_kernels, h->max_ids, h->d_id_size,
                                     out->kernel_page_bitmap, words, out->kernel_stats + PASTA_K_FOOTPRINT,
                                     PASTA_KSTATS, out->kernel_stats + PASTA_K_UNIQUE_PAGES, PASTA_KSTATS,
                                     out->totals + PASTA_T_WS_OBJ, grid, h->stream);
    ++h->launches;
    if (e != cudaSuccess) return PASTA_ECUDA;
  }
  if (out->kernel_stats && n_kernels > 0) {
    Timed t(h, PASTA_PH_FINALIZE, h->stream);
    cudaError_t e = launch_max_kernel(out->kernel_stats, n_kernels, out->kernel_row0,
                                      out->totals + PASTA_T_MAX_KERNEL, h->stream);
    ++h->launches;
    if (e != cudaSuccess) return PASTA_ECUDA;
  }
  if (out->kernel_tensor_counts && out->kernel_tensor_footprint && n_kernels > 0) {
    Timed t(h, PASTA_PH_FINALIZE, h->stream);
    cudaError_t e = launch_footprint(out->kernel_tensor_counts, n_kernels, h->max_tids, h->d_tid_size, nullptr, 0,
                                     out->kernel_tensor_footprint, 1, nullptr, 0, out->totals + PASTA_T_WS_TENSOR,
                                     grid, h->stream);
    ++h->launches;
    if (e != cudaSuccess) return PASTA_ECUDA;
  }
  return PASTA_OK;
}

// Tensor-level output requirements (R18).
int check_tensor_outputs(const pasta_trace* h, const pasta_histograms* out) {
  if (out->tensor_counts && h->max_tids == 0) return PASTA_EINVAL;
  if (out->kernel_tensor_counts && (!out->tensor_counts || !out->kernel_alloc_counts)) return PASTA_EINVAL;
  if (out->kernel_tensor_footprint && !out->kernel_tensor_counts) return PASTA_EINVAL;
  return PASTA_OK;
}

int check_window(const pasta_trace* h, uint32_t page_shift) {
  if (page_shift < 12 || page_shift > 30) return PASTA_EINVAL;
  const uint64_t m = (1ull << page_shift) - 1;
  if ((h->va_lo & m) || (h->va_hi & m)) return PASTA_EINVAL;
  if (((h->va_hi - h->va_lo) >> page_shift) >= 0xFFFFFFFFull) return PASTA_EINVAL;
  return PASTA_OK;
}

int ensure_host_path(pasta_trace* h) {
  if (h->d_stage[0]) return PASTA_OK;
  for (int i = 0; i < 2; ++i) {
    if (cudaMalloc(&h->d_stage[i], h->host_chunk_bytes) != cudaSuccess) return PASTA_ECUDA;
    if (cudaEventCreateWithFlags(&h->ev_copied[i], cudaEventDisableTiming) != cudaSuccess) return PASTA_ECUDA;
    if (cudaEventCreateWithFlags(&h->ev_consumed[i], cudaEventDisableTiming) != cudaSuccess) return PASTA_ECUDA;
  }
  if (cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess) return PASTA_ECUDA;
  return PASTA_OK;
}

}  // namespace

extern "C" {

const char* pasta_strerror(int s) {
  switch (s) {
    case PASTA_OK: return "ok";
    case PASTA_EINVAL: return "invalid argument";
    case PASTA_EOVERLAP: return "range overlaps a live range";
    case PASTA_ENOENT: return "no live range with that base";
    case PASTA_ECAPACITY: return "capacity exceeded (max_live or max_ids)";
    case PASTA_ECUDA: return "CUDA error";
    case PASTA_ESTATE: return "invalid handle state";
    case PASTA_ENOMEM: return "out of host memory";
    default: return "unknown status";
  }
}

int pasta_trace_open(const pasta_open_params* p, pasta_trace** out) {
  if (!p || !out) return PASTA_EINVAL;
  if (p->max_live == 0 || p->max_ids == 0) return PASTA_EINVAL;
  if (p->flags != 0 && p->flags != PASTA_SCHED_CONTIGUOUS && p->flags != PASTA_SCHED_INTERLEAVED)
    return PASTA_EINVAL;
  if (p->va_lo >= p->va_hi || (p->va_lo & 4095) || (p->va_hi & 4095)) return PASTA_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) return PASTA_ECUDA;
  if (p->device < 0 || p->device >= ndev) return PASTA_EINVAL;
  pasta_trace* h = new (std::nothrow) pasta_trace();
  if (!h) return PASTA_ENOMEM;
  h->device = p->device;
  h->stream = reinterpret_cast<cudaStream_t>(p->stream);
  h->va_lo = p->va_lo;
  h->sched = p->flags;
  h->va_hi = p->va_hi;
  h->max_live = p->max_live;
  h->max_ids = p->max_ids;
  h->max_live_tensors = p->max_live_tensors;
  h->max_tids = p->max_tensor_ids;
  if (p->host_chunk_bytes) h->host_chunk_bytes = (p->host_chunk_bytes + 4095) / 4096 * 4096;
  DeviceGuard g(h->device);
  // the scan's chunk map: 4 MiB covers every launch up to ~4.3e9 records, so calls
  // captured into a CUDA graph never allocate
  constexpr size_t kScanScratch0 = 4u << 20;
  h->scan_bytes = kScanScratch0;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device) == cudaSuccess && sms > 0)
    h->sm_count = sms;
  const uint64_t tcap = table_capacity(h);
  bool ok = cudaMalloc(&h->d_bounds, 16ull * tcap) == cudaSuccess &&
            cudaMalloc(&h->d_ids, 4ull * tcap) == cudaSuccess &&
            cudaMallocHost(&h->h_total, sizeof(uint64_t)) == cudaSuccess &&
            cudaMalloc(&h->d_id_size, 8ull * h->max_ids) == cudaSuccess &&
            cudaMalloc(&h->d_scan, kScanScratch0) == cudaSuccess &&
            cudaEventCreateWithFlags(&h->upload_done, cudaEventDisableTiming) == cudaSuccess;
  if (ok) ok = cudaMemsetAsync(h->d_id_size, 0, 8ull * h->max_ids, h->stream) == cudaSuccess;
  if (ok && h->max_tids) {
    ok = cudaMalloc(&h->d_tids, 4ull * tcap) == cudaSuccess &&
         cudaMalloc(&h->d_tid_size, 8ull * h->max_tids) == cudaSuccess &&
         cudaMemsetAsync(h->d_tid_size, 0, 8ull * h->max_tids, h->stream) == cudaSuccess;
  }
  if (!ok) {
    pasta_close(h);
    return PASTA_ECUDA;
  }
  *out = h;
  return PASTA_OK;
}

int pasta_register_alloc(pasta_trace* h, uint64_t base, uint64_t size, uint32_t* out_id) {
  if (!h) return PASTA_EINVAL;
  // size > 0 and base + size <= 2^64 - 1 (the exclusive end is representable)
  if (size == 0 || base > UINT64_MAX - size) return PASTA_EINVAL;
  const uint64_t end = base + size;
  // overlap: the live range with the largest base < end must end at or before base
  auto it = h->live.lower_bound(end);  // first base >= end
  if (it != h->live.begin()) {
    auto pr = std::prev(it);
    if (pr->first + pr->second.first > base) return PASTA_EOVERLAP;
  }
  if (h->live.size() >= h->max_live || h->id_size.size() >= h->max_ids) return PASTA_ECAPACITY;
  const uint32_t id = (uint32_t)h->id_size.size();
  h->id_size.push_back(size);
  h->id_base.push_back(base);
  h->live.emplace(base, std::make_pair(size, id));
  h->dirty = true;
  if (out_id) *out_id = id;
  return PASTA_OK;
}

int pasta_register_free(pasta_trace* h, uint64_t base) {
  if (!h) return PASTA_EINVAL;
  auto it = h->live.find(base);
  if (it == h->live.end()) return PASTA_ENOENT;
  const uint64_t end = base + it->second.first;
  h->live.erase(it);
  // R19: the object's live tensors end with it
  h->tlive.erase(h->tlive.lower_bound(base), h->tlive.lower_bound(end));
  h->dirty = true;
  return PASTA_OK;
}

int pasta_register_tensor(pasta_trace* h, uint64_t base, uint64_t size, uint32_t* out_tid) {
  if (!h || h->max_tids == 0) return PASTA_EINVAL;
  if (size == 0 || base > UINT64_MAX - size) return PASTA_EINVAL;
  const uint64_t end = base + size;
  // containing object: the live object with the largest base <= base must hold [base, end)
  auto ob = h->live.upper_bound(base);
  if (ob == h->live.begin()) return PASTA_EINVAL;
  --ob;
  if (end > ob->first + ob->second.first) return PASTA_EINVAL;
  auto it = h->tlive.lower_bound(end);  // first tensor base >= end
  if (it != h->tlive.begin()) {
    auto pr = std::prev(it);
    if (pr->first + pr->second.first > base) return PASTA_EOVERLAP;
  }
  if (h->tlive.size() >= h->max_live_tensors || h->tid_size.size() >= h->max_tids) return PASTA_ECAPACITY;
  const uint32_t tid = (uint32_t)h->tid_size.size();
  h->tid_size.push_back(size);
  h->tid_base.push_back(base);
  h->tlive.emplace(base, std::make_pair(size, tid));
  h->dirty = true;
  if (out_tid) *out_tid = tid;
  return PASTA_OK;
}

int pasta_register_tensor_free(pasta_trace* h, uint64_t base) {
  if (!h) return PASTA_EINVAL;
  auto it = h->tlive.find(base);
  if (it == h->tlive.end()) return PASTA_ENOENT;
  h->tlive.erase(it);
  h->dirty = true;
  return PASTA_OK;
}

int pasta_analyze_batches(pasta_trace* h, const pasta_batch* batches, uint32_t count, uint32_t page_shift) {
  if (!h || (count > 0 && !batches)) return PASTA_EINVAL;
  for (uint32_t i = 0; i < count; ++i) {
    pasta_histograms out = batches[i].out;
    const int s = pasta_analyze(h, &batches[i].trace, batches[i].n, page_shift, &out);
    if (s != PASTA_OK) return s;
  }
  return PASTA_OK;
}

int pasta_report_memory_usage(pasta_trace* h, uint64_t ptr, int64_t delta, uint32_t* out_id) {
  if (!h || delta == 0 || delta == INT64_MIN) return PASTA_EINVAL;
  const bool tensors = h->max_tids > 0;
  if (delta > 0)
    return tensors ? pasta_register_tensor(h, ptr, (uint64_t)delta, out_id)
                   : pasta_register_alloc(h, ptr, (uint64_t)delta, out_id);
  const uint64_t size = (uint64_t)(-delta);
  auto& table = tensors ? h->tlive : h->live;
  auto it = table.find(ptr);
  if (it == table.end()) return PASTA_ENOENT;
  if (it->second.first != size) return PASTA_EINVAL;
  if (out_id) *out_id = it->second.second;
  return tensors ? pasta_register_tensor_free(h, ptr) : pasta_register_free(h, ptr);
}

int pasta_analyze(pasta_trace* h, const pasta_records* tr, uint64_t n, uint32_t page_shift, pasta_histograms* out) {
  if (!h || !tr || !out) return PASTA_EINVAL;
  if (!out->page_counts || !out->alloc_counts || !out->totals) return PASTA_EINVAL;
  if ((out->kernel_stats || out->kernel_page_bitmap || out->hotness) && !out->kernel_alloc_counts) return PASTA_EINVAL;
  if (out->hotness && out->window_kernels == 0) return PASTA_EINVAL;
  if (tr->flags & ~(PASTA_REC_HOST | PASTA_REC_STABLE | PASTA_REC_CHAINED)) return PASTA_EINVAL;
  if ((tr->flags & PASTA_REC_HOST) && (tr->flags & (PASTA_REC_STABLE | PASTA_REC_CHAINED))) return PASTA_EINVAL;
  int s = check_tensor_outputs(h, out);
  if (s) return s;
  s = check_window(h, page_shift);
  if (s) return s;
  if (n > 0 && (!tr->addr || !aligned8(tr->addr))) return PASTA_EINVAL;
  const uint32_t K = tr->kernel_offsets ? tr->n_kernels : 1;
  if (tr->kernel_offsets && tr->n_kernels == 0) return PASTA_EINVAL;
  const bool host = (tr->flags & PASTA_REC_HOST) != 0;
  if (host && tr->kernel_offsets) {
    if (tr->kernel_offsets[0] != 0 || tr->kernel_offsets[K] != n) return PASTA_EINVAL;
    for (uint32_t k = 0; k < K; ++k)
      if (tr->kernel_offsets[k] > tr->kernel_offsets[k + 1]) return PASTA_EINVAL;
  }
  DeviceGuard g(h->device);
  s = upload_table(h);
  if (s) return s;

  const uint64_t P = (h->va_hi - h->va_lo) >> page_shift;
  ScanArgs a{};
  a.bounds = h->d_bounds;
  a.ids = h->d_ids;
  a.A = h->A_dev;
  a.n_kernels = K;
  a.koffs = tr->kernel_offsets;
  a.va_lo = h->va_lo;
  a.va_hi = h->va_hi;
  a.page_shift = page_shift;
  a.words = (uint32_t)((P + 63) / 64);
  a.max_ids = h->max_ids;
  a.page_counts = out->page_counts;
  a.alloc_counts = out->alloc_counts;
  a.totals = out->totals;
  a.kac = out->kernel_alloc_counts;
  a.kstats = out->kernel_stats;
  a.kpb = out->kernel_page_bitmap;
  a.hot = out->hotness;
  a.P = P;
  a.window_kernels = out->window_kernels ? out->window_kernels : 1;
  a.wk_magic = a.window_kernels > 1 ? UINT64_MAX / a.window_kernels + 1 : 0;
  if (out->tensor_counts) {
    a.tids = h->d_tids;
    a.tensor_counts = out->tensor_counts;
    a.ktc = out->kernel_tensor_counts;
    a.max_tids = h->max_tids;
  }

  if (!host) {
    a.early = (tr->flags & PASTA_REC_CHAINED) ? 2u : (tr->flags & PASTA_REC_STABLE) ? 1u : 0u;
    s = scan_range(h, tr->addr, n, 0, a, h->stream, n);
    if (s) return s;
  } else {
    s = ensure_host_path(h);
    if (s) return s;
    if (tr->kernel_offsets && K > 1) {
      const size_t kb = 8ull * (K + 1);
      if (kb > h->d_koffs_cap) {
        if (h->d_koffs) cudaFree(h->d_koffs);
        h->d_koffs = nullptr;
        if (cudaMalloc(&h->d_koffs, kb) != cudaSuccess) return PASTA_ECUDA;
        h->d_koffs_cap = kb;
      }
      // synchronous upload from pageable memory is fine for the small offset array
      if (cudaMemcpyAsync(h->d_koffs, tr->kernel_offsets, kb, cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
        return PASTA_ECUDA;
      a.koffs = h->d_koffs;
    } else {
      a.n_kernels = 1;
      a.koffs = nullptr;
    }
    const uint64_t chunk = h->host_chunk_bytes / 8;
    uint64_t done = 0;
    int buf = 0;
    bool first = true;
    // the copy stream must not run ahead of work already queued on the compute stream
    cudaEventRecord(h->ev_consumed[0], h->stream);
    cudaEventRecord(h->ev_consumed[1], h->stream);
    while (done < n || first) {
      const uint64_t cnt = std::min<uint64_t>(chunk, n - done);
      if (cnt > 0) {
        {
          Timed t(h, PASTA_PH_COPY, h->copy_stream);
          if (cudaStreamWaitEvent(h->copy_stream, h->ev_consumed[buf], 0) != cudaSuccess) return PASTA_ECUDA;
          if (cudaMemcpyAsync(h->d_stage[buf], tr->addr + done, cnt * 8, cudaMemcpyHostToDevice, h->copy_stream) !=
              cudaSuccess)
            return PASTA_ECUDA;
          if (cudaEventRecord(h->ev_copied[buf], h->copy_stream) != cudaSuccess) return PASTA_ECUDA;
        }
        if (cudaStreamWaitEvent(h->stream, h->ev_copied[buf], 0) != cudaSuccess) return PASTA_ECUDA;
      }
      s = scan_range(h, h->d_stage[buf], cnt, done, a, h->stream, first ? n : 0);
      if (s) return s;
      if (cudaEventRecord(h->ev_consumed[buf], h->stream) != cudaSuccess) return PASTA_ECUDA;
      done += cnt;
      buf ^= 1;
      first = false;
    }
  }
  if (!(out->flags & PASTA_NO_FINALIZE)) {
    s = finalize_impl(h, page_shift, K, out);
    if (s) return s;
  }
  return PASTA_OK;
}

int pasta_analyze_rich(pasta_trace* h, const pasta_rich_records* tr, uint64_t n, uint32_t page_shift,
                       pasta_histograms* out, pasta_rich_outputs* rx) {
  if (!h || !tr || !out || !rx || !rx->rich_totals) return PASTA_EINVAL;
  if (!out->page_counts || !out->alloc_counts || !out->totals) return PASTA_EINVAL;
  if (out->kernel_page_bitmap || out->hotness || out->tensor_counts || out->kernel_tensor_counts ||
      out->kernel_tensor_footprint)
    return PASTA_EINVAL;
  if (out->kernel_stats && !out->kernel_alloc_counts) return PASTA_EINVAL;
  if (tr->grid_lo > tr->grid_hi) return PASTA_EINVAL;
  if (n > 0 && (!tr->records || (reinterpret_cast<uintptr_t>(tr->records) & 15u))) return PASTA_EINVAL;
  int s = check_window(h, page_shift);
  if (s) return s;
  DeviceGuard g(h->device);
  s = upload_table(h);
  if (s) return s;
  const uint64_t P = (h->va_hi - h->va_lo) >> page_shift;
  (void)P;
  RichArgs a{};
  a.grid_lo = tr->grid_lo;
  a.grid_last = tr->grid_hi - tr->grid_lo;
  const uint64_t n_rows = (uint64_t)a.grid_last + 1;
  a.bounds = h->d_bounds;
  a.ids = h->d_ids;
  a.A = h->A_dev;
  a.va_lo = h->va_lo;
  a.va_hi = h->va_hi;
  a.page_shift = page_shift;
  a.max_ids = h->max_ids;
  a.page_counts = out->page_counts;
  a.page_writes = rx->page_write_counts;
  a.alloc_counts = out->alloc_counts;
  a.alloc_writes = rx->alloc_write_counts;
  a.alloc_bytes = rx->alloc_bytes;
  a.totals = out->totals;
  a.rich_totals = rx->rich_totals;
  a.kac = out->kernel_alloc_counts;
  a.kstats = out->kernel_stats;
  if (n_rows > 0xFFFFFFFFull && a.kac) return PASTA_EINVAL;  // 2^32 kernel rows
  const uint64_t per_launch_max = (uint64_t)h->sm_count * (1ull << 30);
  const uint64_t* rec = reinterpret_cast<const uint64_t*>(tr->records);
  for (uint64_t off = 0; off < n; off += per_launch_max) {
    const uint64_t cnt = std::min<uint64_t>(per_launch_max, n - off);
    RichArgs b = a;
    b.rec = rec + 2 * off;
    b.n = cnt;
    const uint64_t slices = (cnt + rich_slice_records() - 1) / rich_slice_records();
    const uint64_t wpc = (uint64_t)rich_warps();
    const int grid = (int)std::min<uint64_t>((uint64_t)h->sm_count, (slices + wpc - 1) / wpc);
    Timed t(h, PASTA_PH_SCAN, h->stream);
    cudaError_t e = launch_rich(b, grid, h->stream);
    ++h->launches;
    if (e != cudaSuccess) return PASTA_ECUDA;
  }
  if (!(out->flags & PASTA_NO_FINALIZE)) {
    const uint32_t K = out->kernel_alloc_counts ? (uint32_t)n_rows : 1;
    s = finalize_impl(h, page_shift, K, out);
    if (s) return s;
  }
  return PASTA_OK;
}

int pasta_finalize(pasta_trace* h, uint32_t page_shift, uint32_t n_kernels, pasta_histograms* out) {
  if (!h || !out || !out->page_counts || !out->totals) return PASTA_EINVAL;
  if ((out->kernel_stats || out->kernel_page_bitmap) && !out->kernel_alloc_counts) return PASTA_EINVAL;
  int s = check_tensor_outputs(h, out);
  if (s) return s;
  s = check_window(h, page_shift);
  if (s) return s;
  DeviceGuard g(h->device);
  s = upload_table(h);  // id sizes must be current for the footprints
  if (s) return s;
  return finalize_impl(h, page_shift, n_kernels, out);
}

int pasta_topk(pasta_trace* h, const uint64_t* page_counts, uint64_t P, uint32_t k, uint64_t* out_page,
               uint64_t* out_count, uint64_t* out_found) {
  if (!h || !page_counts || !out_page || !out_count || !out_found || k == 0 || P == 0) return PASTA_EINVAL;
  DeviceGuard g(h->device);
  const int max_ctas = h->sm_count * 2;  // the cooperative top-K kernel: <= 2 CTAs per SM
  const size_t need = topk_scratch_bytes(k, P, max_ctas);
  if (need > h->topk_bytes) {
    if (h->d_topk) {
      cudaStreamSynchronize(h->stream);
      cudaFree(h->d_topk);
    }
    h->d_topk = nullptr;
    h->topk_bytes = 0;
    h->topk_heads = 0;
    if (cudaMalloc(&h->d_topk, need) != cudaSuccess) return PASTA_ECUDA;
    h->topk_bytes = need;
  }
  int nl = 0;
  Timed t(h, PASTA_PH_TOPK, h->stream);
  cudaError_t e =
      run_topk(page_counts, P, k, out_page, out_count, out_found, h->d_topk, max_ctas, h->stream, &nl, &h->topk_heads);
  if (e != cudaSuccess) h->topk_heads = 0;
  h->launches += (uint64_t)nl;
  return cuda_status(e);
}

int pasta_topk_prefix(pasta_trace* h, const uint64_t* src_page, const uint64_t* src_count, const uint64_t* src_found,
                      uint32_t k_src, uint32_t n_k, const uint32_t* ks, uint64_t* const* out_page,
                      uint64_t* const* out_count, uint64_t* const* out_found) {
  if (!h || !src_page || !src_count || !src_found || k_src == 0 || !ks || !out_page || !out_count || !out_found ||
      n_k == 0 || n_k > kMaxTopkPrefix)
    return PASTA_EINVAL;
  TopkPrefixTable t{};
  t.src_page = src_page;
  t.src_count = src_count;
  t.src_found = src_found;
  for (uint32_t j = 0; j < n_k; ++j) {
    if (ks[j] == 0 || ks[j] > k_src || !out_page[j] || !out_count[j] || !out_found[j]) return PASTA_EINVAL;
    t.e[j] = TopkPrefix{out_page[j], out_count[j], out_found[j], ks[j]};
  }
  t.count = n_k;
  DeviceGuard g(h->device);
  Timed tm(h, PASTA_PH_TOPK, h->stream);
  cudaError_t e = launch_topk_prefix(t, h->sm_count, h->stream);
  if (e == cudaSuccess) h->launches += 1;
  return cuda_status(e);
}

int pasta_topk_many(pasta_trace* h, const uint64_t* page_counts, uint64_t P, uint32_t n_k, const uint32_t* ks,
                    uint64_t* const* out_page, uint64_t* const* out_count, uint64_t* const* out_found) {
  if (!h || !page_counts || P == 0 || !ks || !out_page || !out_count || !out_found || n_k == 0 ||
      n_k > kMaxTopkPrefix)
    return PASTA_EINVAL;
  uint32_t jm = 0;
  for (uint32_t j = 0; j < n_k; ++j) {
    if (ks[j] == 0 || !out_page[j] || !out_count[j] || !out_found[j]) return PASTA_EINVAL;
    if (ks[j] > ks[jm]) jm = j;
  }
  int rc = pasta_topk(h, page_counts, P, ks[jm], out_page[jm], out_count[jm], out_found[jm]);
  if (rc != PASTA_OK || n_k == 1) return rc;
  uint32_t kk[kMaxTopkPrefix];
  uint64_t *op[kMaxTopkPrefix], *oc[kMaxTopkPrefix], *of[kMaxTopkPrefix];
  uint32_t m = 0;
  for (uint32_t j = 0; j < n_k; ++j) {
    if (j == jm) continue;
    kk[m] = ks[j];
    op[m] = out_page[j];
    oc[m] = out_count[j];
    of[m] = out_found[j];
    ++m;
  }
  return pasta_topk_prefix(h, out_page[jm], out_count[jm], out_found[jm], ks[jm], m, kk, op, oc, of);
}

int pasta_topk_merge(pasta_trace* h, const uint64_t* cand_page, const uint64_t* cand_count, uint32_t g, uint32_t k,
                     uint64_t shard_pages, uint64_t* out_page, uint64_t* out_count, uint64_t* out_found) {
  if (!h || !cand_page || !cand_count || !out_page || !out_count || !out_found || g == 0 || k == 0)
    return PASTA_EINVAL;
  DeviceGuard dg(h->device);
  const int grid = h->sm_count * 4;
  const size_t need = topk_merge_scratch_bytes((uint64_t)g * k, grid);
  if (need > h->topk_bytes) {
    if (h->d_topk) {
      cudaStreamSynchronize(h->stream);
      cudaFree(h->d_topk);
    }
    h->d_topk = nullptr;
    h->topk_bytes = 0;
    h->topk_heads = 0;
    if (cudaMalloc(&h->d_topk, need) != cudaSuccess) return PASTA_ECUDA;
    h->topk_bytes = need;
  }
  int nl = 0;
  Timed t(h, PASTA_PH_MERGE, h->stream);
  h->topk_heads = 0;  // the merge carves the same scratch: the next pasta_topk zeroes a head first
  cudaError_t e = run_topk_merge(cand_page, cand_count, g, k, shard_pages, out_page, out_count, out_found, h->d_topk,
                                 grid, h->stream, &nl);
  h->launches += (uint64_t)nl;
  return cuda_status(e);
}

int pasta_bitmap_or(pasta_trace* h, const uint64_t* gathered, uint32_t g, uint64_t words, uint64_t* out_bitmap,
                    uint64_t* out_popcount) {
  if (!h || !gathered || !out_bitmap || g == 0 || words == 0) return PASTA_EINVAL;
  DeviceGuard dg(h->device);
  Timed t(h, PASTA_PH_MERGE, h->stream);
  cudaError_t e = launch_bitmap_or(gathered, g, words, out_bitmap, out_popcount, h->sm_count * 8, h->stream);
  ++h->launches;
  return cuda_status(e);
}

int pasta_peer_reduce(pasta_trace* h, const uint64_t* const* src, uint32_t g, uint64_t lo, uint64_t n, uint32_t op,
                      uint64_t* out, uint64_t* out_bitmap, uint64_t* out_popcount) {
  if (!h || !src || !out || g == 0 || g > (uint32_t)kMaxPeers || n == 0) return PASTA_EINVAL;
  if (op != PASTA_PEER_SUM && op != PASTA_PEER_MAX && op != PASTA_PEER_ARGMAX) return PASTA_EINVAL;
  if (op == PASTA_PEER_ARGMAX && n != 2) return PASTA_EINVAL;
  const bool bits = out_bitmap || out_popcount;
  if (bits && (op != PASTA_PEER_SUM || lo % 64 || n % 64)) return PASTA_EINVAL;
  PeerSrc s{};
  for (uint32_t r = 0; r < g; ++r) {
    if (!src[r]) return PASTA_EINVAL;
    s.p[r] = src[r];
  }
  DeviceGuard dg(h->device);
  Timed t(h, PASTA_PH_MERGE, h->stream);
  cudaError_t e = launch_peer_reduce(s, g, lo, n, op, out, out_bitmap, out_popcount, h->sm_count * 8, h->stream);
  ++h->launches;
  return cuda_status(e);
}

// ---- streaming consumer (NEXT f2) ----
struct pasta_stream {
  pasta_trace* h = nullptr;
  uint32_t slots = 0;
  uint64_t max_batch = 0, spb = 0;
  StreamDesc* d_ring = nullptr;        // [slots] device
  StreamCtl* d_ctl = nullptr;          // device
  StreamDesc* h_ring = nullptr;        // [slots] pinned staging of the descriptors
  unsigned long long* h_vals = nullptr;  // [slots + 1] pinned: tail values, [slots] = end
  unsigned long long* h_consumed = nullptr;  // pinned, mapped: batches read (GPU writes)
  unsigned long long* d_consumed = nullptr;  // its device alias
  cudaStream_t cs = nullptr;           // publishing copies (never behind the consumer)
  uint64_t pushed = 0, seen = 0;
  uint32_t vslot = 0;
  bool closed = false;
  int ctas = 0;
  unsigned long long* d_prof = nullptr;  // PASTA_STREAM_PROF_OUT: per-warp counters
  StreamArgs args{};                     // the consumer's arguments (deferred launch)
  bool deferred = false;                 // PASTA_STREAM_DEFER_LAUNCH profiling hook
};

namespace {
void stream_free(pasta_stream* s) {
  if (s->cs) cudaStreamDestroy(s->cs);
  if (s->d_ring) cudaFree(s->d_ring);
  if (s->d_ctl) cudaFree(s->d_ctl);
  if (s->h_ring) cudaFreeHost(s->h_ring);
  if (s->h_vals) cudaFreeHost(s->h_vals);
  if (s->h_consumed) cudaFreeHost(s->h_consumed);
  delete s;
}

// Publish batches [first, s->pushed) from the pinned staging: the descriptor copies, then
// the new tail (its own pinned word), in order on the publishing stream.
int stream_publish(pasta_stream* s, uint64_t first) {
  uint64_t b = first;
  while (b < s->pushed) {
    const uint32_t i = (uint32_t)(b % s->slots);
    const uint64_t run = std::min<uint64_t>(s->pushed - b, s->slots - i);
    if (cudaMemcpyAsync(s->d_ring + i, s->h_ring + i, run * sizeof(StreamDesc), cudaMemcpyHostToDevice, s->cs) !=
        cudaSuccess)
      return PASTA_ECUDA;
    b += run;
  }
  unsigned long long* v = s->h_vals + s->vslot;
  s->vslot = (s->vslot + 1) % s->slots;
  *v = s->pushed;
  if (cudaMemcpyAsync(&s->d_ctl->tail, v, 8, cudaMemcpyHostToDevice, s->cs) != cudaSuccess) return PASTA_ECUDA;
  return PASTA_OK;
}
}  // namespace

int pasta_stream_open(pasta_trace* h, const pasta_stream_params* p, const pasta_histograms* out, pasta_stream** ps) {
  if (!h || !p || !out || !ps) return PASTA_EINVAL;
  if (!out->page_counts || !out->alloc_counts || !out->totals) return PASTA_EINVAL;
  if ((out->kernel_stats || out->kernel_page_bitmap) && !out->kernel_alloc_counts) return PASTA_EINVAL;
  if (out->hotness || out->tensor_counts || out->kernel_tensor_counts || out->kernel_tensor_footprint)
    return PASTA_EINVAL;
  if (p->slots < 2 || p->slots > 4096 || p->max_batch < 256 || (p->max_batch & 1)) return PASTA_EINVAL;
  int st = check_window(h, p->page_shift);
  if (st) return st;
  DeviceGuard g(h->device);
  st = upload_table(h);
  if (st) return st;
  pasta_stream* s = new (std::nothrow) pasta_stream;
  if (!s) return PASTA_ECUDA;
  s->h = h;
  s->slots = p->slots;
  s->max_batch = p->max_batch;
  s->spb = (p->max_batch + 255) / 256;
  bool ok = cudaStreamCreateWithFlags(&s->cs, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMalloc(&s->d_ring, sizeof(StreamDesc) * s->slots) == cudaSuccess &&
            cudaMalloc(&s->d_ctl, sizeof(StreamCtl)) == cudaSuccess &&
            cudaMallocHost(&s->h_ring, sizeof(StreamDesc) * s->slots) == cudaSuccess &&
            cudaMallocHost(&s->h_vals, 8ull * (s->slots + 1)) == cudaSuccess &&
            cudaHostAlloc(&s->h_consumed, 8, cudaHostAllocMapped) == cudaSuccess &&
            cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->d_consumed), s->h_consumed, 0) == cudaSuccess;
  if (ok) {
    *s->h_consumed = 0;
    s->h_vals[s->slots] = ~0ull;  // ctl.end = "not closed"
    ok = cudaMemsetAsync(s->d_ctl, 0, sizeof(StreamCtl), h->stream) == cudaSuccess &&
         cudaMemcpyAsync(&s->d_ctl->end, s->h_vals + s->slots, 8, cudaMemcpyHostToDevice, h->stream) == cudaSuccess;
    // the publishing copies must not overtake this initialization of the ring
    cudaEvent_t ev = nullptr;
    ok = ok && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventRecord(ev, h->stream) == cudaSuccess && cudaStreamWaitEvent(s->cs, ev, 0) == cudaSuccess;
    if (ev) cudaEventDestroy(ev);
  }
  if (!ok) {
    stream_free(s);
    return PASTA_ECUDA;
  }
  const uint64_t P = (h->va_hi - h->va_lo) >> p->page_shift;
  StreamArgs a{};
  a.s.bounds = h->d_bounds;
  a.s.ids = h->d_ids;
  a.s.A = h->A_dev;
  a.s.n_kernels = 1;
  a.s.va_lo = h->va_lo;
  a.s.va_hi = h->va_hi;
  a.s.page_shift = p->page_shift;
  a.s.words = (uint32_t)((P + 63) / 64);
  a.s.max_ids = h->max_ids;
  a.s.page_counts = out->page_counts;
  a.s.alloc_counts = out->alloc_counts;
  a.s.totals = out->totals;
  a.s.kac = out->kernel_alloc_counts;
  a.s.kstats = out->kernel_stats;
  a.s.kpb = out->kernel_page_bitmap;
  a.s.P = P;
  a.s.window_kernels = 1;
  a.s.log_ic = -1;
  a.ring = s->d_ring;
  a.slots = s->slots;
  a.ctl = s->d_ctl;
  a.spb = s->spb;
  a.consumed = s->d_consumed;
  a.prof = nullptr;
  if (getenv("PASTA_STREAM_PROF_OUT")) {  // profiling builds only (PASTA_STREAM_PROF)
    if (cudaMalloc(&s->d_prof, 8ull * 8 * kStreamMaxCtas * 32) == cudaSuccess) {
      cudaMemsetAsync(s->d_prof, 0, 8ull * 8 * kStreamMaxCtas * 32, h->stream);
      a.prof = s->d_prof;
    }
  }
  // Profiling hook (PASTA_STREAM_DEFER_LAUNCH set): launch the consumer only at close,
  // after every batch is published (needs slots >= batches), so that a replaying profiler
  // (ncu) sees a kernel whose inputs are all in device memory at launch.
  s->args = a;
  s->deferred = getenv("PASTA_STREAM_DEFER_LAUNCH") != nullptr;
  if (!s->deferred) {
    Timed t(h, PASTA_PH_SCAN, h->stream);
    const cudaError_t e = launch_stream_consumer(a, h->stream, &s->ctas);
    ++h->launches;
    if (e != cudaSuccess) {
      cudaGetLastError();
      stream_free(s);
      return PASTA_ECUDA;
    }
  }
  h->streams.push_back(s);
  *ps = s;
  return PASTA_OK;
}

int pasta_stream_push(pasta_stream* s, const pasta_stream_batch* batches, uint32_t count) {
  if (!s || (count && !batches)) return PASTA_EINVAL;
  if (s->closed) return PASTA_ESTATE;
  for (uint32_t i = 0; i < count; ++i) {
    const pasta_stream_batch& b = batches[i];
    if (b.n > s->max_batch || (b.n & 1) || (b.n && (!b.addr || (reinterpret_cast<uintptr_t>(b.addr) & 15u))))
      return PASTA_EINVAL;
    if (b.kernel_offsets && b.n_kernels == 0) return PASTA_EINVAL;
  }
  DeviceGuard g(s->h->device);
  uint64_t first = s->pushed;  // first batch not yet published
  for (uint32_t i = 0; i < count; ++i) {
    const uint64_t b = s->pushed;
    const uint64_t quarter = std::max<uint64_t>(1, s->slots / 4);
    if (b + 1 > s->seen + s->slots) {
      // the ring slot still holds an unread batch: publish what is staged, then wait
      // until a quarter of the ring (or what is left of this call) is free, so that each
      // publication (three small copies) covers many batches
      if (first < s->pushed) {
        const int st = stream_publish(s, first);
        if (st) return st;
        first = s->pushed;
      }
      const uint64_t want = std::min<uint64_t>(quarter, count - i);
      const auto t0 = std::chrono::steady_clock::now();
      for (;;) {
        const unsigned long long c = *reinterpret_cast<volatile unsigned long long*>(s->h_consumed);
        if (c > s->seen) s->seen = c;  // GPU writes may land out of order: keep the max
        if (b + want <= s->seen + s->slots) break;
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30)) return PASTA_ESTATE;
      }
    }
    StreamDesc& d = s->h_ring[b % s->slots];
    d.rec = batches[i].addr;
    d.n = batches[i].n;
    d.koffs = batches[i].kernel_offsets;
    d.nk = batches[i].kernel_offsets ? batches[i].n_kernels : 1;
    d.k0 = batches[i].kernel_row0;
    s->pushed = b + 1;
    // publish in runs of a quarter ring, so the consumer is fed while the host waits
    if (s->pushed - first >= quarter) {
      const int st = stream_publish(s, first);
      if (st) return st;
      first = s->pushed;
    }
  }
  if (first < s->pushed) return stream_publish(s, first);
  return PASTA_OK;
}

int pasta_stream_consumed(pasta_stream* s, uint64_t* out) {
  if (!s || !out) return PASTA_EINVAL;
  const unsigned long long c = *reinterpret_cast<volatile unsigned long long*>(s->h_consumed);
  if (c > s->seen) s->seen = c;
  *out = std::min<uint64_t>(s->seen, s->pushed);
  return PASTA_OK;
}

int pasta_stream_close(pasta_stream* s) {
  if (!s) return PASTA_EINVAL;
  if (s->closed) return PASTA_OK;
  DeviceGuard g(s->h->device);
  s->closed = true;
  s->h_vals[s->slots] = s->pushed;
  cudaError_t e = cudaMemcpyAsync(&s->d_ctl->end, s->h_vals + s->slots, 8, cudaMemcpyHostToDevice, s->cs);
  if (e == cudaSuccess && s->deferred) {  // profiling hook: everything is published now
    cudaEvent_t ev = nullptr;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(ev, s->cs);
      cudaStreamWaitEvent(s->h->stream, ev, 0);
      cudaEventDestroy(ev);
    }
    e = launch_stream_consumer(s->args, s->h->stream, &s->ctas);
    ++s->h->launches;
  }
  return cuda_status(e);
}

int pasta_stream_destroy(pasta_stream* s) {
  if (!s) return PASTA_OK;
  DeviceGuard g(s->h->device);
  auto& v = s->h->streams;
  v.erase(std::remove(v.begin(), v.end(), s), v.end());
  int st = PASTA_OK;
  if (!s->closed) st = pasta_stream_close(s);
  if (cudaStreamSynchronize(s->h->stream) != cudaSuccess) st = PASTA_ECUDA;
  if (s->d_prof) {
    const char* path = getenv("PASTA_STREAM_PROF_OUT");
    std::vector<unsigned long long> v(8ull * kStreamMaxCtas * 32);
    cudaMemcpy(v.data(), s->d_prof, 8 * v.size(), cudaMemcpyDeviceToHost);
    if (FILE* f = path ? fopen(path, "a") : nullptr) {
      for (size_t i = 0; i + 7 < v.size(); i += 8)
        if (v[i + 3])
          fprintf(f, "%zu %llu %llu %llu %llu %llu %llu\n", i / 8, v[i], v[i + 1], v[i + 2], v[i + 3], v[i + 4],
                  v[i + 5]);
      fclose(f);
    }
    cudaFree(s->d_prof);
  }
  stream_free(s);
  return st;
}

int pasta_peer_reduce_small(pasta_trace* h, const uint64_t* const* src, uint32_t g, uint64_t lo, uint64_t n,
                            const pasta_peer_slot* slots, uint32_t n_slots, uint64_t* out) {
  if (!h || !src || !out || g == 0 || g > (uint32_t)kMaxPeers || n == 0 || n_slots > 16) return PASTA_EINVAL;
  if (n_slots && !slots) return PASTA_EINVAL;
  PeerSrc s{};
  for (uint32_t r = 0; r < g; ++r) {
    if (!src[r]) return PASTA_EINVAL;
    s.p[r] = src[r];
  }
  PeerSlots sl{};
  sl.n = n_slots;
  for (uint32_t i = 0; i < n_slots; ++i) {
    const uint32_t op = slots[i].op;
    if (op != PASTA_PEER_MAX && op != PASTA_PEER_ARGMAX && op != PASTA_PEER_ZERO) return PASTA_EINVAL;
    if ((uint64_t)slots[i].index >= n || (op == PASTA_PEER_ARGMAX && (uint64_t)slots[i].index + 1 >= n))
      return PASTA_EINVAL;
    sl.idx[i] = slots[i].index;
    sl.op[i] = op;
  }
  DeviceGuard dg(h->device);
  Timed t(h, PASTA_PH_MERGE, h->stream);
  cudaError_t e = launch_peer_small(s, g, lo, n, sl, out, h->sm_count * 4, h->stream);
  ++h->launches;
  return cuda_status(e);
}

int pasta_peer_gather(pasta_trace* h, const pasta_peer_copy* table, uint32_t count) {
  if (!h || !table || count == 0 || count > kMaxCopies) return PASTA_EINVAL;
  PeerCopyTable t{};
  t.count = count;
  for (uint32_t j = 0; j < count; ++j) {
    const pasta_peer_copy& c = table[j];
    if (c.op != PASTA_COPY && c.op != PASTA_COPY_ADD) return PASTA_EINVAL;
    if (c.n && (!c.src || !c.dst)) return PASTA_EINVAL;
    t.e[j].src = c.src;
    t.e[j].dst = c.dst;
    t.e[j].n = c.n;
    t.e[j].op = c.op;
  }
  DeviceGuard dg(h->device);
  Timed tm(h, PASTA_PH_MERGE, h->stream);
  cudaError_t e = launch_peer_gather(t, h->sm_count * 4, h->stream);
  ++h->launches;
  return cuda_status(e);
}

namespace {
// cuMemGetAddressRange through the runtime's driver entry point (no -lcuda link).
typedef int (*MemGetAddressRangeFn)(unsigned long long* base, size_t* size, unsigned long long ptr);
MemGetAddressRangeFn mem_range_fn() {
  static MemGetAddressRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<MemGetAddressRangeFn>(p);
  }
  return fn;
}
}  // namespace

int pasta_ipc_export(pasta_trace* h, const void* ptr, pasta_ipc_handle* out) {
  if (!h || !ptr || !out) return PASTA_EINVAL;
  DeviceGuard dg(h->device);
  MemGetAddressRangeFn range = mem_range_fn();
  if (!range) return PASTA_ECUDA;
  unsigned long long base = 0;
  size_t bytes = 0;
  if (range(&base, &bytes, (unsigned long long)(uintptr_t)ptr) != 0) return PASTA_EINVAL;  // not device memory
  cudaIpcMemHandle_t hnd;
  cudaError_t e = cudaIpcGetMemHandle(&hnd, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return PASTA_ECUDA;
  }
  std::memset(out, 0, sizeof(*out));
  static_assert(sizeof(hnd) <= sizeof(out->handle), "IPC handle size");
  std::memcpy(out->handle, &hnd, sizeof(hnd));
  out->offset = (uint64_t)((uintptr_t)ptr - (uintptr_t)base);
  out->block_bytes = (uint64_t)bytes;
  out->device = h->device;
  return PASTA_OK;
}

int pasta_ipc_open(pasta_trace* h, const pasta_ipc_handle* in, void** out_ptr) {
  if (!h || !in || !out_ptr || in->offset >= in->block_bytes) return PASTA_EINVAL;
  DeviceGuard dg(h->device);
  const std::string key(reinterpret_cast<const char*>(in->handle), sizeof(cudaIpcMemHandle_t));
  auto it = h->ipc_blocks.find(key);
  void* base = nullptr;
  if (it != h->ipc_blocks.end()) {
    base = it->second.first;
    ++it->second.second;
  } else {
    cudaIpcMemHandle_t hnd;
    std::memcpy(&hnd, in->handle, sizeof(hnd));
    cudaError_t e = cudaIpcOpenMemHandle(&base, hnd, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return PASTA_ECUDA;
    }
    h->ipc_blocks[key] = {base, 1};
  }
  void* p = static_cast<char*>(base) + in->offset;
  *out_ptr = p;
  auto& e = h->ipc_ptrs[p];
  e.first = key;
  ++e.second;
  return PASTA_OK;
}

int pasta_ipc_close(pasta_trace* h, void* ptr) {
  if (!h || !ptr) return PASTA_EINVAL;
  auto it = h->ipc_ptrs.find(ptr);
  if (it == h->ipc_ptrs.end()) return PASTA_ENOENT;
  const std::string key = it->second.first;
  if (--it->second.second <= 0) h->ipc_ptrs.erase(it);
  auto b = h->ipc_blocks.find(key);
  if (b != h->ipc_blocks.end() && --b->second.second <= 0) {
    DeviceGuard dg(h->device);
    cudaStreamSynchronize(h->stream);  // no enqueued kernel may still read the block
    cudaIpcCloseMemHandle(b->second.first);
    h->ipc_blocks.erase(b);
  }
  return PASTA_OK;
}

int pasta_enable_peer(pasta_trace* h, int peer_device) {
  if (!h) return PASTA_EINVAL;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || peer_device < 0 || peer_device >= count) return PASTA_EINVAL;
  if (peer_device == h->device) return PASTA_OK;
  DeviceGuard dg(h->device);
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, h->device, peer_device) != cudaSuccess || !can) return PASTA_ECUDA;
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky-free status
    return PASTA_OK;
  }
  return cuda_status(e);
}

int pasta_prefetch_plan(pasta_trace* h, const uint64_t* rows, uint32_t n_kernels, uint32_t level,
                        uint64_t* plan_offsets, uint64_t* plan_ranges, uint64_t cap, uint64_t* out_total) {
  if (!h || !rows || !plan_offsets || !out_total || n_kernels == 0) return PASTA_EINVAL;
  if (level != PASTA_LEVEL_OBJECT && level != PASTA_LEVEL_TENSOR) return PASTA_EINVAL;
  if (level == PASTA_LEVEL_TENSOR && h->max_tids == 0) return PASTA_EINVAL;
  if (cap > 0 && !plan_ranges) return PASTA_EINVAL;
  const std::vector<uint64_t>& base = level == PASTA_LEVEL_TENSOR ? h->tid_base : h->id_base;
  const std::vector<uint64_t>& size = level == PASTA_LEVEL_TENSOR ? h->tid_size : h->id_size;
  const uint64_t n_ids = level == PASTA_LEVEL_TENSOR ? h->max_tids : h->max_ids;
  const uint32_t n = (uint32_t)base.size();  // ids issued so far (the rest have no counts)
  DeviceGuard g(h->device);
  // ids in base order (ties by id): the warp walk's visiting order
  std::vector<uint32_t> order(n);
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) {
    return base[x] != base[y] ? base[x] < base[y] : x < y;
  });
  const size_t need = 20ull * n + 64;
  if (need > h->plan_bytes) {
    if (h->d_plan) {
      cudaStreamSynchronize(h->stream);
      cudaFree(h->d_plan);
    }
    h->d_plan = nullptr;
    h->plan_bytes = 0;
    if (cudaMalloc(&h->d_plan, need) != cudaSuccess) return PASTA_ECUDA;
    h->plan_bytes = need;
  }
  uint64_t* d_base = reinterpret_cast<uint64_t*>(h->d_plan);
  uint64_t* d_size = d_base + n;
  uint32_t* d_order = reinterpret_cast<uint32_t*>(d_size + n);
  cudaStream_t st = h->stream;
  if (n) {
    // pageable sources: cudaMemcpyAsync stages them before returning
    if (cudaMemcpyAsync(d_base, base.data(), 8ull * n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(d_size, size.data(), 8ull * n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaMemcpyAsync(d_order, order.data(), 4ull * n, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return PASTA_ECUDA;
  }
  {
    Timed t(h, PASTA_PH_PLAN, st);
    int nl = 0;
    cudaError_t e = launch_plan_count(rows, n_kernels, n_ids, d_order, n, d_base, d_size, plan_offsets, st, &nl);
    h->launches += (uint64_t)nl;
    if (e != cudaSuccess) return PASTA_ECUDA;
  }
  if (cudaMemcpyAsync(h->h_total, plan_offsets + n_kernels, sizeof(uint64_t), cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return PASTA_ECUDA;
  *out_total = *h->h_total;
  if (*out_total > cap) return PASTA_ECAPACITY;
  Timed t(h, PASTA_PH_PLAN, st);
  cudaError_t e = launch_plan_write(rows, n_kernels, n_ids, d_order, n, d_base, d_size, plan_offsets, plan_ranges, st);
  ++h->launches;
  return cuda_status(e);
}

int pasta_sync(pasta_trace* h) {
  if (!h) return PASTA_EINVAL;
  DeviceGuard g(h->device);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e == cudaSuccess && h->copy_stream) e = cudaStreamSynchronize(h->copy_stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  return cuda_status(e);
}

int pasta_close(pasta_trace* h) {
  if (!h) return PASTA_OK;
  DeviceGuard g(h->device);
  // a consumer still running would never finish: publish its end, then wait and free it
  while (!h->streams.empty()) pasta_stream_destroy(h->streams.back());
  cudaStreamSynchronize(h->stream);
  if (h->copy_stream) {
    cudaStreamSynchronize(h->copy_stream);
    cudaStreamDestroy(h->copy_stream);
  }
  for (auto& t : h->pending) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : h->free_events) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (h->d_stage[i]) cudaFree(h->d_stage[i]);
    if (h->ev_copied[i]) cudaEventDestroy(h->ev_copied[i]);
    if (h->ev_consumed[i]) cudaEventDestroy(h->ev_consumed[i]);
  }
  for (auto& b : h->ipc_blocks) cudaIpcCloseMemHandle(b.second.first);
  h->ipc_blocks.clear();
  h->ipc_ptrs.clear();
  if (h->d_koffs) cudaFree(h->d_koffs);
  if (h->d_topk) cudaFree(h->d_topk);
  if (h->d_scan) cudaFree(h->d_scan);
  if (h->d_tids) cudaFree(h->d_tids);
  if (h->d_tid_size) cudaFree(h->d_tid_size);
  if (h->d_plan) cudaFree(h->d_plan);
  if (h->h_total) cudaFreeHost(h->h_total);
  if (h->d_bounds) cudaFree(h->d_bounds);
  if (h->d_ids) cudaFree(h->d_ids);
  if (h->d_id_size) cudaFree(h->d_id_size);
  if (h->upload_done) cudaEventDestroy(h->upload_done);
  if (h->h_stage) cudaFreeHost(h->h_stage);
  delete h;
  return PASTA_OK;
}

int pasta_set_timing(pasta_trace* h, int enable) {
  if (!h) return PASTA_EINVAL;
  h->timing = enable != 0;
  return PASTA_OK;
}

int pasta_get_timing(pasta_trace* h, double* out_ms, uint64_t* out_launches) {
  if (!h) return PASTA_EINVAL;
  DeviceGuard g(h->device);
  int status = PASTA_OK;
  for (auto& t : h->pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(t.b) != cudaSuccess || cudaEventElapsedTime(&ms, t.a, t.b) != cudaSuccess)
      status = PASTA_ECUDA;
    else
      h->ms[t.phase] += ms;
    h->free_events.push_back(t.a);
    h->free_events.push_back(t.b);
  }
  h->pending.clear();
  if (out_ms)
    for (int i = 0; i < PASTA_PHASES; ++i) out_ms[i] = h->ms[i];
  if (out_launches) *out_launches = h->launches;
  return status;
}

int pasta_reset_timing(pasta_trace* h) {
  if (!h) return PASTA_EINVAL;
  uint64_t l = 0;
  pasta_get_timing(h, nullptr, &l);
  for (int i = 0; i < PASTA_PHASES; ++i) h->ms[i] = 0;
  h->launches = 0;
  return PASTA_OK;
}

}  // extern "C"
