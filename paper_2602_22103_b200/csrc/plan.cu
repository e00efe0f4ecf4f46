// plan.cu -- prefetch-plan builder (NEXT f3; S:488-514 build_prefetch_plan, P:899-904;
// DESIGN.md R20): for every kernel row, the sorted disjoint union of the registered
// ranges [base, base + size) of the ids (objects or tensors) the kernel touched.
//
// One warp per row walks the ids in base order (`order`, built on the host) 32 at a
// time: lane i takes id order[c + i], selected if row[id] != 0. With ends e_i of the
// selected lanes, the exclusive prefix max of e (a 5-step shuffle scan, plus the carry
// of earlier chunks) is the end of the union interval still open before lane i; lane i
// starts a new interval iff nothing was selected before it or its base exceeds that
// end (touching intervals merge, as in the definition). The rank of a start among the
// starts (ballot + popc) is its output slot; a start also closes the previous interval
// by writing that prefix max as its end, and lane 0 closes the last one. Pass 1 only
// counts (then one block scans the counts into CSR offsets); pass 2 writes.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace pasta {
namespace {

using namespace dev;

constexpr int kBlock = 256;

template <bool kWrite>
__global__ void __launch_bounds__(kBlock) plan_kernel(const uint64_t* __restrict__ rows, uint32_t K, uint64_t n_ids,
                                                      const uint32_t* __restrict__ order, uint32_t n_order,
                                                      const uint64_t* __restrict__ base,
                                                      const uint64_t* __restrict__ size, uint64_t* offsets,
                                                      uint64_t* __restrict__ ranges) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;  // lanes below this one
  const uint64_t gw = ((uint64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * kBlock) >> 5;
  for (uint64_t k = gw; k < K; k += nw) {
    const uint64_t* row = rows + k * n_ids;
    const uint64_t o = kWrite ? offsets[k] : 0;
    uint64_t carry = 0;  // max end of every selected id in earlier chunks
    bool have = false;   // an id was selected in an earlier chunk
    uint64_t cnt = 0;    // intervals started so far in this row
    for (uint32_t c0 = 0; c0 < n_order; c0 += 32) {
      const uint32_t i = c0 + lane;
      bool sel = false;
      uint64_t b = 0, e = 0;
      if (i < n_order) {
        const uint32_t id = __ldg(order + i);
        if (__ldg(row + id) != 0) {
          sel = true;
          b = __ldg(base + id);
          e = b + __ldg(size + id);
        }
      }
      // inclusive prefix max of the selected ends
      uint64_t pm = sel ? e : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t v = __shfl_up_sync(kFull, pm, d);
        if (lane >= (unsigned)d) pm = v > pm ? v : pm;
      }
      uint64_t ex = __shfl_up_sync(kFull, pm, 1);
      if (lane == 0) ex = 0;
      if (carry > ex) ex = carry;
      const unsigned selm = __ballot_sync(kFull, sel);
      const bool before = have || (selm & lt) != 0;
      const bool start = sel && (!before || b > ex);
      const unsigned stm = __ballot_sync(kFull, start);
      if (kWrite && start) {
        const uint64_t slot = cnt + __popc(stm & lt);
        ranges[2 * (o + slot)] = b;
        if (slot > 0) ranges[2 * (o + slot - 1) + 1] = ex;
      }
      cnt += __popc(stm);
      const uint64_t cm = __shfl_sync(kFull, pm, 31);
      if (cm > carry) carry = cm;
      have = have || selm != 0;
    }
    if (lane == 0) {
      if (kWrite) {
        if (cnt > 0) ranges[2 * (o + cnt - 1) + 1] = carry;
      } else {
        offsets[k + 1] = cnt;
      }
    }
  }
}

// offsets[0] = 0, offsets[1..K] = counts -> exclusive scan in place (one block).
__global__ void __launch_bounds__(1024) scan_offsets_kernel(uint64_t* offsets, uint32_t K) {
  __shared__ uint64_t part[1024];
  const uint32_t t = threadIdx.x;
  const uint64_t per = ((uint64_t)K + 1023) / 1024;
  const uint64_t lo = 1 + t * per, hi = lo + per < (uint64_t)K + 1 ? lo + per : (uint64_t)K + 1;
  uint64_t s = 0;
  for (uint64_t i = lo; i < hi; ++i) s += offsets[i];
  part[t] = s;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {  // Hillis-Steele inclusive scan of the partials
    const uint64_t v = t >= (uint32_t)d ? part[t - d] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  uint64_t run = t ? part[t - 1] : 0;
  for (uint64_t i = lo; i < hi; ++i) {
    run += offsets[i];
    offsets[i] = run;
  }
  if (t == 0) offsets[0] = 0;
}

int plan_grid(uint32_t K) {
  uint64_t b = ((uint64_t)K + kBlock / 32 - 1) / (kBlock / 32);
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return (int)b;
}

}  // namespace

cudaError_t launch_plan_count(const uint64_t* rows, uint32_t n_kernels, uint64_t n_ids, const uint32_t* order,
                              uint32_t n_order, const uint64_t* base, const uint64_t* size, uint64_t* offsets,
                              cudaStream_t st, int* launches) {
  plan_kernel<false><<<plan_grid(n_kernels), kBlock, 0, st>>>(rows, n_kernels, n_ids, order, n_order, base, size,
                                                             offsets, nullptr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  scan_offsets_kernel<<<1, 1024, 0, st>>>(offsets, n_kernels);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_plan_write(const uint64_t* rows, uint32_t n_kernels, uint64_t n_ids, const uint32_t* order,
                              uint32_t n_order, const uint64_t* base, const uint64_t* size, const uint64_t* offsets,
                              uint64_t* ranges, cudaStream_t st) {
  plan_kernel<true><<<plan_grid(n_kernels), kBlock, 0, st>>>(rows, n_kernels, n_ids, order, n_order, base, size,
                                                            const_cast<uint64_t*>(offsets), ranges);
  return cudaGetLastError();
}

}  // namespace pasta
