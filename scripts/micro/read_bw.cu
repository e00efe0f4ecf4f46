// Microbenchmark: HBM read bandwidth of the scan's access pattern without the analysis
// (is the scan at the read roofline, or issue-bound below it?). Per-warp 1-D TMA bulk
// copies of 2 KiB slices into a per-warp ring of S slots (mbarrier complete_tx), the
// consumer reads one word per lane per slice; and a plain LDG.128 streaming sum.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw read_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n)); }
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t par) {
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(a), "r"(par) : "memory");
}
__device__ __forceinline__ void expect_tx(uint32_t b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory"); }
__device__ __forceinline__ void tma1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t evict_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }

template <int W, int S, int SB, int SCHED, int R = 0>
__global__ void __launch_bounds__(W * 32, 1) tma_read(const uint64_t* rec, uint64_t nsl, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[W * S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ring = smem_u32(sm) + warp * S * SB, bar = smem_u32(bars + warp * S);
  const uint64_t gw = blockIdx.x * (uint64_t)W + warp, nw = (uint64_t)gridDim.x * W;
  uint64_t s0 = gw * nsl / nw, s1 = (gw + 1) * nsl / nw, n = s1 - s0;
  // slice index of this warp's j-th slice
  auto gs = [&](uint64_t j) -> uint64_t {
    if (SCHED == 1) return ((j >> 6) * nw + gw) * 64 + (j & 63);          // chunks of 64 interleaved over warps
    if (SCHED == 2) { const uint64_t c0 = blockIdx.x * (nsl / gridDim.x); return c0 + j * W + warp; }  // CTA region, warps interleaved
    return s0 + j;
  };
  if (SCHED == 1) n = (nsl / (64 * nw)) * 64;  // whole rounds of chunks only (the remainder is dropped)
  if (SCHED == 2) n = (nsl / gridDim.x) / W;
  if (lane == 0) { for (int j = 0; j < S; ++j) mbar_init(bar + 8 * j, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  const uint64_t pol = evict_first();
  if (lane == 0) for (uint64_t j = 0; j < S && j < n; ++j) { expect_tx(bar + 8 * j, SB); tma1d(ring + j * SB, (const char*)rec + gs(j) * SB, SB, bar + 8 * j, pol); }
  uint64_t acc = 0; uint32_t slot = 0, ph = 0;
  for (uint64_t j = 0; j < n; ++j) {
    mbar_wait(bar + 8 * slot, ph);
    if (R == 0) {
      uint64_t v; asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(ring + slot * SB + 8 * lane));
      acc += v;
    } else {
      // synthetic analysis load: every 2 KiB sub-slice as the scan reads it (4 LDS.128 per
      // lane) and R dependent rounds of integer mixing per value
#pragma unroll 1
      for (uint32_t h = 0; h < SB / 2048; ++h) {
        uint64_t a[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a[2 * i]), "=l"(a[2 * i + 1]) : "r"(ring + slot * SB + h * 2048 + 16 * lane + 512 * i));
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int i = 0; i < 8; ++i) a[i] = (a[i] ^ (a[i] >> 13)) + 0x9E3779B9u;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += a[i];
      }
    }
    __syncwarp();
    if (lane == 0 && j + S < n) { expect_tx(bar + 8 * slot, SB); tma1d(ring + slot * SB, (const char*)rec + gs(j + S) * SB, SB, bar + 8 * slot, pol); }
    if (++slot == S) { slot = 0; ph ^= 1; }
  }
  if (acc == 0x1234567) atomicAdd(out, acc);
}
__global__ void ldg_read(const ulonglong2* p, uint64_t n2, unsigned long long* out) {
  uint64_t acc = 0;
  const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n2; i += 4 * st) {
    ulonglong2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i + u * st < n2 ? __ldcs(p + i + u * st) : make_ulonglong2(0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x ^ v[u].y;
  }
  if (acc == 0x1234567) atomicAdd(out, acc);
}
template <int W, int S, int SB, int SCHED = 0, int R = 0>
void run(const char* name, const uint64_t* d, uint64_t bytes, unsigned long long* out, int sms) {
  auto fn = tma_read<W, S, SB, SCHED, R>;
  const int smem = W * S * SB;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); fn<<<sms, W * 32, smem>>>(d, bytes / SB, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
  }
  const uint64_t nsl = bytes / SB, nw = (uint64_t)sms * W;
  const uint64_t used = SCHED == 1 ? (nsl / (64 * nw)) * 64 * nw * SB : SCHED == 2 ? ((nsl / sms) / W) * W * sms * SB : bytes;
  cudaError_t err = cudaGetLastError();
  printf("%-44s %8.1f GB/s  (%.3f ms)  %s\n", name, used / best / 1e6, best, cudaGetErrorString(err));
  if (err != cudaSuccess) exit(1);
}
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const uint64_t bytes = 32ull << 30;
  uint64_t* d; if (cudaMalloc(&d, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(d, 1, bytes);
  unsigned long long* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<24, 4, 2048>("TMA 24 warps x 4 x 2 KiB (the scan's ring)", d, bytes, out, sms);
  run<24, 4, 2048, 1>("TMA 24x4x2K, 64-slice chunks interleaved (scan)", d, bytes, out, sms);
  run<24, 2, 4096, 1>("TMA 24x2x4K, chunks interleaved", d, bytes, out, sms);
  run<8, 4, 4096>("TMA 8 warps x 4 x 4 KiB", d, bytes, out, sms);
  run<4, 6, 8192>("TMA 4 warps x 6 x 8 KiB", d, bytes, out, sms);
  for (int rr = 0; rr < 1; ++rr) {
    run<24, 4, 2048, 1, 4>("+ALU R=4: 24x4x2K interleaved", d, bytes, out, sms);
    run<24, 2, 4096, 1, 4>("+ALU R=4: 24x2x4K interleaved", d, bytes, out, sms);
    run<24, 4, 2048, 1, 8>("+ALU R=8: 24x4x2K interleaved", d, bytes, out, sms);
    run<24, 2, 4096, 1, 8>("+ALU R=8: 24x2x4K interleaved", d, bytes, out, sms);
    run<24, 3, 2048, 1, 8>("+ALU R=8: 24x3x2K interleaved", d, bytes, out, sms);
    run<16, 3, 4096, 1, 8>("+ALU R=8: 16x3x4K interleaved", d, bytes, out, sms);
    run<24, 4, 2048, 1, 12>("+ALU R=12: 24x4x2K interleaved", d, bytes, out, sms);
    run<24, 2, 4096, 1, 12>("+ALU R=12: 24x2x4K interleaved", d, bytes, out, sms);
    run<24, 4, 2048, 1, 16>("+ALU R=16: 24x4x2K interleaved", d, bytes, out, sms);
    run<24, 2, 4096, 1, 16>("+ALU R=16: 24x2x4K interleaved", d, bytes, out, sms);
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bpsm : {4, 8}) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); ldg_read<<<sms * bpsm, 512>>>((const ulonglong2*)d, bytes / 16, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    printf("LDG.128 x4 streaming sum, %d x 512 thr/SM           %8.1f GB/s  (%.3f ms)\n", bpsm, bytes / best / 1e6, best);
  }
  // copy (read + write) like MEASURED_PEAKS
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); cudaMemcpyAsync((char*)d + bytes / 2, d, bytes / 2, cudaMemcpyDeviceToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
  }
  printf("cudaMemcpy D2D 16 GiB (read + write bytes)  %8.1f GB/s\n", bytes / best / 1e6);
  return 0;
}
