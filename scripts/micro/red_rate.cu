// Microbenchmark: L2 RED throughput for scattered u64 / u32 counters (S-perm question:
// does grouping lanes onto shared sectors / lines raise the RED rate?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_rate red_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
// group = lanes sharing one "base" index; lanes within a group hit base + (lane % group) * spread
template <typename T>
__global__ void red2(T* a, uint64_t nelem, uint64_t iters, int group, int spread) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const unsigned lane = threadIdx.x & 31;
  const uint64_t gid = tid / group;
  for (uint64_t i = 0; i < iters; ++i) {
    const uint64_t base = mix(gid * 0x9E3779B97F4A7C15ull + i) % (nelem / 64) * 64;
    const uint64_t idx = base + (uint64_t)(lane % group) * spread;
    if (sizeof(T) == 8)
      asm volatile("red.global.add.u64 [%0], 1;" ::"l"(a + idx) : "memory");
    else
      asm volatile("red.global.add.u32 [%0], 1;" ::"l"(a + idx) : "memory");
  }
}
int main() {
  const uint64_t nelem = 4ull << 20;  // 4 Mi counters (gpt2m page count)
  void* buf; cudaMalloc(&buf, nelem * 8); cudaMemset(buf, 0, nelem * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512; const uint64_t iters = 512;
  const double total = (double)blocks * threads * iters;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int bytes, group, spread; const char* what; } cfgs[] = {
    {8, 1, 0, "u64 every lane random"}, {4, 1, 0, "u32 every lane random"},
    {8, 2, 1, "u64 pairs of lanes on adjacent counters (same 32B sector)"},
    {8, 4, 1, "u64 4 lanes per 32B sector"}, {8, 16, 1, "u64 16 lanes per 128B line"},
    {8, 32, 1, "u64 32 lanes on 2 lines"}, {8, 4, 4, "u64 4 lanes per 128B line, distinct sectors"},
    {4, 8, 1, "u32 8 lanes per 32B sector"}, {8, 32, 0, "u64 32 lanes same counter"}};
  for (auto& c : cfgs) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (c.bytes == 8) red2<uint64_t><<<blocks, threads>>>((uint64_t*)buf, nelem, iters, c.group, c.spread);
      else red2<uint32_t><<<blocks, threads>>>((uint32_t*)buf, nelem * 2, iters, c.group, c.spread);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-60s %8.1f G RED ops/s  (%.3f ms)\n", c.what, total / ms / 1e6, ms);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
