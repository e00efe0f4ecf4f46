// tracegen/gen_dev.cu -- device implementation of the synthetic trace generator.
//
// SEEDED INPUT GENERATOR (test/bench infrastructure, not the product): written
// from tracegen/GENERATOR.md independently of tracegen/gen_host.c. It holds none of
// the analysis method's arithmetic. Each warp writes a contiguous tile of records
// with lane-interleaved (coalesced) stores; every lane locates its stream once by
// bisection and then walks forward.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

struct Stream {  // GENERATOR.md section 2
  unsigned long long start, kind, base, size, p0, p1, p2, pad;
};

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ unsigned long long address_of(const Stream& s, const unsigned long long* __restrict__ cdf,
                                         unsigned long long t) {
  const unsigned long long k = s.kind;
  if (k == 0) {  // sweep: base + e * ((o + t) mod (S/e))
    unsigned long long e = s.p0, m = s.size / e;
    unsigned long long x = t % m + s.p1;
    if (x >= m) x -= m;
    return s.base + x * e;
  }
  if (k == 1) {  // strided: base + ((t mod (S >> q)) << q)
    unsigned q = (unsigned)s.p0;
    return s.base + ((t % (s.size >> q)) << q);
  }
  if (k == 2) {  // permutation: base + e * ((alpha t + c) mod M), M = S/e power of two
    unsigned long long e = s.p0, mask = s.size / e - 1;
    return s.base + e * ((s.p1 * t + s.p2) & mask);
  }
  if (k == 3) {  // zipf row gather
    unsigned e = (unsigned)(s.p0 & 0xFF), re = (unsigned)((s.p0 >> 8) & 0xFF);
    unsigned long long off = s.p2 >> 32, R = s.p2 & 0xFFFFFFFFull;
    unsigned long long h = mix64(s.p1 + (t >> re));
    // count of thresholds <= h  == index of first threshold > h
    unsigned long long a = 0, n = R;
    while (n > 0) {
      unsigned long long half = n >> 1;
      if (cdf[off + a + half] <= h) { a += half + 1; n -= half + 1; }
      else n = half;
    }
    if (a >= R) a = R - 1;
    unsigned long long i = t & ((1ull << re) - 1);
    return s.base + a * ((unsigned long long)e << re) + i * e;
  }
  if (k == 4) {  // tiled reuse: permuted tile order, contiguous inside a tile
    unsigned e = (unsigned)(s.p0 & 0xFF), lt = (unsigned)((s.p0 >> 8) & 0xFF),
             ln = (unsigned)((s.p0 >> 16) & 0xFF);
    unsigned long long tile = (s.p2 + (t >> lt) * s.p1) & ((1ull << ln) - 1);
    unsigned long long elem = (tile << lt) | (t & ((1ull << lt) - 1));
    return s.base + elem * e;
  }
  if (k == 5) {  // stray: hashed offset inside a power-of-two region, aligned to e
    unsigned long long h = mix64(s.p1 + t) & (s.size - 1);
    return s.base + (h & ~(s.p0 - 1));
  }
  return 0ull;
}

constexpr int kPerLane = 16;  // records per lane per warp tile

__global__ void __launch_bounds__(256) gen_kernel(const Stream* __restrict__ st, unsigned long long ns,
                                                  const unsigned long long* __restrict__ cdf,
                                                  unsigned long long j0, unsigned long long j1,
                                                  unsigned long long* __restrict__ out) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  const unsigned long long tile = 32ull * kPerLane;
  for (unsigned long long t0 = j0 + warp * tile; t0 < j1; t0 += nwarps * tile) {
    unsigned long long j = t0 + lane;
    if (j >= j1) continue;
    // bisection: largest s with st[s].start <= j
    unsigned long long a = 0, b = ns - 1;
    while (a < b) {
      unsigned long long m = (a + b + 1) >> 1;
      if (st[m].start <= j) a = m; else b = m - 1;
    }
    for (int r = 0; r < kPerLane; ++r, j += 32) {
      if (j >= j1) break;
      while (a + 1 < ns && st[a + 1].start <= j) ++a;
      Stream s = st[a];
      out[j - j0] = address_of(s, cdf, j - s.start);
    }
  }
}

}  // namespace

extern "C" int tracegen_device(const void* d_streams, unsigned long long ns, const unsigned long long* d_cdf,
                               unsigned long long j0, unsigned long long j1, unsigned long long* d_out,
                               void* stream) {
  if (j1 < j0) return -1;
  if (j1 == j0) return 0;
  if (!d_streams || ns == 0 || !d_out) return -1;
  unsigned long long n = j1 - j0;
  unsigned long long tiles = (n + 32ull * kPerLane - 1) / (32ull * kPerLane);
  unsigned long long blocks = (tiles + 7) / 8;
  if (blocks > 148ull * 64) blocks = 148ull * 64;
  gen_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((const Stream*)d_streams, ns, d_cdf, j0, j1,
                                                                   d_out);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
