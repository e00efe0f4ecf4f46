/* hand_worked.c -- the C ABI (include/pasta.h) used from plain C, no Python: the
 * hand-worked trace of tests/golden/hand_worked.json analyzed
 * on the GPU and checked against its hand-derived results.
 *
 *   make examples/hand_worked && ./examples/hand_worked      (needs a CUDA device)
 *
 * Prints "hand_worked ok" and exits 0 when every output matches; exits 1 on a mismatch,
 * 2 on an API error. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "pasta.h"

#define CHECK(x)                                                                   \
  do {                                                                             \
    int st_ = (x);                                                                 \
    if (st_ != PASTA_OK) {                                                         \
      fprintf(stderr, "%s: %s (%d)\n", #x, pasta_strerror(st_), st_);              \
      return 2;                                                                    \
    }                                                                              \
  } while (0)
#define CUDA(x)                                                                    \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                     \
      return 2;                                                                    \
    }                                                                              \
  } while (0)

static int expect_u64(const char* what, const uint64_t* got, const uint64_t* want, int n) {
  for (int i = 0; i < n; ++i)
    if (got[i] != want[i]) {
      fprintf(stderr, "%s[%d]: got %llu, want %llu\n", what, i, (unsigned long long)got[i],
              (unsigned long long)want[i]);
      return 1;
    }
  return 0;
}

int main(void) {
  /* R = {id0: [0x1000, 0x3000), id1: [0x5000, 0x5800)}, window [0, 0x8000), 4 KiB pages */
  const uint64_t rec[9] = {0x1000, 0x1008, 0x2FF8, 0x3000, 0x5000, 0x57FF, 0x5800, 0x9000, 0x2000};
  const uint64_t koffs[3] = {0, 4, 9};
  enum { P = 8, IDS = 2, K = 2, TOPK = 3 };

  pasta_open_params prm;
  memset(&prm, 0, sizeof(prm));
  prm.device = 0;
  prm.max_live = 4;
  prm.max_ids = IDS;
  prm.va_lo = 0;
  prm.va_hi = 0x8000;
  pasta_trace* h = NULL;
  CHECK(pasta_trace_open(&prm, &h));
  uint32_t id = 99;
  CHECK(pasta_register_alloc(h, 0x1000, 0x2000, &id));
  CHECK(pasta_register_alloc(h, 0x5000, 0x800, &id));

  uint64_t *d_rec, *d_koffs, *d_out, *d_top;
  /* outputs in one block: pages | allocs | totals | bitmap | kernel rows | kernel stats | kernel page bits */
  const size_t n_out = P + IDS + PASTA_TOTALS + 1 + K * IDS + K * PASTA_KSTATS + K * 1;
  CUDA(cudaMalloc((void**)&d_rec, sizeof(rec)));
  CUDA(cudaMalloc((void**)&d_koffs, sizeof(koffs)));
  CUDA(cudaMalloc((void**)&d_out, 8 * n_out));
  CUDA(cudaMalloc((void**)&d_top, 8 * (2 * TOPK + 1)));
  CUDA(cudaMemcpy(d_rec, rec, sizeof(rec), cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(d_koffs, koffs, sizeof(koffs), cudaMemcpyHostToDevice));
  CUDA(cudaMemset(d_out, 0, 8 * n_out));

  pasta_histograms out;
  memset(&out, 0, sizeof(out));
  out.page_counts = d_out;
  out.alloc_counts = d_out + P;
  out.totals = d_out + P + IDS;
  out.page_bitmap = d_out + P + IDS + PASTA_TOTALS;
  out.kernel_alloc_counts = d_out + P + IDS + PASTA_TOTALS + 1;
  out.kernel_stats = out.kernel_alloc_counts + K * IDS;
  out.kernel_page_bitmap = out.kernel_stats + K * PASTA_KSTATS;
  pasta_records tr = {d_rec, d_koffs, K, 0};
  CHECK(pasta_analyze(h, &tr, 9, 12, &out));  /* scan + finalize */
  CHECK(pasta_topk(h, out.page_counts, P, TOPK, d_top, d_top + TOPK, d_top + 2 * TOPK));
  CHECK(pasta_sync(h));

  uint64_t o[64], top[2 * TOPK + 1];
  CUDA(cudaMemcpy(o, d_out, 8 * n_out, cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(top, d_top, sizeof(top), cudaMemcpyDeviceToHost));
  const uint64_t* pages = o;
  const uint64_t* allocs = o + P;
  const uint64_t* tot = o + P + IDS;
  const uint64_t* kac = o + P + IDS + PASTA_TOTALS + 1;
  const uint64_t* ks = kac + K * IDS;
  const uint64_t* kpb = ks + K * PASTA_KSTATS;

  const uint64_t w_pages[P] = {0, 2, 2, 1, 0, 3, 0, 0};
  const uint64_t w_allocs[IDS] = {4, 2};
  const uint64_t w_tot[5] = {9, 3, 1, 4, 10240}; /* records, unattributed, out of window, unique pages, WS_obj */
  const uint64_t w_kac[K * IDS] = {3, 0, 1, 2};
  const uint64_t w_ks[K * PASTA_KSTATS] = {3, 1, 8192, 3, 3, 2, 10240, 2};
  const uint64_t w_top[2 * TOPK + 1] = {5, 1, 2, 3, 2, 2, 3}; /* pages, counts, found */
  int bad = expect_u64("page_counts", pages, w_pages, P) | expect_u64("alloc_counts", allocs, w_allocs, IDS) |
            expect_u64("totals", tot, w_tot, 5) | expect_u64("kernel_alloc_counts", kac, w_kac, K * IDS) |
            expect_u64("kernel_stats", ks, w_ks, K * PASTA_KSTATS) | expect_u64("top3", top, w_top, 2 * TOPK + 1);
  if (o[P + IDS + PASTA_TOTALS] != 0x2E) {
    fprintf(stderr, "bitmap word 0x%llx\n", (unsigned long long)o[P + IDS + PASTA_TOTALS]);
    bad = 1;
  }
  if (kpb[0] != 0x0E || kpb[1] != 0x24) { /* kernel 0: pages 1,2,3; kernel 1: pages 2,5 */
    fprintf(stderr, "kernel page bits 0x%llx 0x%llx\n", (unsigned long long)kpb[0], (unsigned long long)kpb[1]);
    bad = 1;
  }
  if (tot[PASTA_T_MAX_KERNEL] != 1 || tot[PASTA_T_MAX_KERNEL_RECORDS] != 5) { /* kernel 1: 5 records */
    fprintf(stderr, "max kernel %llu / %llu\n", (unsigned long long)tot[PASTA_T_MAX_KERNEL],
            (unsigned long long)tot[PASTA_T_MAX_KERNEL_RECORDS]);
    bad = 1;
  }
  cudaFree(d_rec);
  cudaFree(d_koffs);
  cudaFree(d_out);
  cudaFree(d_top);
  CHECK(pasta_close(h));
  if (bad) return 1;
  printf("hand_worked ok\n");
  return 0;
}
