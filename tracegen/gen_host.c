/* tracegen/gen_host.c -- host implementation of the synthetic trace generator.
 *
 * SEEDED INPUT GENERATOR, shared by both sides of the parity contract (oracle and
 * CUDA path). It holds none of the analysis method's arithmetic: no range lookup,
 * no page indexing, no counting. It only maps a global record index j to an
 * 8-byte address, following the written spec in tracegen/GENERATOR.md.
 *
 * The device implementation (tracegen/gen_dev.cu) is written independently from
 * the same spec; tests/test_tracegen.py cross-checks the two byte for byte.
 */
#include <stdint.h>
#include <stddef.h>

/* One stream of the plan: 8 x u64, layout fixed by GENERATOR.md section 2. */
typedef struct {
    uint64_t start; /* global index of the stream's first record */
    uint64_t kind;  /* pattern id, GENERATOR.md section 3 */
    uint64_t base;  /* region base address */
    uint64_t size;  /* region size S in bytes */
    uint64_t p0, p1, p2;
    uint64_t pad;
} tg_stream;

enum { TG_SWEEP = 0, TG_STRIDED = 1, TG_PERM = 2, TG_ZIPF = 3, TG_TILED = 4, TG_STRAY = 5 };

static uint64_t tg_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Address of local record t of stream s (GENERATOR.md section 3). */
static uint64_t tg_addr(const tg_stream* s, const uint64_t* cdf, uint64_t t) {
    switch (s->kind) {
    case TG_SWEEP: { /* p0 = element size e, p1 = start element o (< S/e) */
        uint64_t e = s->p0, m = s->size / e;
        return s->base + e * ((s->p1 + t % m) % m);
    }
    case TG_STRIDED: { /* p0 = q, stride 2^q; (t << q) mod S with S a multiple of 2^q */
        uint64_t q = s->p0;
        uint64_t m = s->size >> q;
        return s->base + ((t % m) << q);
    }
    case TG_PERM: { /* p0 = e, p1 = alpha (odd), p2 = c; M = S/e is a power of two */
        uint64_t e = s->p0, M = s->size / e;
        return s->base + e * ((s->p1 * t + s->p2) & (M - 1));
    }
    case TG_ZIPF: { /* p0 = e | re<<8, p1 = seed, p2 = cdf_off<<32 | R */
        uint64_t e = s->p0 & 0xFF, re = (s->p0 >> 8) & 0xFF;
        uint64_t off = s->p2 >> 32, R = s->p2 & 0xFFFFFFFFULL;
        uint64_t g = t >> re, i = t & ((1ULL << re) - 1);
        uint64_t h = tg_splitmix64(s->p1 + g);
        /* row = first r with cdf[r] > h (bisection), clamped to R-1 */
        uint64_t lo = 0, hi = R; /* invariant: answer in [lo, hi] */
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (cdf[off + mid] > h) hi = mid; else lo = mid + 1;
        }
        uint64_t row = lo < R ? lo : R - 1;
        return s->base + row * (e << re) + i * e;
    }
    case TG_TILED: { /* p0 = e | lt<<8 | ln<<16, p1 = beta (odd), p2 = tile0 */
        uint64_t e = s->p0 & 0xFF, lt = (s->p0 >> 8) & 0xFF, ln = (s->p0 >> 16) & 0xFF;
        uint64_t r = t & ((1ULL << lt) - 1), u = t >> lt;
        uint64_t tile = (s->p2 + u * s->p1) & ((1ULL << ln) - 1);
        return s->base + ((tile << lt) + r) * e;
    }
    case TG_STRAY: { /* p0 = e (power of two), p1 = seed; S is a power of two */
        uint64_t h = tg_splitmix64(s->p1 + t);
        return s->base + ((h & (s->size - 1)) & ~(s->p0 - 1));
    }
    default:
        return 0;
    }
}

/* Fill out[0 .. j1-j0) with records j0 .. j1-1. streams sorted by start, ns >= 1,
 * streams[ns-1] covers up to the trace end. Returns 0, or -1 on bad arguments. */
int tracegen_host(const tg_stream* streams, uint64_t ns, const uint64_t* cdf,
                  uint64_t j0, uint64_t j1, uint64_t* out) {
    if (j1 < j0) return -1;
    if (j1 == j0) return 0;
    if (!streams || ns == 0 || !out) return -1;
    /* locate the stream holding j0: last s with start <= j0 */
    uint64_t lo = 0, hi = ns;
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (streams[mid].start <= j0) lo = mid; else hi = mid;
    }
    uint64_t s = lo;
    for (uint64_t j = j0; j < j1; ++j) {
        while (s + 1 < ns && streams[s + 1].start <= j) ++s;
        out[j - j0] = tg_addr(&streams[s], cdf, j - streams[s].start);
    }
    return 0;
}

/* SplitMix64 exported so the plan builder and tests use the same mixer. */
uint64_t tracegen_splitmix64(uint64_t x) { return tg_splitmix64(x); }
