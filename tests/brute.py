"""A second, deliberately dumb oracle for tiny inputs (test-only pin of oracle/).

Linear scan over the live ranges, dense Python lists, O(P*K) repeated-maximum
selection for top-K. Written from the definitions (P:797-799, P:843-844, P:795,
P:916; readings R2-R14) independently of oracle/oracle.cpp:
no std::map, no hashing, no sorting.
"""
from __future__ import annotations

U64MAX = (1 << 64) - 1


def owner_of(a, live):
    """live: list of (base, size, id). Returns the id whose [base, base+size) holds a."""
    hit = None
    for base, size, i in live:
        if base <= a <= base + size - 1:
            assert hit is None, "live ranges overlap"
            hit = i
    return hit


def analyze(live, records, kernel_offsets, va_lo, va_hi, s, max_ids, window_kernels=1):
    P = (va_hi - va_lo) >> s
    page = [0] * P
    alloc = [0] * max_ids
    nk = len(kernel_offsets) - 1
    kac = [[0] * max_ids for _ in range(nk)]
    kun = [0] * nk
    kpages = [[0] * P for _ in range(nk)]
    nw = (nk + window_kernels - 1) // window_kernels
    hot = [[0] * P for _ in range(nw)]
    unattr = 0
    oow = 0
    for k in range(nk):
        for j in range(kernel_offsets[k], kernel_offsets[k + 1]):
            a = records[j]
            o = owner_of(a, live)
            if o is None:
                unattr += 1
                kun[k] += 1
            else:
                alloc[o] += 1
                kac[k][o] += 1
            if va_lo <= a and a < va_hi:
                p = 0
                lo = va_lo
                while not (lo <= a < lo + (1 << s)):  # walk pages, no shift/division
                    lo += 1 << s
                    p += 1
                page[p] += 1
                kpages[k][p] = 1
                hot[k // window_kernels][p] += 1
            else:
                oow += 1
    return dict(page=page, alloc=alloc, kac=kac, kun=kun, kpages=kpages, unattr=unattr, oow=oow, hot=hot)


def bitmap_words(page):
    P = len(page)
    words = []
    for w in range((P + 63) // 64):
        x = 0
        for b in range(64):
            p = 64 * w + b
            if p < P and page[p] != 0:
                x += 2 ** b
        words.append(x)
    return words


def footprints(kac, sizes):
    return [sum(sizes[i] for i in range(len(row)) if row[i] != 0) for row in kac]


def topk(page, K):
    """Repeatedly take the maximum count, earliest page first; stop at zero counts."""
    taken = [False] * len(page)
    out = []
    for _ in range(K):
        best = None
        for p in range(len(page)):
            if taken[p] or page[p] == 0:
                continue
            if best is None or page[p] > page[best]:
                best = p
        if best is None:
            out.append((U64MAX, 0))
        else:
            taken[best] = True
            out.append((best, page[best]))
    found = sum(1 for p, c in out if c != 0)
    return out, found


def analyze_rich(live, recs, grid_lo, grid_hi, va_lo, va_hi, s, max_ids):
    """recs: list of (addr, grid, size, is_write, shared) tuples (R21-R23)."""
    P = (va_hi - va_lo) >> s
    nk = grid_hi - grid_lo + 1
    r = dict(page=[0] * P, pw=[0] * P, alloc=[0] * max_ids, aw=[0] * max_ids, ab=[0] * max_ids,
             kac=[[0] * max_ids for _ in range(nk)], kun=[0] * nk, records=0, unattr=0, oow=0,
             filtered=0, shared=0, writes=0, bytes=0)
    for a, g, size, w, sh in recs:
        if not (grid_lo <= g <= grid_hi):
            r["filtered"] += 1
            continue
        if sh:
            r["shared"] += 1
            continue
        k = g - grid_lo
        r["records"] += 1
        o = owner_of(a, live)
        if o is None:
            r["unattr"] += 1
            r["kun"][k] += 1
        else:
            r["alloc"][o] += 1
            r["aw"][o] += w
            r["ab"][o] += size
            r["kac"][k][o] += 1
        if va_lo <= a < va_hi:
            p = 0
            lo = va_lo
            while not (lo <= a < lo + (1 << s)):
                lo += 1 << s
                p += 1
            r["page"][p] += 1
            r["pw"][p] += w
        else:
            r["oow"] += 1
        r["writes"] += w
        r["bytes"] += size
    return r
