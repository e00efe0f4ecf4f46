"""Synthetic trace *plans* for the five BASELINE.json configs (tracegen/GENERATOR.md).

SEEDED INPUT GENERATOR -- shared by the oracle side and the CUDA side; it holds
none of the analysis method's arithmetic (no range lookup, no page indexing, no
counting). A plan is a small host-side description of a trace:

* ``allocs``: the registration list ``[(base, size), ...]`` (alloc ids 0, 1, ... in
  order), laid out by a caching-allocator model (512 B rounding, >= 2 MiB chunks at
  2 MiB-aligned bases, best fit);
* ``kernel_offsets``: CSR segment offsets, one segment per kernel launch;
* ``streams``: an ``(ns, 8)`` uint64 table; record ``j`` belongs to the last stream
  whose ``start <= j`` and its address is the stream pattern evaluated at the local
  index (GENERATOR.md section 3);
* ``cdf``: the integer Zipf threshold table shared by all ZIPF streams.

Records are produced from a plan by ``tracegen.host_records`` (C, host) or
``tracegen.device_records`` (CUDA), two independent implementations of the spec.
Workload shapes are stipulated, not pinned.
"""
from __future__ import annotations

import math
import random
from dataclasses import dataclass, field

import numpy as np

MiB = 1 << 20
GiB = 1 << 30

SWEEP, STRIDED, PERM, ZIPF, TILED, STRAY = range(6)
KIND_NAMES = {SWEEP: "sweep", STRIDED: "strided", PERM: "perm", ZIPF: "zipf", TILED: "tiled", STRAY: "stray"}

U64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """SplitMix64 (GENERATOR.md section 1); pure-Python copy used only for seeds."""
    z = (x + 0x9E3779B97F4A7C15) & U64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & U64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & U64
    return z ^ (z >> 31)


@dataclass
class Plan:
    name: str
    seed: int
    n: int
    va_lo: int
    va_hi: int
    page_shift: int
    allocs: list  # [(base, size)] in registration order => ids 0..A-1
    kernel_offsets: np.ndarray  # uint64 [K+1]
    streams: np.ndarray  # uint64 [ns, 8]
    cdf: np.ndarray  # uint64 [total rows]
    topk: list = field(default_factory=lambda: [16])
    want_kernel_rows: bool = True
    want_kernel_pages: bool = False
    note: str = ""
    # the allocator's pool chunks [(base, size)]: the object level when ``allocs`` (the
    # tensors) are registered as a second level (NEXT f3); each alloc lies in one chunk
    objects: list = field(default_factory=list)

    @property
    def n_kernels(self) -> int:
        return len(self.kernel_offsets) - 1

    @property
    def n_pages(self) -> int:
        return (self.va_hi - self.va_lo) >> self.page_shift

    @property
    def max_ids(self) -> int:
        return len(self.allocs)

    def kind_mix(self) -> dict:
        """Records per pattern kind (for DESIGN.md's recipe table)."""
        out = {}
        starts = [int(x) for x in self.streams[:, 0]] + [self.n]
        for i in range(len(self.streams)):
            k = KIND_NAMES[int(self.streams[i, 1])]
            out[k] = out.get(k, 0) + starts[i + 1] - starts[i]
        return out

    def shard(self, rank: int, world: int):
        """Kernel-aligned contiguous shard [j0, j1) and its kernel range [k0, k1)
        (SURVEY.md section 8e): the cut for rank r is the kernel boundary nearest
        r*n/world (ties to the lower boundary)."""
        offs = [int(x) for x in self.kernel_offsets]

        def cut(r):
            if r <= 0:
                return 0
            if r >= world:
                return len(offs) - 1
            target = self.n * r // world
            best = 0
            for k, o in enumerate(offs):
                if abs(o - target) < abs(offs[best] - target):
                    best = k
            return best

        k0, k1 = cut(rank), cut(rank + 1)
        return offs[k0], offs[k1], k0, k1


class _Allocator:
    """Caching-allocator model: 512 B rounding, chunks of
    max(chunk_min, roundup(size, 2 MiB)) at 2 MiB-aligned bases, best fit with ties to
    the lowest address. Every ``hole_every``-th chunk is followed by an unmapped
    2 MiB hole (a target for stray records)."""

    def __init__(self, base: int, chunk_min: int = 2 * MiB, hole_every: int = 8):
        self.next = base
        self.chunk_min = chunk_min
        self.hole_every = hole_every
        self.free = []  # [(addr, len)]
        self.chunks = []  # [(base, size)]
        self.holes = []  # [(base, size)]

    def alloc(self, size: int) -> int:
        r = (size + 511) // 512 * 512
        best = None
        for i, (a, ln) in enumerate(self.free):
            if ln >= r and (best is None or ln < self.free[best][1] or (ln == self.free[best][1] and a < self.free[best][0])):
                best = i
        if best is None:
            csz = max(self.chunk_min, (r + 2 * MiB - 1) // (2 * MiB) * (2 * MiB))
            cb = self.next
            self.chunks.append((cb, csz))
            self.next = cb + csz
            if self.hole_every and len(self.chunks) % self.hole_every == 0:
                self.holes.append((self.next, 2 * MiB))
                self.next += 2 * MiB
            self.free.append((cb, csz))
            best = len(self.free) - 1
        a, ln = self.free[best]
        if ln == r:
            self.free.pop(best)
        else:
            self.free[best] = (a + r, ln - r)
        return a


def _zipf_cdf(rows: int, alpha: float) -> np.ndarray:
    """Integer thresholds cdf[r] = floor(2^64 * F(r)), F the Zipf(alpha) CDF over
    ranks 0..rows-1; last entry forced to 2^64-1. Monotone non-decreasing."""
    w = [1.0 / (r + 1) ** alpha for r in range(rows)]
    tot = math.fsum(w)
    acc = 0.0
    out = np.empty(rows, dtype=np.uint64)
    prev = 0
    for r in range(rows):
        acc += w[r]
        v = min(U64, int(acc / tot * float(1 << 64)))
        v = max(v, prev)
        out[r] = v
        prev = v
    out[-1] = U64
    return out


def _pow2_floor(x: int) -> int:
    return 1 << (x.bit_length() - 1)


class _Builder:
    """Accumulates kernels -> streams; record counts are assigned at the end so the
    total is exactly n (integer cumulative apportionment)."""

    def __init__(self, seed: int):
        self.rng = random.Random(seed)
        self.seed = seed
        self.kernels = []  # list of list of (weight, kind, base, size, p0, p1, p2)
        self.cdf_parts = []
        self.cdf_len = 0

    def zipf_table(self, rows: int, alpha: float = 1.1) -> int:
        off = self.cdf_len
        self.cdf_parts.append(_zipf_cdf(rows, alpha))
        self.cdf_len += rows
        return off

    def stream_seed(self) -> int:
        return splitmix64(self.seed ^ (self.rng.getrandbits(40) << 20))

    # --- pattern constructors: return a stream tuple (weight filled by caller) ---
    def sweep(self, base, size, e):
        m = size // e
        return (SWEEP, base, m * e, e, self.rng.randrange(m), 0)

    def strided(self, base, size, q):
        m = size >> q
        return (STRIDED, base, m << q, q, 0, 0)

    def perm(self, base, size, e):
        S = _pow2_floor(size)
        M = S // e
        alpha = (self.rng.getrandbits(40) << 1) | 1
        return (PERM, base, S, e, alpha, self.rng.randrange(M))

    def tiled(self, base, size, e, tile_bytes=4096):
        S = _pow2_floor(size)
        lt = (tile_bytes // e).bit_length() - 1
        ntiles = max(1, S // tile_bytes)
        ln = ntiles.bit_length() - 1
        beta = (self.rng.getrandbits(30) << 1) | 1
        return (TILED, base, (1 << ln) * tile_bytes, e | (lt << 8) | (ln << 16), beta, self.rng.randrange(1 << ln))

    def zipf(self, base, rows, row_elems, e, cdf_off):
        re = row_elems.bit_length() - 1
        assert 1 << re == row_elems
        return (ZIPF, base, rows * row_elems * e, e | (re << 8), self.stream_seed(), (cdf_off << 32) | rows)

    def stray(self, base, size_pow2, e=4):
        return (STRAY, base, size_pow2, e, self.stream_seed(), 0)

    def add_kernel(self, parts):
        """parts: [(weight, stream_tuple)]"""
        self.kernels.append(parts)

    def finish(self, n: int, kernel_records=None):
        """Assign record counts: globally proportional to stream weights (integer
        cumulative apportionment), or, if ``kernel_records`` is given, exactly that
        many records per kernel split by weight inside the kernel."""
        if kernel_records is None:
            budgets = None
        else:
            budgets = [int(x) for x in kernel_records]
            assert len(budgets) == len(self.kernels) and sum(budgets) == n
        rows = []
        kernel_offsets = [0]
        prev = 0
        if budgets is None:
            W = sum(int(w) for parts in self.kernels for w, _ in parts)
            assert W > 0
            cum = 0
            for parts in self.kernels:
                for w, st in parts:
                    cum += int(w)
                    end = n * cum // W
                    rows.append([prev, *st, 0])
                    prev = end
                kernel_offsets.append(prev)
        else:
            for parts, bud in zip(self.kernels, budgets):
                W = sum(int(w) for w, _ in parts)
                k0 = prev
                cum = 0
                for w, st in parts:
                    cum += int(w)
                    end = k0 + bud * cum // W
                    rows.append([prev, *st, 0])
                    prev = end
                kernel_offsets.append(prev)
        assert prev == n and len(kernel_offsets) == len(self.kernels) + 1
        streams = np.array(rows, dtype=np.uint64).reshape(-1, 8)
        cdf = np.concatenate(self.cdf_parts) if self.cdf_parts else np.array([U64], dtype=np.uint64)
        return np.array(kernel_offsets, dtype=np.uint64), streams, cdf


# ----------------------------------------------------------------------------------------
# config 1: tiny
# ----------------------------------------------------------------------------------------
def plan_tiny(seed: int = 42, n: int = 1 << 20) -> Plan:
    va_lo = 0x7F0000000000
    b = _Builder(seed)
    allocs = [(va_lo + i * 4 * MiB, 64 * 1024 * (i + 1)) for i in range(16)]
    zoff = b.zipf_table(64)
    # 8 kernels: 2 sweep, 2 strided, 2 perm, 1 zipf, 1 mixed + 1% stray
    b.add_kernel([(1, b.sweep(*allocs[0], 4)), (1, b.sweep(*allocs[1], 8))])
    b.add_kernel([(1, b.sweep(*allocs[2], 16)), (1, b.sweep(*allocs[3], 4))])
    b.add_kernel([(1, b.strided(allocs[4][0], allocs[4][1], 12))])
    b.add_kernel([(1, b.strided(allocs[5][0], allocs[5][1], 7)), (1, b.strided(allocs[6][0], allocs[6][1], 13))])
    b.add_kernel([(1, b.perm(*allocs[7], 4))])
    b.add_kernel([(1, b.perm(*allocs[8], 8)), (1, b.perm(*allocs[9], 16))])
    # zipf rows of 256 fp32 elements (1 KiB) inside alloc 15 (1 MiB => 64 rows)
    b.add_kernel([(1, b.zipf(allocs[15][0], 64, 256, 4, zoff))])
    # mixed kernel: sweep + tiled + perm, plus 1% stray split between an allocator gap
    # (inside the window) and outside the window
    b.add_kernel([
        (33, b.sweep(*allocs[10], 8)),
        (33, b.tiled(*allocs[11], 16)),
        (33, b.perm(*allocs[12], 4)),
        (1, b.stray(allocs[13][0] + allocs[13][1] + 64 * 1024, 1 << 20)),  # gap after alloc 13
        (1, b.stray(va_lo + 64 * MiB + 8 * MiB, 1 << 20)),  # above the window
    ])
    # each of the 8 kernels holds exactly n/8 records
    ko, st, cdf = b.finish(n, kernel_records=[n // 8 + (1 if i < n % 8 else 0) for i in range(8)])
    return Plan("tiny", seed, n, va_lo, va_lo + 64 * MiB, 12, allocs, ko, st, cdf, topk=[16],
                want_kernel_rows=True, want_kernel_pages=True,
                note="16 allocs at va_lo+i*4MiB of 64KiB*(i+1); 8 kernels",
                objects=[(va_lo + i * 4 * MiB, 4 * MiB) for i in range(16)])


# ----------------------------------------------------------------------------------------
# DL-shaped plans (configs 2-5)
# ----------------------------------------------------------------------------------------
@dataclass
class _Tensor:
    name: str
    size: int
    base: int = 0
    role: str = "act"  # weight | grad | act | workspace | embed


def _place(tensors, va_lo, chunk_min, hole_every=8):
    al = _Allocator(va_lo, chunk_min=chunk_min, hole_every=hole_every)
    for t in tensors:
        t.base = al.alloc(t.size)
    return al


def _transformer_tensors(n_layers, d, ff, vocab, tokens, eb, train, attn_scores_bytes=0):
    """Tensor list of a GPT-style decoder (sizes in bytes, element size eb)."""
    ts = [_Tensor("wte", vocab * d * eb, role="embed"), _Tensor("wpe", 2048 * d * eb, role="weight")]
    if train:
        ts.append(_Tensor("wte.grad", vocab * d * eb, role="grad"))
    for l in range(n_layers):
        ws = [("ln1.w", d), ("ln1.b", d), ("qkv.w", d * 3 * d), ("qkv.b", 3 * d), ("o.w", d * d), ("o.b", d),
              ("ln2.w", d), ("ln2.b", d), ("fc1.w", d * ff), ("fc1.b", ff), ("fc2.w", ff * d), ("fc2.b", d)]
        for nm, el in ws:
            ts.append(_Tensor(f"h{l}.{nm}", el * eb, role="weight"))
        acts = [("x", tokens * d), ("ln1", tokens * d), ("qkv", tokens * 3 * d), ("attn", tokens * d),
                ("o", tokens * d), ("ln2", tokens * d), ("fc1", tokens * ff), ("gelu", tokens * ff)]
        if attn_scores_bytes:
            ts.append(_Tensor(f"h{l}.scores", attn_scores_bytes, role="act"))
        for nm, el in acts:
            ts.append(_Tensor(f"h{l}.{nm}", el * eb, role="act"))
        if train:
            for nm, el in ws:
                ts.append(_Tensor(f"h{l}.{nm}.grad", el * eb, role="grad"))
            for nm, el in acts[:6]:
                ts.append(_Tensor(f"h{l}.{nm}.dgrad", el * eb, role="act"))
    ts.append(_Tensor("lnf.w", d * eb, role="weight"))
    ts.append(_Tensor("logits", tokens * min(vocab, 8192) * eb, role="act"))
    ts.append(_Tensor("workspace", 32 * MiB, role="workspace"))
    return ts


def _dl_kernels(b: _Builder, tensors, n_kernels, rng, cdf_off=None, embed_rows=0, embed_row_elems=0, eb=4,
                stray_every=97, gap_regions=(), oow_base=None, tokens=0):
    """Kernel sequence of a layered model: every kernel touches a small, time-local
    set of tensors (one layer's weights re-read as tiles, that layer's activations
    swept), so per-kernel footprints are much smaller than the whole footprint (the
    working-set gap of P:801-803). Weights are persistent hot data re-read in every
    pass; activations are transient."""
    by_layer = {}
    globals_ = []
    for t in tensors:
        if t.name.startswith("h") and "." in t.name:
            l = int(t.name[1:t.name.index(".")])
            by_layer.setdefault(l, []).append(t)
        else:
            globals_.append(t)
    layers = sorted(by_layer)
    embed = [t for t in globals_ if t.role == "embed"]
    others = [t for t in globals_ if t.role != "embed"]
    # one pass = forward over layers then backward over layers (if grads exist)
    seq = []
    for l in layers:
        seq.append(("fwd", l))
    if any(t.role == "grad" for t in tensors):
        for l in reversed(layers):
            seq.append(("bwd", l))
    per_pass_layers = len(seq)
    k = 0
    while k < n_kernels:
        phase, l = seq[(k // 12) % per_pass_layers] if per_pass_layers else ("fwd", 0)
        sub = k % 12
        lt = by_layer[l]
        weights = [t for t in lt if t.role == "weight"]
        grads = [t for t in lt if t.role == "grad"]
        acts = [t for t in lt if t.role == "act"]
        parts = []
        if sub == 0 and embed and embed_rows and l == layers[0]:
            # embedding gather (fwd) / gradient scatter (bwd): one Zipf-drawn row per
            # token, read in full (P:916-920 hot blocks); plus the activation write
            parts.append((tokens * embed_row_elems, b.zipf(embed[0].base, embed_rows, embed_row_elems, eb, cdf_off)))
            parts.append((acts[0].size // 16, b.sweep(acts[0].base, acts[0].size, 16)))
        else:
            w = weights[sub % len(weights)] if weights else None
            a_in = acts[sub % len(acts)]
            a_out = acts[(sub + 1) % len(acts)]
            if w is not None and w.size >= 64 * 1024:
                parts.append((w.size // 16 * 2, b.tiled(w.base, w.size, 16)))
            elif w is not None:
                parts.append((w.size // 4, b.sweep(w.base, w.size, 4)))
            parts.append((a_in.size // 16, b.sweep(a_in.base, a_in.size, 16)))
            parts.append((a_out.size // 16, b.sweep(a_out.base, a_out.size, 8)))
            if phase == "bwd" and grads:
                g = grads[sub % len(grads)]
                parts.append((g.size // 8, b.sweep(g.base, g.size, 8)))
            if sub == 5 and a_in.size >= 1 << 16:
                # attention-style scattered access: permutation inside one activation
                parts.append((a_in.size // 64, b.perm(a_in.base, a_in.size, 4)))
            if sub == 9 and a_out.size >= 1 << 16:
                parts.append((a_out.size // 256, b.strided(a_out.base, a_out.size, 12)))
            if sub == 11 and others:
                o = others[(k // 12) % len(others)]
                parts.append((o.size // 16 + 1, b.sweep(o.base, o.size - o.size % 16 or 16, 16)))
        if stray_every and k % stray_every == stray_every - 1:
            tot = sum(p[0] for p in parts)
            wgt = max(1, tot // 200)  # ~1% of every 97th kernel => ~0.01-0.02% overall
            if gap_regions:
                g = gap_regions[(k // stray_every) % len(gap_regions)]
                parts.append((wgt, b.stray(g[0], g[1], 4)))
            if oow_base is not None:
                parts.append((wgt, b.stray(oow_base, 2 * MiB, 4)))
        b.add_kernel(parts)
        k += 1


def plan_dl(name: str, seed: int, n: int, *, window: int, page_shift: int, n_layers: int, d: int, ff: int,
            vocab: int, tokens: int, eb: int, train: bool, n_kernels: int, chunk_min: int = 2 * MiB,
            topk=(1024,), want_kernel_rows=True, want_kernel_pages=False, embed_row_elems=None,
            attn_scores_bytes=0, extra_tensors=0, va_lo=0x7E0000000000, note=""):
    tensors = _transformer_tensors(n_layers, d, ff, vocab, tokens, eb, train, attn_scores_bytes)
    rng = random.Random(seed ^ 0x5EED)
    for i in range(extra_tensors):
        tensors.append(_Tensor(f"misc{i}", (rng.randrange(1, 64) * 16 * 1024), role="workspace"))
    al = _place(tensors, va_lo, chunk_min)
    top = al.next
    if top > va_lo + window:
        raise ValueError(f"{name}: tensors need {(top - va_lo) / GiB:.2f} GiB > window {window / GiB:.2f} GiB")
    b = _Builder(seed)
    cdf_off = None
    erows = 0
    if embed_row_elems:
        erows = vocab
        cdf_off = b.zipf_table(vocab)
    gaps = list(al.holes)
    # chunk tails (free space inside chunks) are also gaps: take power-of-two aligned pieces
    for a, ln in al.free:
        if ln >= 64 * 1024:
            sz = _pow2_floor(min(ln, 2 * MiB))
            start = (a + sz - 1) // sz * sz
            if start + sz <= a + ln:
                gaps.append((start, sz))
    oow = va_lo + window + 2 * MiB if va_lo + window + 4 * MiB < (1 << 64) else None
    _dl_kernels(b, tensors, n_kernels, rng, cdf_off, erows, embed_row_elems or 0, eb,
                gap_regions=gaps[:64], oow_base=oow, tokens=tokens)
    ko, st, cdf = b.finish(n)
    allocs = [(t.base, t.size) for t in tensors]
    return Plan(name, seed, n, va_lo, va_lo + window, page_shift, allocs, ko, st, cdf, topk=list(topk),
                want_kernel_rows=want_kernel_rows, want_kernel_pages=want_kernel_pages, note=note,
                objects=list(al.chunks))


def plan_rn50(seed: int = 42, n: int = 500_000_000) -> Plan:
    """Config 2: ResNet-50-training-step-shaped: ~300 tensor allocations, ~3000
    kernels, 4 KiB pages over a 4.5 GiB window. Built
    from the decoder template with CNN-like sizes: 16 'stages' of conv-like weights."""
    p = plan_dl("rn50", seed, n, window=4608 * MiB, page_shift=12, n_layers=8, d=512, ff=2048, vocab=1000,
                tokens=8192, eb=4, train=True, n_kernels=3000, extra_tensors=12, topk=(16, 1024),
                want_kernel_rows=True, note="~300 tensors, 3000 kernels, fp32 training step")
    return p


def plan_gpt2m(seed: int = 42, n: int = 2_000_000_000) -> Plan:
    """Config 3: GPT-2-medium fwd/bwd: 24 layers, d=1024, fp32, ~1000 tensors incl.
    the 50257x1024 embedding (Zipf-gathered), ~4000 kernels, 16 GiB window, 4 KiB."""
    return plan_dl("gpt2m", seed, n, window=16 * GiB, page_shift=12, n_layers=24, d=1024, ff=4096, vocab=50257,
                   tokens=4096, eb=4, train=True, n_kernels=4000, embed_row_elems=1024,
                   attn_scores_bytes=64 * MiB, topk=(1024,), want_kernel_rows=True,
                   note="GPT-2 345M train b4 s1024, fp32")


def plan_uvm(seed: int = 42, n: int = 4_000_000_000) -> Plan:
    """Config 4: UVM oversubscription: 400 GiB managed window at 2 MiB pages, ~200
    pool chunks of >= 2 GiB holding ~2000 tensors (tensor-level registration,
    P:899-902), 2000 kernels, per-kernel 2 MiB page bitmaps, top-68266 and top-1024."""
    return plan_dl("uvm", seed, n, window=400 * GiB, page_shift=21, n_layers=44, d=10240, ff=4 * 10240,
                   vocab=50257, tokens=4096, eb=2, train=True, n_kernels=2000, chunk_min=2 * GiB,
                   topk=(68266, 1024), want_kernel_rows=True, want_kernel_pages=True,
                   note="~175B-class bf16 model, 3x oversubscription of a 133 GB GPU")


def plan_llama(seed: int = 42, n: int = 10 * (1 << 30)) -> Plan:
    """Config 5: Llama-style DP trace: 32 layers, d=4096, ff=11008, bf16, ~1500
    tensors, ~10000 kernels, 64 GiB window at 4 KiB pages (P = 16,777,216)."""
    return plan_dl("llama", seed, n, window=64 * GiB, page_shift=12, n_layers=32, d=4096, ff=11008,
                   vocab=32000, tokens=4096, eb=2, train=True, n_kernels=10000, embed_row_elems=4096,
                   topk=(1024,), want_kernel_rows=True, note="Llama-7B-shaped bf16 train step, s4096")


# ----------------------------------------------------------------------------------------
# stress rows (SURVEY.md section 8d "Stress rows"; reported separately, never the headline)
# ----------------------------------------------------------------------------------------
def plan_s_perm(seed: int = 42, n: int = 2_000_000_000) -> Plan:
    """S-perm: the gpt2m plan with every stream replaced by the permutation pattern over
    the same allocation (its largest power-of-two prefix), element size 4: worst-case
    locality -- consecutive records of a stream land on unrelated pages of the tensor.
    Stray streams stay strays (they are already scattered). Same allocations, kernels and
    record counts as gpt2m."""
    p = plan_gpt2m(seed, n)
    rng = random.Random(seed ^ 0x9E7A)
    st = p.streams.copy()
    for r in range(st.shape[0]):
        if int(st[r, 1]) == STRAY:
            continue
        base, S = int(st[r, 2]), int(st[r, 3])
        S2 = _pow2_floor(S)
        e = 4 if S2 >= 4 else 1
        M = S2 // e
        st[r, 1:7] = [PERM, base, S2, e, (rng.getrandbits(40) << 1) | 1, rng.randrange(M)]
    p.streams = st
    p.name = "s_perm"
    p.note = "gpt2m with every stream a permutation (scattered pages inside each tensor)"
    return p


def plan_s_hot(seed: int = 42, n: int = 1 << 31) -> Plan:
    """S-hot: 2^31 records all on one 4 KiB page (one 4 KiB allocation), 1,000 kernels
    alternating a sweep (e = 8, every lane a different word) and a permutation (e = 4) of
    the page: maximum same-address contention on one page counter and one alloc bin."""
    va_lo = 0x7D0000000000
    b = _Builder(seed)
    page = va_lo + 0x1000 * 37
    allocs = [(page, 4096)]
    for k in range(1000):
        b.add_kernel([(1, b.sweep(page, 4096, 8) if k % 2 == 0 else b.perm(page, 4096, 4))])
    ko, st, cdf = b.finish(n)
    return Plan("s_hot", seed, n, va_lo, va_lo + 2 * MiB, 12, allocs, ko, st, cdf, topk=[16],
                want_kernel_rows=True, want_kernel_pages=False,
                note="2^31 records on one 4 KiB page, 1000 kernels", objects=[(va_lo, 2 * MiB)])


def plan_s_manyranges(seed: int = 42, n: int = 500_000_000, A: int = 65_536) -> Plan:
    """S-manyranges: the rn50 kernel sequence with A = 65,536 live ranges (the range table
    no longer fits shared memory: the scan's global-memory table). The rn50 tensors plus
    small tensors (512 B .. 32 KiB, 512 B steps) up to A; every kernel also sweeps 24 of
    the small tensors in turn (all of them over the 3,000 kernels; ~30 % of the records), so
    interval changes and table searches are frequent. 8 GiB window at 4 KiB pages."""
    window = 8 * GiB
    va_lo = 0x7E0000000000
    tensors = _transformer_tensors(8, 512, 2048, 1000, 8192, 4, True)
    rng = random.Random(seed ^ 0xA11C)
    rng2 = random.Random(seed ^ 0x5EED)
    base_count = len(tensors)
    for i in range(A - base_count):
        tensors.append(_Tensor(f"small{i}", 512 * rng.randrange(1, 65), role="workspace"))
    small = tensors[base_count:]
    al = _place(tensors, va_lo, 2 * MiB)
    assert al.next <= va_lo + window
    b = _Builder(seed)
    gaps = list(al.holes)
    _dl_kernels(b, tensors[:base_count], 3000, rng2, gap_regions=gaps[:64], oow_base=va_lo + window + 2 * MiB)
    per = 24
    w_base = sum(int(w) for parts in b.kernels for w, _ in parts)
    w_small = sum(small[i % len(small)].size // 8 for i in range(len(b.kernels) * per))
    rep = max(1, -(-3 * w_base // (7 * w_small)))  # small tensors get ~30 % of the records
    for k, parts in enumerate(b.kernels):
        for q in range(per):
            t = small[(k * per + q) % len(small)]
            parts.append((rep * (t.size // 8), b.sweep(t.base, t.size, 8)))
    ko, st, cdf = b.finish(n)
    allocs = [(t.base, t.size) for t in tensors]
    return Plan("s_manyranges", seed, n, va_lo, va_lo + window, 12, allocs, ko, st, cdf, topk=[16, 1024],
                want_kernel_rows=True, want_kernel_pages=False,
                note=f"rn50 kernels + {A - base_count} small tensors (A = {A})", objects=list(al.chunks))


CONFIGS = {
    "tiny": plan_tiny,
    "rn50": plan_rn50,
    "gpt2m": plan_gpt2m,
    "uvm": plan_uvm,
    "llama": plan_llama,
    "s_perm": plan_s_perm,
    "s_hot": plan_s_hot,
    "s_manyranges": plan_s_manyranges,
}
STRESS = ("s_perm", "s_hot", "s_manyranges")


def build_plan(name: str, seed: int = 42, n: int | None = None) -> Plan:
    f = CONFIGS[name]
    return f(seed) if n is None else f(seed, n)
