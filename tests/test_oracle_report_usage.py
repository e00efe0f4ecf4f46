"""Pins of the oracle's signed-size registration (SURVEY.md 8(b) deferred helper;
include/pasta.h pasta_report_memory_usage; CPU only).

P:540 names c10::reportMemoryUsage as PASTA's PyTorch hook; SPEC S:121-124 fixes its
dialect: "a single signed size (negative = release, no action flag)", normalized to
positive sizes with an action (S:48, S:118-120 RawEventNVX). The pin: a random RMX
event stream through report_memory_usage gives exactly the statuses, ids, live tables
and analysis results of the same stream converted to the NVX form (positive size +
action) and fed to the already-pinned register_* / *_free calls, at the object level
and at the tensor level; plus the error cases the header states.
"""
import random

import numpy as np
import pytest

import oracle
from oracle import OracleTrace


@pytest.fixture(autouse=True)
def _lib(built):
    return built


def _to_nvx(events):
    """RMX (ptr, signed size) -> NVX (ptr, positive size, action)."""
    return [(p, abs(d), "alloc" if d > 0 else "free") for p, d in events]


def _rmx_stream(rng, base, n_slots, n_events):
    """Allocate / release events over n_slots 4 KiB-aligned slots; some releases carry a
    wrong size, some name no live range, a few sizes are zero."""
    live = {}
    ev = []
    for _ in range(n_events):
        s = rng.randrange(n_slots)
        p = base + s * 65536
        r = rng.random()
        if r < 0.03:
            ev.append((p, 0))
        elif s in live and r < 0.6:
            sz = live.pop(s)
            ev.append((p, -(sz + (1 if rng.random() < 0.1 else 0))))
            if ev[-1][1] != -sz:
                live[s] = sz
        elif s not in live:
            sz = rng.randint(1, 65536)
            live[s] = sz
            ev.append((p, sz))
        else:
            ev.append((p + 8, -1))  # no live range starts here
    return ev


def _replay_nvx(o, events, tensors):
    out = []
    for p, sz, act in events:
        if sz == 0:
            out.append((oracle.EINVAL, None))
            continue
        table = o.tlive if tensors else o.live
        if act == "alloc":
            out.append(o.register_tensor(p, sz) if tensors else o.register_alloc(p, sz))
        elif p not in table:
            out.append((oracle.ENOENT, None))
        elif table[p][0] != sz:
            out.append((oracle.EINVAL, None))
        else:
            ident = table[p][1]
            out.append(((o.register_tensor_free(p) if tensors else o.register_free(p)), ident))
    return out


def _analyze(o, rng, lo, hi):
    rec = np.array([rng.randrange(lo, hi) for _ in range(5000)], dtype=np.uint64)
    o.analyze(rec, [0, 2000, 5000], 12, kernel_rows=True)
    return o


def test_rmx_stream_equals_nvx_registration():
    rng = random.Random(540)
    base = 0x7F0000000000
    for tensors in (False, True):
        for trial in range(20):
            ev = _rmx_stream(rng, base, 24, 300)
            kw = dict(max_live_tensors=64, max_tensor_ids=400) if tensors else {}
            a = OracleTrace(base, base + (1 << 24), 64, 400, **kw)
            b = OracleTrace(base, base + (1 << 24), 64, 400, **kw)
            if tensors:  # one object holding every tensor slot
                assert a.register_alloc(base, 24 * 65536)[0] == oracle.OK
                assert b.register_alloc(base, 24 * 65536)[0] == oracle.OK
            got = [a.report_memory_usage(p, d) for p, d in ev]
            want = _replay_nvx(b, _to_nvx(ev), tensors)
            assert got == want, (tensors, trial)
            assert a.live == b.live and a.tlive == b.tlive
            seed = rng.random()
            ra = _analyze(a, random.Random(seed), base, base + 24 * 65536)
            rb = _analyze(b, random.Random(seed), base, base + 24 * 65536)
            assert np.array_equal(ra.alloc_counts, rb.alloc_counts)
            assert np.array_equal(ra.kernel_rows, rb.kernel_rows)
            if tensors:
                assert np.array_equal(ra.tensor_counts, rb.tensor_counts)


def test_report_usage_errors():
    base = 0x10000000
    o = OracleTrace(base, base + (1 << 24), 4, 8)
    assert o.report_memory_usage(base, 0) == (oracle.EINVAL, None)
    assert o.report_memory_usage(base, -(1 << 63)) == (oracle.EINVAL, None)
    assert o.report_memory_usage(base, 4096) == (oracle.OK, 0)
    assert o.report_memory_usage(base + 100, 4096)[0] == oracle.EOVERLAP
    assert o.report_memory_usage(base, -4095) == (oracle.EINVAL, None)  # wrong size: nothing released
    assert base in o.live
    assert o.report_memory_usage(base + 4096, -10) == (oracle.ENOENT, None)
    assert o.report_memory_usage(base, -4096) == (oracle.OK, 0)
    assert o.report_memory_usage(base, 4096) == (oracle.OK, 1)  # ids are never reused
