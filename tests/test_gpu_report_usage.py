"""GPU parity of pasta_report_memory_usage (signed-size registration, P:540
c10::reportMemoryUsage): random signed-size event streams through the
C ABI and through the oracle give the same statuses and ids, and the analysis of the
same records after them is bit-exact, at the object level and at the tensor level."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2602_22103_b200 as pb  # noqa: E402
import oracle  # noqa: E402
from oracle import OracleTrace  # noqa: E402
from tests.harness import u64  # noqa: E402
from tests.test_oracle_report_usage import _rmx_stream  # noqa: E402

DEV = torch.device("cuda:0")


def _gpu_event(tr, p, d):
    try:
        return oracle.OK, tr.report_memory_usage(p, d)
    except pb.PastaError as e:
        return e.status, None


@pytest.mark.parametrize("tensors", [False, True])
def test_report_usage_streams(tensors):
    rng = random.Random(1540 + tensors)
    base = 0x7F0000000000
    span = 24 * 65536
    for trial in range(6):
        ev = _rmx_stream(rng, base, 24, 400)
        kw = dict(max_live_tensors=64, max_tensor_ids=500) if tensors else {}
        tr = pb.Trace(DEV, base, base + (1 << 24), 64, 500, **kw)
        o = OracleTrace(base, base + (1 << 24), 64, 500, **kw)
        if tensors:
            tr.register_alloc(base, span)
            o.register_alloc(base, span)
        for p, d in ev:
            assert _gpu_event(tr, p, d) == o.report_memory_usage(p, d), (trial, p, d)
        rec = np.array([rng.randrange(base - 4096, base + span + 4096) for _ in range(200_000)], dtype=np.uint64)
        ko = [0, 50_000, 50_000, 200_000]
        h = tr.histograms(12, n_kernels=3, kernel_rows=True)
        tr.analyze(torch.from_numpy(rec.view(np.int64)).to(DEV), 12, h,
                   kernel_offsets=torch.tensor(ko, dtype=torch.int64, device=DEV))
        tr.sync()
        o.analyze(rec, ko, 12, kernel_rows=True)
        assert np.array_equal(u64(h.page_counts), o.page_counts)
        assert np.array_equal(u64(h.alloc_counts), o.alloc_counts)
        assert np.array_equal(u64(h.kernel_alloc_counts).reshape(3, -1), o.kernel_rows)
        assert u64(h.totals)[:3].tolist() == o.totals.tolist()
        if tensors:
            assert np.array_equal(u64(h.tensor_counts), o.tensor_counts)
            assert int(u64(h.totals)[pb.T_UNTENSORED]) == o.untensored
        tr.close()
