"""Batch planning of the streaming mode (host logic, CPU only)."""
import numpy as np

from paper_2602_22103_b200.stream import plan_batches


def test_plan_batches_cover_and_rebase():
    ko = [0, 5, 5, 17, 40, 41, 100]
    n = 100
    for batch in (1, 3, 7, 16, 40, 100, 1000):
        bs = plan_batches(ko, n, batch)
        assert bs[0][0] == 0 and bs[-1][1] == n
        for (a, b, k0, sub), nxt in zip(bs, bs[1:] + [None]):
            if nxt is not None:
                assert nxt[0] == b
            assert sub[0] == 0 and sub[-1] == b - a and np.all(np.diff(sub) >= 0)
            # every record j of the batch maps to the same kernel as in the global offsets
            for j in range(a, b):
                kg = int(np.searchsorted(ko, j, side="right")) - 1
                kl = int(np.searchsorted(sub, j - a, side="right")) - 1
                assert k0 + kl == kg, (batch, a, j)
