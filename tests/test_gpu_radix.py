"""K1 (onesweep LSD radix sort) against numpy's stable argsort: keys and the
stable order of values, bit-exact."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2406_18111_b200 import build
    build.build()
    from paper_2406_18111_b200 import Context
    return Context(0)


@pytest.mark.parametrize("n,lo,hi,dup", [(0, 0, 64, 1), (1, 0, 64, 1), (4095, 0, 64, 1), (4097, 3, 17, 1),
                                         (100_003, 0, 41, 1), (100_003, 0, 41, 5000), (300_001, 5, 59, 7),
                                         (1 << 20, 0, 64, 1), (65536, 10, 11, 1)])
def test_radix_sort_stable(ctx, n, lo, hi, dup):
    rng = np.random.default_rng(n + lo)
    k = rng.integers(0, 2**63, size=n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=n, dtype=np.uint64)
    if dup > 1:  # heavy duplicates
        k = k[rng.integers(0, max(n // dup, 1), size=n)] if n else k
    v = np.arange(n, dtype=np.uint32)
    mask = np.uint64(((1 << (hi - lo)) - 1) << lo) if hi - lo < 64 else np.uint64(2**64 - 1)
    sk = (k & mask) >> np.uint64(lo)
    order = np.argsort(sk, kind="stable")
    dk = torch.from_numpy(k.copy()).cuda()
    dv = torch.from_numpy(v.view(np.int32).copy()).cuda()
    ctx.radix_sort(dk, dv, lo, hi)
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), v[order])
    assert np.array_equal(dk.cpu().numpy(), k[order])
