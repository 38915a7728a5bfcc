"""The hot path replaces int/int divisions (the itl L-average, simengine.py:235-237,
and the admission estimate's L, sched_scorpio.py:104) by a reciprocal-table
division with one FMA correction (div_small, sl_device.cuh).  It must equal the
correctly rounded quotient -- Python's int / int -- bit for bit: exhaustively for
small numerators and on random numerators up to 2^53."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    import torch

    from paper_2505_23022_b200 import _native as N

    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    out = torch.empty_like(ta)
    rc = N.lib().sl_selftest_div_small(ta.data_ptr(), tb.data_ptr(), out.data_ptr(), a.size,
                                       torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    return out.cpu().numpy()


def test_div_small_exhaustive_small_numerators():
    a0 = np.arange(1 << 20, dtype=np.float64)
    for b in range(1, 131):
        bb = np.full(a0.size, b, np.int32)
        got = _run(a0, bb)
        want = a0 / np.float64(b)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), b


def test_div_small_random_large_numerators():
    rng = np.random.default_rng(7)
    n = 1 << 22
    for hi in (32, 40, 53):
        a = np.floor(rng.random(n) * 2.0 ** hi)
        b = rng.integers(1, 131, n).astype(np.int32)
        got = _run(a, b)
        want = a / b.astype(np.float64)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), hi
