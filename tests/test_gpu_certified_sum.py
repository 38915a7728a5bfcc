"""The certified CPython sum (DD / dd_certify, sl_device.cuh) that replaces the
sequential sum(1/slo) and vbs folds of the few-large-segments guard
(sched_scorpio.py:121, 312-315; plan_large.cuh): whenever the certificate holds,
its value must equal CPython's own sum() of the same list bit for bit; sums whose
exact value sits on or next to a rounding midpoint -- where CPython's Neumaier
result and the correctly rounded sum can differ -- must not be certified."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(sums: list[list[float]]) -> np.ndarray:
    import torch

    from paper_2505_23022_b200 import _native as N

    x = np.concatenate([np.asarray(v, np.float64) for v in sums])
    begin = np.concatenate([[0], np.cumsum([len(v) for v in sums])]).astype(np.int64)
    tx, tb = torch.from_numpy(x).cuda(), torch.from_numpy(begin).cuda()
    out = torch.empty(3 * len(sums), dtype=torch.float64, device="cuda")
    rc = N.lib().sl_selftest_certified_sum(tx.data_ptr(), tb.data_ptr(), len(sums),
                                           out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    return out.cpu().numpy().reshape(-1, 3)


def _random_sums(seed: int) -> list[list[float]]:
    # Python floats: CPython's sum() takes its compensated float path only for
    # exact floats (numpy scalars are added plainly)
    rng = np.random.default_rng(seed)
    sums = []
    for n in (1, 2, 3, 31, 32, 33, 64, 100, 1000, 4096, 32768):
        sums.append(list(rng.uniform(0.5, 2.0, n)))
        # 1/slo and min/slo terms of the tiers (few distinct values: structured sums)
        tp = np.array([0.03, 0.05, 0.1])[rng.integers(0, 3, n)]
        sums.append(list(1.0 / tp))
        sums.append(list(0.03 / tp))
        sums.append(list(np.exp(rng.uniform(-14.0, 14.0, n))))  # wide dynamic range
        sums.append([1.0 / 0.03] * n)  # all equal
    return [[float(x) for x in v] for v in sums]


def test_certified_values_equal_cpython_sum():
    sums = _random_sums(1) + _random_sums(2)
    out = _run(sums)
    certified = 0
    for v, (r, _, _) in zip(sums, out):
        if not np.isnan(r):
            certified += 1
            assert r == sum(v), (len(v), r, sum(v))
    # the certificate fails only for sums within ~n^2 u^2 of a rounding midpoint:
    # sums of a few terms land exactly on one often (their exact sum has few bits
    # beyond the 53rd), long sums (the guard's folds) practically never
    assert certified >= 0.9 * len(sums)
    assert all(not np.isnan(r) for v, (r, _, _) in zip(sums, out) if len(v) >= 1000)


def test_midpoint_sums_are_not_certified():
    u = 2.0 ** -53
    cases = [
        [1.0, u],                    # exact midpoint (CPython: 1.0, ties to even)
        [1.0, u, 2.0 ** -100],       # just above it: RN(S) = 1 + 2u, but CPython returns 1.0
        [1.0] + [2.0 ** -60] * 128,  # a midpoint reached through the compensation term
        [3.0, 2 * u],                # midpoint in another binade
        [1.5, 0.5 - u],              # midpoint just below a power of two (half the gap)
        [3.0, 3 * u],                # near, not on, a midpoint: certified
        [1.5, 0.5 - u / 2],          # below a power of two, off the midpoint: certified
    ]
    out = _run(cases)
    for v, (r, _, _) in zip(cases, out):
        assert np.isnan(r) or r == sum(v), (v[:3], r, sum(v))
    assert all(np.isnan(out[i, 0]) for i in range(5))
    assert out[5, 0] == sum(cases[5]) and out[6, 0] == sum(cases[6])
