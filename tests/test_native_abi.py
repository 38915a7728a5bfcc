"""CPU-side checks of the C ABI: the library loads, its struct layouts match the
bindings, and it exports every symbol include/scorpio_b200.h declares."""

import ctypes as C

import numpy as np
import pytest


def test_library_exports_every_declared_symbol():
    from paper_2505_23022_b200 import _native as N

    L = N.lib()
    syms = N.exported_symbols()
    assert "sl_run_batch" in syms
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_abi_layout_matches_bindings():
    from paper_2505_23022_b200 import _native as N

    N._check_layout(N.lib())


@pytest.mark.parametrize("slos,scale,wide", [
    ([0.03, 0.05], 1.0, 0), ([0.03, 0.05], 2.0, 0), ([1.0, 10.0], 1.0, 0),
    ([0.01, 10.0], 1.0, 0), ([0.001, 10.0], 1.0, 1), ([0.03], 0.5, 0)])
def test_credit_params(slos, scale, wide):
    from paper_2505_23022_b200 import _native as N

    E, w = N.credit_params(np.array(slos), scale)
    assert w == wide
    for s in slos:
        v = s * scale
        S = np.ldexp(v, -E)
        assert S == np.floor(S) and S >= 1  # exact integer fixed point


def test_credit_params_rejects_bad_slo():
    from paper_2505_23022_b200 import _native as N

    with pytest.raises(ValueError):
        N.credit_params(np.array([0.0, 0.03]), 1.0)


def test_no_cpu_fallback_without_device():
    import torch

    from paper_2505_23022_b200 import _native as N

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(N.NativeUnavailable):
        N.require_cuda()
