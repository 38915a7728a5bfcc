"""Output-length prediction (slosim.predictor API, pkg/src/slosim/predictor.py).

``Bucketing`` carries the boundary table; ``LengthPredictor.predict_batch`` runs
the predictor for many requests in one device launch (``sl_predict_batch``):
oracle mode returns the true length, ``noisy_bucket`` perturbs the true bucket
with numpy's ``default_rng([rng_seed, id])`` stream replicated on device
(predictor.py:115-126).  Predictions depend only on (rng_seed, id, length), so a
sweep computes them once per trace and shares them across SLO scales.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import Request

EQUAL_WIDTH = "equal_width"
EQUAL_FREQUENCY = "equal_frequency"
ORACLE = "oracle"
NOISY_BUCKET = "noisy_bucket"


@dataclass(frozen=True)
class Bucketing:
    """Half-open length intervals ``(b[k-1], b[k]]`` (predictor.py:34-90)."""

    strategy: str
    num_buckets: int
    max_len: int
    boundaries: tuple[float, ...]

    def __post_init__(self) -> None:
        if self.num_buckets < 1:
            raise ValueError("num_buckets must be >= 1")
        if len(self.boundaries) != self.num_buckets:
            raise ValueError("boundary count must equal num_buckets")
        if any(hi <= lo for lo, hi in zip(self.boundaries, self.boundaries[1:])):
            raise ValueError("boundaries must be strictly increasing")

    @classmethod
    def equal_width(cls, num_buckets: int, max_len: int) -> "Bucketing":
        if max_len < num_buckets:
            raise ValueError("max_len must be >= num_buckets")
        return cls(EQUAL_WIDTH, num_buckets, max_len,
                   tuple(max_len * k / num_buckets for k in range(1, num_buckets + 1)))

    @classmethod
    def equal_frequency(cls, num_buckets: int, sample: list[int]) -> "Bucketing":
        if not sample:
            raise ValueError("equal-frequency bucketing needs a training sample")
        qs = [k / num_buckets for k in range(1, num_buckets + 1)]
        bounds = tuple(float(q) for q in np.quantile(np.asarray(sample, float), qs))
        if any(hi <= lo for lo, hi in zip(bounds, bounds[1:])):
            raise ValueError("sample too tied for equal-frequency bucketing: duplicate quantiles")
        return cls(EQUAL_FREQUENCY, num_buckets, int(max(sample)), bounds)

    def bucket_of(self, length: int) -> int:
        """Interval index of ``length``; above the last boundary clamps to the last."""
        if length < 1:
            raise ValueError("length must be >= 1")
        if length > self.boundaries[-1]:
            return self.num_buckets - 1
        lo, hi = 0, self.num_buckets
        while lo < hi:
            mid = (lo + hi) // 2
            if self.boundaries[mid] < length:
                lo = mid + 1
            else:
                hi = mid
        return lo

    def representative(self, bucket: int) -> int:
        if not 0 <= bucket < self.num_buckets:
            raise ValueError(f"bucket index {bucket} out of range")
        lo = self.boundaries[bucket - 1] if bucket else 0.0
        return max(1, math.ceil((lo + self.boundaries[bucket]) / 2.0))


@dataclass(frozen=True)
class LengthPredictor:
    """Oracle or bucket-noise predictor (predictor.py:93-126)."""

    mode: str
    bucketing: Bucketing
    error_prob: float = 0.0
    error_spread: int = 1
    rng_seed: int = 0

    def __post_init__(self) -> None:
        if self.mode not in (ORACLE, NOISY_BUCKET):
            raise ValueError(f"unknown predictor mode {self.mode!r}")
        if not 0.0 <= self.error_prob <= 1.0:
            raise ValueError("error_prob must be in [0, 1]")
        if self.error_spread < 1:
            raise ValueError("error_spread must be a positive integer")

    def predict(self, req: Request) -> int:
        if self.mode == ORACLE:
            return req.true_output_len
        return int(predict_many(self, np.array([req.id]), np.array([req.true_output_len]))[0])

    def predict_batch(self, ids: np.ndarray, true_out: np.ndarray, device=None,
                      return_clamps: bool = False):
        """Predicted lengths for many requests in one device launch (host arrays
        in, host array out; see predict_device for device tensors)."""
        return predict_many(self, ids, true_out, device, return_clamps)

    def predict_device(self, ids_t, true_out_t, stream=None):
        """Device tensors in (int64 ids, int32 lengths), device tensor out."""
        return predict_device(self, ids_t, true_out_t, stream)


def predict_many(predictor, ids: np.ndarray, true_out: np.ndarray, device=None,
                 return_clamps: bool = False):
    """``predictor.predict`` for many requests in one launch.  ``predictor`` is
    any LengthPredictor-shaped object (this package's or the reference's,
    predictor.py:93-126): only its fields are read."""
    torch = N.require_cuda()
    dev = torch.device(device if device is not None else "cuda")
    ids_t = torch.from_numpy(np.ascontiguousarray(ids, np.int64)).to(dev)
    tout_t = torch.from_numpy(np.ascontiguousarray(true_out, np.int32)).to(dev)
    out, clamps = predict_device(predictor, ids_t, tout_t)
    res = out.cpu().numpy()
    return (res, int(clamps.item())) if return_clamps else res


def predict_device(predictor, ids_t, true_out_t, stream=None):
    """Device tensors in (int64 ids, int32 lengths), device tensor out."""
    torch = N.require_cuda()
    p_ = predictor
    if len(ids_t) and int(true_out_t.min().item()) < 1:
        raise ValueError("length must be >= 1")
    if p_.rng_seed < 0 or p_.rng_seed >= 1 << 64 or (len(ids_t) and int(ids_t.min().item()) < 0):
        raise ValueError("seed and request ids must be non-negative 64-bit integers")
    dev = ids_t.device
    bk = p_.bucketing
    bounds = torch.tensor([float(b) for b in bk.boundaries], dtype=torch.float64, device=dev)
    out = torch.empty(len(ids_t), dtype=torch.int32, device=dev)
    clamps = torch.zeros(1, dtype=torch.int64, device=dev)
    p = N.SlPredictor(N.PREDICT_ORACLE if p_.mode == ORACLE else N.PREDICT_NOISY_BUCKET,
                      int(bk.num_buckets), bounds.data_ptr(), float(p_.error_prob),
                      int(p_.error_spread), 0, int(p_.rng_seed))
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    rc = N.lib().sl_predict_batch(ids_t.data_ptr(), true_out_t.data_ptr(), len(ids_t),
                                  C.byref(p), out.data_ptr(), clamps.data_ptr(), s.cuda_stream)
    if rc != 0:
        raise RuntimeError(f"sl_predict_batch failed with code {rc}")
    return out, clamps
