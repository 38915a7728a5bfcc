"""Analytic latency models (slosim.costmodel API, pkg/src/slosim/costmodel.py:31-154).

Parameter records with the reference's validation, plus the scalar formulas for
callers of the API.  The device evaluates the same expressions, in the same
left-to-right unfused fp64 order, inside the kernels (sl_device.cuh); model
fitting is offline and out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

DECODE = "decode"
PREFILL = "prefill"


@dataclass(frozen=True)
class ItlParams:
    """Decode-iteration latency alpha*B*L + beta*B + gamma*L + delta; epsilon cushion."""

    alpha: float
    beta: float
    gamma: float
    delta: float
    epsilon: float = 1.1

    def __post_init__(self) -> None:
        if self.epsilon < 1.0:
            raise ValueError("epsilon must be >= 1.0")

    def as_tuple(self) -> tuple[float, float, float, float, float]:
        return itl_coeffs(self)


@dataclass(frozen=True)
class PrefillParams:
    """Prefill latency: phi up to theta tokens, alpha_p*n + beta_p beyond."""

    phi: float
    theta: float
    alpha_p: float
    beta_p: float

    def __post_init__(self) -> None:
        if self.phi <= 0:
            raise ValueError("phi must be positive")
        if self.theta < 0:
            raise ValueError("theta must be >= 0")
        if self.alpha_p * self.theta + self.beta_p < 0:
            raise ValueError("linear regime must be non-negative at theta")

    def as_tuple(self) -> tuple[float, float, float, float]:
        return prefill_coeffs(self)


def itl_coeffs(p) -> tuple[float, float, float, float, float]:
    """(alpha, beta, gamma, delta, epsilon) of any ItlParams-shaped object
    (this package's or the reference's, costmodel.py:31-47)."""
    return (float(p.alpha), float(p.beta), float(p.gamma), float(p.delta), float(p.epsilon))


def prefill_coeffs(p) -> tuple[float, float, float, float]:
    """(phi, theta, alpha_p, beta_p) of any PrefillParams-shaped object (costmodel.py:50-65)."""
    return (float(p.phi), float(p.theta), float(p.alpha_p), float(p.beta_p))


def itl(params: ItlParams, batch_size: float, avg_len: float) -> float:
    if batch_size <= 0:
        raise ValueError("batch_size must be positive")
    if avg_len <= 0:
        raise ValueError("avg_len must be positive")
    p = params
    return p.alpha * batch_size * avg_len + p.beta * batch_size + p.gamma * avg_len + p.delta


def estimated_tpot(params: ItlParams, vbs: float, avg_len: float, predicted_len: float) -> float:
    if vbs <= 0:
        raise ValueError("vbs must be positive")
    if avg_len <= 0:
        raise ValueError("avg_len must be positive")
    if predicted_len < 1:
        raise ValueError("predicted_len must be >= 1")
    p = params
    return p.epsilon * ((p.alpha * vbs + p.gamma) * (avg_len + predicted_len / 2.0)
                        + p.beta * vbs + p.delta)


def prefill_time(params: PrefillParams, prompt_len: int) -> float:
    if prompt_len < 1:
        raise ValueError("prompt_len must be >= 1")
    return params.phi if prompt_len <= params.theta else params.alpha_p * prompt_len + params.beta_p


def estimated_ttft(params: PrefillParams, queue_ahead: list[int], elapsed_wait: float) -> float:
    if not queue_ahead:
        raise ValueError("queue_ahead must include the request's own prompt")
    if elapsed_wait < 0:
        raise ValueError("elapsed_wait must be >= 0")
    return elapsed_wait + sum(prefill_time(params, n) for n in queue_ahead)
