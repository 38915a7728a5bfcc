"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the C restatement (liborc.so).

Only tests/, ``__graft_entry__.smoke()`` and bench.py (cpu_baseline leg and
``--impl reference``) may import this module, as the parity checker or the
CPU baseline.  The product package never imports it.

``run_sim`` restates ``slosim.simengine.run`` (pkg/src/slosim/simengine.py:168)
for one simulation over SoA numpy arrays that are already rate/SLO scaled.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liborc.so")

POLICY = {"scorpio": 0, "greedy": 1, "sjf": 2, "early_reject": 3}
FLAG_TTFT_GUARD, FLAG_TPOT_GUARD, FLAG_R_ONLY, FLAG_HAS_HORIZON, FLAG_PREFILL_PRIORITY = 1, 2, 4, 8, 16
STATUS_NAMES = ("completed", "rejected_ttft", "rejected_admission", "incomplete")


class Cost(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("alpha", "beta", "gamma", "delta", "epsilon", "phi", "theta", "alpha_p", "beta_p")]


class SimParams(C.Structure):
    _fields_ = [("policy", C.c_int32), ("flags", C.c_int32), ("max_batch_size", C.c_int32),
                ("_pad", C.c_int32), ("horizon", C.c_double), ("cost", Cost)]


class Trace(C.Structure):
    _fields_ = [("n", C.c_int64), ("arrival", C.c_void_p), ("ttft_slo", C.c_void_p),
                ("tpot_slo", C.c_void_p), ("prompt_len", C.c_void_p), ("true_out", C.c_void_p),
                ("id", C.c_void_p), ("predicted", C.c_void_p)]


class Outcomes(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("status", "compliant", "completion_step",
                                          "first_token_time", "completion_time", "ttft", "tpot")]


SUMMARY_FIELDS = ("status", "n_steps", "n_plans", "n_idle_skips", "request_steps", "total",
                  "completed", "compliant", "rejected_ttft", "rejected_admission", "incomplete",
                  "ttft_violations", "tpot_violations")


class Summary(C.Structure):
    _fields_ = [(n, C.c_int64) for n in SUMMARY_FIELDS] + [
        ("sim_end", C.c_double), ("horizon", C.c_double), ("goodput", C.c_double),
        ("adherence", C.c_double), ("digest", C.c_uint64)]


class Log(C.Structure):
    _fields_ = [("step_cap", C.c_int64), ("id_cap", C.c_int64)] + [
        (n, C.c_void_p) for n in ("now", "end", "prefill_s", "decode_s", "vbs", "min_slo",
                                  "n_admitted", "n_rejected", "n_batch", "ids")] + [
        ("n_steps", C.c_int64), ("n_ids", C.c_int64), ("overflow", C.c_int32)]


_lib = None


def build() -> str:
    """Compile liborc.so with the committed Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.orc_run.argtypes = [C.POINTER(Trace), C.POINTER(SimParams), C.POINTER(Outcomes),
                              C.POINTER(Summary), C.POINTER(Log)]
        L.orc_run.restype = C.c_int
        L.orc_digest_item.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64]
        L.orc_digest_item.restype = C.c_uint64
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def make_params(policy="scorpio", ttft_guard=True, tpot_guard=True, admission_min="r_prime",
                horizon=None, max_batch_size=256, prefill_priority=False, itl=None,
                prefill=None) -> SimParams:
    """``itl`` = (alpha, beta, gamma, delta, epsilon); ``prefill`` = (phi, theta, alpha_p, beta_p)."""
    flags = 0
    if ttft_guard:
        flags |= FLAG_TTFT_GUARD
    if tpot_guard:
        flags |= FLAG_TPOT_GUARD
    if admission_min == "r_only":
        flags |= FLAG_R_ONLY
    if horizon is not None:
        flags |= FLAG_HAS_HORIZON
    if prefill_priority:
        flags |= FLAG_PREFILL_PRIORITY
    a, b, g, d, e = itl
    phi, th, ap, bp = prefill
    cost = Cost(a, b, g, d, e, phi, th, ap, bp)
    return SimParams(POLICY[policy], flags, int(max_batch_size), 0,
                     float(horizon) if horizon is not None else 0.0, cost)


def run_sim(arrival, ttft_slo, tpot_slo, prompt_len, true_out, ids, predicted, params: SimParams,
            log_steps: int = 0, log_ids: int = 0) -> dict:
    """Run one simulation; arrays are per request in trace (arrival) order."""
    n = len(arrival)
    arrs = [np.ascontiguousarray(arrival, np.float64), np.ascontiguousarray(ttft_slo, np.float64),
            np.ascontiguousarray(tpot_slo, np.float64), np.ascontiguousarray(prompt_len, np.int32),
            np.ascontiguousarray(true_out, np.int32), np.ascontiguousarray(ids, np.int64),
            np.ascontiguousarray(predicted, np.int32)]
    tr = Trace(n, *[_ptr(a) for a in arrs])
    m = max(n, 1)
    out = {
        "status": np.empty(m, np.int8), "compliant": np.empty(m, np.int8),
        "completion_step": np.empty(m, np.int32), "first_token_time": np.empty(m),
        "completion_time": np.empty(m), "ttft": np.empty(m), "tpot": np.empty(m),
    }
    oc = Outcomes(*[_ptr(out[k]) for k in ("status", "compliant", "completion_step",
                                           "first_token_time", "completion_time", "ttft", "tpot")])
    sm = Summary()
    lg = None
    logbufs = None
    if log_steps:
        logbufs = {k: np.zeros(log_steps) for k in ("now", "end", "prefill_s", "decode_s", "vbs",
                                                     "min_slo")}
        for k in ("n_admitted", "n_rejected", "n_batch"):
            logbufs[k] = np.zeros(log_steps, np.int32)
        logbufs["ids"] = np.zeros(max(log_ids, 1), np.int64)
        lg = Log(log_steps, log_ids, *[_ptr(logbufs[k]) for k in (
            "now", "end", "prefill_s", "decode_s", "vbs", "min_slo", "n_admitted", "n_rejected",
            "n_batch", "ids")], 0, 0, 0)
    rc = lib().orc_run(C.byref(tr), C.byref(params), C.byref(oc), C.byref(sm),
                       C.byref(lg) if lg is not None else None)
    res = {k: v[:n] for k, v in out.items()}
    res["rc"] = rc
    res["summary"] = {f: getattr(sm, f) for f, _ in Summary._fields_}
    if lg is not None:
        ns, ni = lg.n_steps, lg.n_ids
        res["log"] = {k: v[:ns] for k, v in logbufs.items() if k != "ids"}
        res["log"]["ids"] = logbufs["ids"][:ni]
        res["log"]["overflow"] = lg.overflow
    return res


def digest_item(step: int, tag: int, pos: int, val: int) -> int:
    return lib().orc_digest_item(step, tag, pos, val & 0xFFFFFFFFFFFFFFFF)


def run_many(jobs, threads: int | None = None) -> list[dict]:
    """Run independent sims on host threads (ctypes drops the GIL per call).

    ``jobs`` is a list of kwargs dicts for :func:`run_sim`.
    """
    threads = threads or len(os.sched_getaffinity(0))
    lib()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda kw: run_sim(**kw), jobs))
