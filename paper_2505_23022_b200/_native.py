"""Loader and ctypes mirror of the C ABI in include/scorpio_b200.h.

The CUDA library ``lib/libscorpio_b200.so`` is built in-tree (``build_native``)
for sm_100a.  There is no CPU fallback: every entry point that needs the GPU
raises ``NativeUnavailable`` when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_DIR = os.path.join(PKG, "lib")
LIB_PATH = os.environ.get("SL_LIB_PATH") or os.path.join(LIB_DIR, "libscorpio_b200.so")
INCLUDE = os.path.join(ROOT, "include")
CSRC = os.path.join(PKG, "csrc")
SOURCES = ("sim_kernel.cu", "plan_kernels.cu", "predict_kernel.cu", "report_kernel.cu")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]

# ---- constants (scorpio_b200.h)
SL_OK = 0
SIM_NO_WORK_RUNNING, SIM_NO_PROGRESS, SIM_LOG_OVERFLOW = 1, 2, 4
COMPLETED, REJECTED_TTFT, REJECTED_ADMISSION, INCOMPLETE = 0, 1, 2, 3
POLICY = {"scorpio": 0, "greedy": 1, "sjf": 2, "early_reject": 3}
FLAG_TTFT_GUARD, FLAG_TPOT_GUARD, FLAG_R_ONLY, FLAG_HAS_HORIZON, FLAG_PREFILL_PRIORITY = (
    1, 2, 4, 8, 16)
FLAG_GENERAL_ONLY = 32
SIM_CAPACITY = 8
MODE_AUTO, MODE_GENERAL = 0, 1

COST_FIELDS = ("alpha", "beta", "gamma", "delta", "epsilon", "phi", "theta", "alpha_p", "beta_p")

SIM_DTYPE = np.dtype({
    "names": ["trace", "policy", "flags", "max_batch_size", "slo_scale", "rate_factor",
              "horizon", "credit_exp", "credit_wide", "ws_offset", "out_offset", "log_slot"]
    + list(COST_FIELDS),
    "formats": ["<i4"] * 4 + ["<f8"] * 3 + ["<i4"] * 2 + ["<i8"] * 3 + ["<f8"] * 9,
    "offsets": [0, 4, 8, 12, 16, 24, 32, 40, 44, 48, 56, 64] + [72 + 8 * k for k in range(9)],
    "itemsize": 144,
})

RESULT_INT_FIELDS = ("n_steps", "n_plans", "n_idle_skips", "request_steps", "total", "completed",
                     "compliant", "rejected_ttft", "rejected_admission", "incomplete",
                     "ttft_violations", "tpot_violations")
RESULT_DTYPE = np.dtype({
    "names": ["status", "_pad"] + list(RESULT_INT_FIELDS)
    + ["sim_end", "horizon", "goodput", "adherence", "digest"],
    "formats": ["<i4", "<i4"] + ["<i8"] * 12 + ["<f8"] * 4 + ["<u8"],
    "offsets": [0, 4] + [8 + 8 * k for k in range(12)] + [104, 112, 120, 128, 136],
    "itemsize": 144,
})


REPORT_DTYPE = np.dtype({  # sl_report_row
    "names": ["ttft_p50", "ttft_p90", "ttft_p99", "tpot_ms_p50", "tpot_ms_p90", "tpot_ms_p99",
              "n_completed", "status_first"],
    "formats": ["<f8"] * 6 + ["<i8", ("<i8", (4,))],
    "offsets": [8 * k for k in range(8)],
    "itemsize": 88,
})


class NativeUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is missing; there is no CPU fallback."""


class SlTraces(C.Structure):
    _fields_ = [("n_traces", C.c_int32), ("_pad", C.c_int32)] + [
        (n, C.c_void_p) for n in ("begin", "arrival", "ttft_slo", "tpot_slo", "prompt_len",
                                  "true_out", "predicted", "id")]


class SlOutcomes(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("status", "compliant", "completion_step",
                                          "first_token_time", "completion_time", "ttft", "tpot")]


class SlLog(C.Structure):
    _fields_ = [("step_cap", C.c_int64), ("id_cap", C.c_int64)] + [
        (n, C.c_void_p) for n in ("now", "end", "prefill_s", "decode_s", "vbs", "min_slo",
                                  "n_admitted", "n_rejected", "n_batch", "adm_ids", "rej_ids",
                                  "batch_ids", "n_steps", "adm_rec")] + [
        ("skip_cap", C.c_int64)] + [
        (n, C.c_void_p) for n in ("skip_now", "skip_target", "skip_waiting", "n_skips")]


class SlCost(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("alpha", "beta", "gamma", "delta", "epsilon", "phi",
                                          "theta", "alpha_p", "beta_p")]


class SlPlanState(C.Structure):
    _fields_ = [("n_segments", C.c_int32), ("_pad", C.c_int32)] + [
        (n, C.c_void_p) for n in ("w_begin", "r_begin", "w_arrival", "w_ttft", "w_tpot",
                                  "w_prefill", "w_prompt", "w_pred", "w_id", "r_tpot",
                                  "r_cur_len", "r_id", "r_credit", "r_exclude", "now",
                                  "credit_exp")]


class SlPlanConfig(C.Structure):
    _fields_ = [("flags", C.c_int32), ("_pad", C.c_int32), ("cost", SlCost)]


class SlPlanOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("perm", "scratch", "adm_order", "w_status", "w_pos",
                                          "w_rec", "r_credit_out", "r_batch", "r_pos",
                                          "seg_counts", "seg_min_fixed", "seg_vbs",
                                          "seg_min_slo")]


PLAN_WAITING, PLAN_REJECTED_TTFT, PLAN_REJECTED_ADMISSION, PLAN_ADMITTED = 0, 1, 2, 3
PLAN_GUARD_ONLY = 64
PLAN_FCFS_WALK = 128
PLAN_EXACT_WALK = 256


class SlPredictor(C.Structure):
    _fields_ = [("mode", C.c_int32), ("num_buckets", C.c_int32), ("boundaries", C.c_void_p),
                ("error_prob", C.c_double), ("error_spread", C.c_int32), ("_pad", C.c_int32),
                ("rng_seed", C.c_uint64)]


PREDICT_ORACLE, PREDICT_NOISY_BUCKET = 0, 1


def build_native(verbose: bool = False) -> str:
    """Compile every CUDA source into lib/libscorpio_b200.so for sm_100a."""
    os.makedirs(LIB_DIR, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    cmd = ["nvcc", *NVCC_FLAGS, "-I" + INCLUDE, "-o", LIB_PATH, *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return LIB_PATH


_lib = None


def lib():
    """The loaded native library (ctypes.CDLL) with argtypes declared."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing; run __graft_entry__.build() (nvcc, sm_100a)")
    L = C.CDLL(LIB_PATH)
    L.sl_workspace_bytes.argtypes = [C.c_int64, C.c_int32]
    L.sl_workspace_bytes.restype = C.c_int64
    L.sl_credit_params.argtypes = [C.c_int64, C.c_void_p, C.c_double, C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32)]
    L.sl_credit_params.restype = C.c_int
    L.sl_run_batch.argtypes = [C.POINTER(SlTraces), C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                               C.c_int64, C.c_void_p, C.POINTER(SlOutcomes), C.POINTER(SlLog),
                               C.c_void_p]
    L.sl_run_batch.restype = C.c_int
    L.sl_run_batch_ex.argtypes = [C.POINTER(SlTraces), C.c_void_p, C.c_void_p, C.c_int32,
                                  C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(SlOutcomes),
                                  C.POINTER(SlLog), C.c_int32, C.c_void_p]
    L.sl_run_batch_ex.restype = C.c_int
    L.sl_run_batch_launches.restype = C.c_int
    L.sl_report_batch.argtypes = [C.POINTER(SlTraces), C.c_void_p, C.c_int32,
                                  C.POINTER(SlOutcomes), C.c_void_p, C.c_int32, C.c_void_p,
                                  C.c_void_p, C.c_void_p]
    L.sl_report_batch.restype = C.c_int
    L.sl_cumulative_batch.argtypes = [C.POINTER(SlTraces), C.c_void_p, C.c_int32,
                                      C.POINTER(SlOutcomes), C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
    L.sl_cumulative_batch.restype = C.c_int
    L.sl_selftest_div_small.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    L.sl_selftest_div_small.restype = C.c_int
    L.sl_selftest_certified_sum.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                            C.c_void_p]
    L.sl_selftest_certified_sum.restype = C.c_int
    L.sl_abi_layout.argtypes = [C.POINTER(C.c_int64), C.c_int32]
    L.sl_abi_layout.restype = C.c_int
    L.sl_device_info.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.sl_device_info.restype = C.c_int
    L.sl_predict_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(SlPredictor),
                                   C.c_void_p, C.c_void_p, C.c_void_p]
    L.sl_predict_batch.restype = C.c_int
    P = C.POINTER
    L.sl_ttft_sort_batch.argtypes = [P(SlPlanState), C.c_int64, P(SlPlanOut), C.c_void_p]
    L.sl_guard_admit_batch.argtypes = [P(SlPlanState), P(SlPlanConfig), P(SlPlanOut), C.c_void_p]
    L.sl_credit_select_batch.argtypes = [P(SlPlanState), P(SlPlanConfig), P(SlPlanOut), C.c_int32,
                                         C.c_void_p]
    L.sl_plan_step_batch.argtypes = [P(SlPlanState), P(SlPlanConfig), C.c_int64, P(SlPlanOut),
                                     C.c_void_p]
    L.sl_vbs_batch.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p]
    for fn in ("sl_ttft_sort_batch", "sl_guard_admit_batch", "sl_credit_select_batch",
               "sl_plan_step_batch", "sl_vbs_batch"):
        getattr(L, fn).restype = C.c_int
    for name, args in _OPTIONAL_SIGS.items():
        if hasattr(L, name):
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
    _check_layout(L)
    _lib = L
    return L


_OPTIONAL_SIGS: dict = {}


def _check_layout(L) -> None:
    out = (C.c_int64 * 8)()
    if L.sl_abi_layout(out, 8) != 0:
        raise NativeUnavailable("sl_abi_layout failed")
    want = (SIM_DTYPE.itemsize, RESULT_DTYPE.itemsize, C.sizeof(SlTraces), C.sizeof(SlOutcomes),
            C.sizeof(SlLog), 8 * len(COST_FIELDS), C.sizeof(SlPredictor), REPORT_DTYPE.itemsize)
    if tuple(out) != want:
        raise NativeUnavailable(f"ABI layout mismatch: library {tuple(out)} vs binding {want}")


def exported_symbols() -> list[str]:
    """Function names declared in include/scorpio_b200.h."""
    import re

    text = open(os.path.join(INCLUDE, "scorpio_b200.h")).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(sl_\w+)\(", text, flags=re.M)))


def require_cuda():
    """torch with a visible CUDA device, else NativeUnavailable (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the scheduling hot path runs only on GPU")
    lib()
    return torch


def credit_params(tpot_slo: np.ndarray, slo_scale: float) -> tuple[int, int]:
    """(E, wide) for one sim's fixed-point credits (sl_credit_params)."""
    arr = np.ascontiguousarray(tpot_slo, np.float64)
    e = C.c_int32()
    w = C.c_int32()
    rc = lib().sl_credit_params(len(arr), arr.ctypes.data, float(slo_scale), C.byref(e), C.byref(w))
    if rc != 0:
        raise ValueError("TPOT SLOs must be positive normal doubles within the credit range")
    return e.value, w.value
