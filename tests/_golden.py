"""Loader for the reference-generated fixtures in tests/golden (see make_golden.py)."""

from __future__ import annotations

import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
OUTCOME_FIELDS = ("status", "compliant", "completion_step", "first_token_time",
                  "completion_time", "ttft", "tpot")
TRACE_FIELDS = ("arrival", "ttft_slo", "tpot_slo", "prompt_len", "true_out", "id", "category",
                "predicted")


def load_cases() -> list[dict]:
    meta = json.load(open(os.path.join(HERE, "sims.json")))
    blobs = np.load(os.path.join(HERE, "sims.npz"))
    cases = []
    for ci, m in enumerate(meta):
        c = dict(m)
        p = f"c{ci}_"
        c["trace"] = {k: blobs[p + k] for k in TRACE_FIELDS}
        c["outcomes"] = {k: blobs[p + k] for k in OUTCOME_FIELDS}
        if m["keep_log"]:
            c["log"] = {k: blobs[p + "log_" + k] for k in ("now", "end", "prefill_s", "decode_s",
                                                            "vbs", "min_slo", "counts", "ids")}
        c["digest"] = int(m["digest"])
        cases.append(c)
    return cases


def oracle_params(case):
    from oracle import oracle as orc

    return orc.make_params(policy=case["policy"], ttft_guard=case["ttft_guard"],
                           tpot_guard=case["tpot_guard"], admission_min=case["admission_min"],
                           horizon=case["horizon"], max_batch_size=case["max_batch_size"],
                           prefill_priority=case["prefill_priority"], itl=case["itl"],
                           prefill=case["prefill"])


def same_float(a, b) -> bool:
    """Bitwise equality of fp64 arrays, NaN == NaN."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return a.shape == b.shape and bool(np.all(a.view(np.uint64) == b.view(np.uint64)))
