"""Seeded scheduler-state snapshots for config 2: S independent
SchedulerStates ("segments") with W waiting and R running requests each.

Tiers as config 1 (TTFT/TPOT (0.5 s, 30 ms), (2.0 s, 50 ms), (7.5 s, 100 ms)),
arrivals U[now - 0.4, now], prompt U[20, 600], output U[5, 400], tokens
U[1, output), credits reachable fixed-point values (k * MIN mod S, i.e. the
credit after k credit phases).  Arrays only (numpy), so the same snapshot can be
materialised as objects of either the reference or this package.
"""

from __future__ import annotations

import math

import numpy as np

TIERS = ((0.5, 0.030), (2.0, 0.050), (7.5, 0.100))
ACC_PREFILL = (0.004, 128.0, 2e-5, 1.5e-3)


def _prefill(phi, theta, ap, bp, n):
    return phi if n <= theta else ap * n + bp


def config2_arrays(n_segments: int, w: int, r: int, seed: int, now: float = 10.0,
                   prefill=ACC_PREFILL, tie_grid: float | None = None) -> dict[str, np.ndarray]:
    """tie_grid: round waiting arrivals to multiples of this (a power of two) so
    that deadlines tie exactly, between equal arrivals (then the id decides)
    and between different ones (a1 + t1 == a2 + t2)."""
    rng = np.random.default_rng(seed)
    S = n_segments
    # w / r: per-segment counts (ragged batches) or one count for every segment
    ws = np.full(S, w, np.int64) if np.isscalar(w) else np.asarray(w, np.int64)
    rs = np.full(S, r, np.int64) if np.isscalar(r) else np.asarray(r, np.int64)
    assert len(ws) == S and len(rs) == S
    W, R = int(ws.sum()), int(rs.sum())
    tier_w = rng.integers(0, 3, W)
    tier_r = rng.integers(0, 3, R)
    out_w = rng.integers(5, 401, W)
    out_r = rng.integers(5, 401, R)
    a = {
        "w_begin": np.concatenate([[0], np.cumsum(ws)]).astype(np.int64),
        "r_begin": np.concatenate([[0], np.cumsum(rs)]).astype(np.int64),
        "w_id": np.arange(W, dtype=np.int64),
        "w_arrival": now - rng.uniform(0.0, 0.4, W),
        "w_ttft": np.array([TIERS[t][0] for t in tier_w]),
        "w_tpot": np.array([TIERS[t][1] for t in tier_w]),
        "w_prompt": rng.integers(20, 601, W).astype(np.int32),
        "w_pred": out_w.astype(np.int32),
        "r_id": np.arange(W, W + R, dtype=np.int64),
        "r_tpot": np.array([TIERS[t][1] for t in tier_r]),
        "r_prompt": rng.integers(20, 601, R).astype(np.int32),
        "r_out": out_r.astype(np.int32),
        "r_tokens": np.array([int(rng.integers(1, o)) for o in out_r], np.int32),
        "r_k": rng.integers(0, 1000, R),
        "now": np.full(S, now),
    }
    if tie_grid:
        a["w_arrival"] = np.round(a["w_arrival"] / tie_grid) * tie_grid
        # TTFT SLOs off their tier by whole grid steps: equal deadlines then also
        # come from different arrivals (exact: everything is on the 2^-k grid)
        a["w_ttft"] = a["w_ttft"] + tie_grid * (np.arange(W) % 4)
        # ids in descending arrival-independent order, so the id tie-break is
        # visible (equal (deadline, arrival) pairs order by id, not position)
        a["w_id"] = a["w_id"][::-1].copy()
    a["w_prefill"] = np.array([_prefill(*prefill, int(n)) for n in a["w_prompt"]])
    # credit numerators: after k phases at the strictest tier, (k * MIN) mod S_e
    E = min(math.frexp(t)[1] for _, t in TIERS) - 53
    smin = int(np.ldexp(TIERS[0][1], -E))
    a["r_credit_num"] = np.array(
        [(int(k) * smin) % int(np.ldexp(t, -E)) for k, t in zip(a["r_k"], a["r_tpot"])],
        dtype=object)
    a["credit_exp"] = np.full(S, E, np.int32)
    return a


def config2_plan_arrays_fast(n_segments: int, w: int, r: int, seed: int, now: float = 10.0,
                            prefill=ACC_PREFILL) -> dict[str, np.ndarray]:
    """Vectorised sl_plan_state SoA with config2_arrays' distributions (a different
    random stream) for large benchmark batches; bench.py times these, and 256
    segments of the 262,144-segment batch are pinned to the reference's
    plan_step (tests/golden/make_plan_golden.py, states_from_plan_arrays)."""
    rng = np.random.default_rng(seed)
    S, W, R = n_segments, n_segments * w, n_segments * r
    ttft = np.array([t[0] for t in TIERS])
    tpot = np.array([t[1] for t in TIERS])
    tw = rng.integers(0, 3, W)
    tr = rng.integers(0, 3, R)
    prompt_w = rng.integers(20, 601, W)
    phi, theta, ap, bp = prefill
    out_r = rng.integers(5, 401, R)
    tokens = 1 + np.floor(rng.random(R) * (out_r - 1)).astype(np.int64)
    E = min(math.frexp(t)[1] for _, t in TIERS) - 53
    smin = np.uint64(int(np.ldexp(TIERS[0][1], -E)))
    s_e = np.ldexp(tpot[tr], -E).astype(np.uint64)
    k = rng.integers(0, 1000, R).astype(np.uint64)
    return {
        "w_begin": np.arange(S + 1, dtype=np.int64) * w,
        "r_begin": np.arange(S + 1, dtype=np.int64) * r,
        "w_arrival": now - rng.uniform(0.0, 0.4, W), "w_ttft": ttft[tw], "w_tpot": tpot[tw],
        "w_prefill": np.where(prompt_w <= theta, phi, ap * prompt_w + bp),
        "w_prompt": prompt_w.astype(np.int32), "w_pred": rng.integers(5, 401, W).astype(np.int32),
        "w_id": np.arange(W, dtype=np.int64), "r_tpot": tpot[tr],
        "r_cur_len": (rng.integers(20, 601, R) + tokens).astype(np.int32),
        "r_id": np.arange(W, W + R, dtype=np.int64), "r_credit": (k * smin) % s_e,
        "now": np.full(S, now), "credit_exp": np.full(S, E, np.int32),
    }


def plan_arrays(a: dict) -> dict[str, np.ndarray]:
    """The sl_plan_state SoA (PlanBatch(arrays=...)) of a snapshot, no objects."""
    out = {k: a[k] for k in ("w_begin", "r_begin", "w_arrival", "w_ttft", "w_tpot", "w_prefill",
                             "w_prompt", "w_pred", "w_id", "r_tpot", "r_id", "now", "credit_exp")}
    out["r_cur_len"] = (a["r_prompt"] + a["r_tokens"]).astype(np.int32)
    out["r_credit"] = np.array([int(x) for x in a["r_credit_num"]], np.uint64)
    return out


def states_from_arrays(a: dict, types) -> list:
    """Materialise SchedulerState objects with `types` = module-like object with
    Request, WaitingItem, RunningEntry, SchedulerState (reference or drop-in)."""
    from fractions import Fraction

    S = len(a["now"])
    out = []
    E = int(a["credit_exp"][0])
    for s in range(S):
        st = types.SchedulerState(now=float(a["now"][s]))
        for i in range(int(a["w_begin"][s]), int(a["w_begin"][s + 1])):
            req = types.Request(id=int(a["w_id"][i]), arrival_time=float(a["w_arrival"][i]),
                                prompt_len=int(a["w_prompt"][i]),
                                true_output_len=int(a["w_pred"][i]),
                                ttft_slo=float(a["w_ttft"][i]), tpot_slo=float(a["w_tpot"][i]))
            st.waiting.append(types.WaitingItem(request=req, predicted_len=int(a["w_pred"][i]),
                                                prefill_s=float(a["w_prefill"][i])))
        for j in range(int(a["r_begin"][s]), int(a["r_begin"][s + 1])):
            req = types.Request(id=int(a["r_id"][j]), arrival_time=0.0,
                                prompt_len=int(a["r_prompt"][j]),
                                true_output_len=int(a["r_out"][j]), ttft_slo=1.0,
                                tpot_slo=float(a["r_tpot"][j]))
            e = types.RunningEntry(request=req, predicted_len=int(a["r_out"][j]), prefill_s=0.0)
            e.tokens_generated = int(a["r_tokens"][j])
            e.credit = Fraction(int(a["r_credit_num"][j])) * Fraction(2) ** E / \
                Fraction(float(a["r_tpot"][j]))
            st.running.append(e)
        out.append(st)
    return out


def states_from_plan_arrays(a: dict, types, segments) -> list:
    """SchedulerState objects for selected segments of an sl_plan_state SoA
    (e.g. config2_plan_arrays_fast): a running entry's current length is split
    as prompt = cur_len - 1 plus one generated token (plan_step reads only the
    sum), its credit restored exactly from the fixed-point numerator."""
    from fractions import Fraction

    E = int(a["credit_exp"][0])
    out = []
    for s in segments:
        st = types.SchedulerState(now=float(a["now"][s]))
        for i in range(int(a["w_begin"][s]), int(a["w_begin"][s + 1])):
            req = types.Request(id=int(a["w_id"][i]), arrival_time=float(a["w_arrival"][i]),
                                prompt_len=int(a["w_prompt"][i]),
                                true_output_len=int(a["w_pred"][i]),
                                ttft_slo=float(a["w_ttft"][i]), tpot_slo=float(a["w_tpot"][i]))
            st.waiting.append(types.WaitingItem(request=req, predicted_len=int(a["w_pred"][i]),
                                                prefill_s=float(a["w_prefill"][i])))
        for j in range(int(a["r_begin"][s]), int(a["r_begin"][s + 1])):
            cur = int(a["r_cur_len"][j])
            req = types.Request(id=int(a["r_id"][j]), arrival_time=0.0, prompt_len=cur - 1,
                                true_output_len=cur + 1000, ttft_slo=1.0,
                                tpot_slo=float(a["r_tpot"][j]))
            e = types.RunningEntry(request=req, predicted_len=400, prefill_s=0.0)
            e.tokens_generated = 1
            e.credit = Fraction(int(a["r_credit"][j])) * Fraction(2) ** E / \
                Fraction(float(a["r_tpot"][j]))
            st.running.append(e)
        out.append(st)
    return out
