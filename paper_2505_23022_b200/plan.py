"""Batched plan_step over many SchedulerStates on the device (config 2 path).

``PlanBatch`` packs S reference-shaped ``SchedulerState`` objects into the
``sl_plan_state`` SoA (one segment per state), runs the sort / guard+admit /
credit-select kernels (``sl_ttft_sort_batch``, ``sl_guard_admit_batch``,
``sl_credit_select_batch``) and returns per-state results that
``sched_scorpio`` applies back to the objects.  Credits cross the boundary as
exact integers credit * tpot_slo / 2^E.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _native as N
from .schedtypes import SchedulerState


@dataclass
class PlanResult:
    w_status: np.ndarray  # per waiting item, input order (SL_PLAN_*)
    w_pos: np.ndarray
    w_rec: np.ndarray | None  # [W, 5] admission record inputs
    adm_order: np.ndarray  # waiting indices (input order) in admission order
    r_credit: list[Fraction]  # new credits, per running entry
    r_batch: np.ndarray
    r_pos: np.ndarray
    kept: int
    admitted: int
    rejected: int
    batch: int
    vbs: float
    min_slo: float | None


def _dyadic_exp(x: Fraction) -> int:
    """Largest E with x * 2^-E integral (x dyadic)."""
    q = x.denominator
    if q & (q - 1):
        raise ValueError("credit is not a dyadic rational")
    if x.numerator == 0:
        return 1 << 20
    e = -(q.bit_length() - 1)
    n = x.numerator
    while n % 2 == 0:
        n //= 2
        e += 1
    return e


def segment_exponent(tpots: list[float], credits: list[tuple[Fraction, float]],
                     need_credits: bool = True) -> int:
    """Fixed-point exponent E for one state: every SLO and every credit*slo
    must be an integer multiple of 2^E.  Without a credit phase (ttft_guard,
    admit, the early-reject walk) the span limit does not apply."""
    if not need_credits:
        return 0
    E = 1 << 20
    for t in tpots:
        m, e = math.frexp(t)
        E = min(E, e - 53)
    for cr, t in credits:
        if cr:
            E = min(E, _dyadic_exp(Fraction(cr) * Fraction(t)))
    if tpots:
        span = max(math.frexp(t)[1] for t in tpots) - (E + 53)
        if 53 + span + 1 > 64:
            raise NotImplementedError(
                "SLO span needs 128-bit credits; use the sweep engine (sl_run_batch)")
    return 0 if E == 1 << 20 else E


class PlanBatch:
    """Device SoA for a batch of SchedulerStates (segments)."""

    def __init__(self, states: list[SchedulerState] | None = None, device=None,
                 arrays: dict | None = None, need_credits: bool = True):
        torch = N.require_cuda()
        self.torch = torch
        self.dev = torch.device(device if device is not None else "cuda")
        self.states = states
        host = arrays if arrays is not None else self._pack(states, need_credits)
        # negative prefills (alpha_p < 0 past -beta_p/alpha_p) disable the walk's
        # monotone shortcuts in the kernels
        self.exact_walk = bool(len(host["w_prefill"]) and (host["w_prefill"] < 0).any())
        S = len(host["now"])
        self.w_begin = host["w_begin"]
        self.r_begin = host["r_begin"]
        self.E = host["credit_exp"]
        W, R = int(self.w_begin[-1]), int(self.r_begin[-1])
        self.max_w = int(np.diff(self.w_begin).max()) if S else 0
        self.d = {}
        for k in ("w_begin", "r_begin", "w_arrival", "w_ttft", "w_tpot", "w_prefill", "w_prompt",
                  "w_pred", "w_id", "r_tpot", "r_cur_len", "r_id", "r_credit", "now",
                  "credit_exp"):
            v = np.ascontiguousarray(host[k])
            if v.dtype == np.uint64:
                v = v.view(np.int64)
            self.d[k] = (torch.from_numpy(v).to(self.dev) if len(v) else
                         torch.zeros(1, dtype=torch.float64, device=self.dev))
        self.d["r_exclude"] = torch.zeros(max(R, 1), dtype=torch.uint8, device=self.dev)
        self.W, self.R, self.S = W, R, S
        self.st = N.SlPlanState(S, 0, *[self.d[k].data_ptr() for k in (
            "w_begin", "r_begin", "w_arrival", "w_ttft", "w_tpot", "w_prefill", "w_prompt",
            "w_pred", "w_id", "r_tpot", "r_cur_len", "r_id", "r_credit", "r_exclude", "now",
            "credit_exp")])
        i32 = dict(dtype=torch.int32, device=self.dev)
        w1, r1 = max(W, 1), max(R, 1)
        self.o = {
            "perm": torch.zeros(w1, **i32), "scratch": torch.zeros(w1, **i32),
            "adm_order": torch.zeros(w1, **i32), "w_status": torch.full((w1,), -1, **i32),
            "w_pos": torch.zeros(w1, **i32),
            "w_rec": torch.zeros(w1 * 5, dtype=torch.float64, device=self.dev),
            "r_credit_out": torch.zeros(r1, dtype=torch.int64, device=self.dev),
            "r_batch": torch.zeros(r1, dtype=torch.uint8, device=self.dev),
            "r_pos": torch.zeros(r1, **i32), "seg_counts": torch.zeros(4 * max(S, 1), **i32),
            "seg_min_fixed": torch.zeros(max(S, 1), dtype=torch.int64, device=self.dev),
            "seg_vbs": torch.zeros(max(S, 1), dtype=torch.float64, device=self.dev),
            "seg_min_slo": torch.zeros(max(S, 1), dtype=torch.float64, device=self.dev),
        }
        self.out = N.SlPlanOut(*[self.o[k].data_ptr() for k in (
            "perm", "scratch", "adm_order", "w_status", "w_pos", "w_rec", "r_credit_out",
            "r_batch", "r_pos", "seg_counts", "seg_min_fixed", "seg_vbs", "seg_min_slo")])

    @staticmethod
    def _pack(states: list[SchedulerState], need_credits: bool = True) -> dict[str, np.ndarray]:
        S = len(states)
        w_begin = np.zeros(S + 1, np.int64)
        r_begin = np.zeros(S + 1, np.int64)
        np.cumsum([len(s.waiting) for s in states], out=w_begin[1:])
        np.cumsum([len(s.running) for s in states], out=r_begin[1:])
        items = [w for s in states for w in s.waiting]
        ents = [e for s in states for e in s.running]
        E = np.array([segment_exponent(
            [w.request.tpot_slo for w in s.waiting] + [e.request.tpot_slo for e in s.running],
            [(e.credit, e.request.tpot_slo) for e in s.running], need_credits)
            for s in states], np.int32)
        credit = np.zeros(len(ents), np.uint64)
        k = 0
        for si, s in enumerate(states if need_credits else []):
            scale = Fraction(2) ** (-int(E[si]))
            for e in s.running:
                n = Fraction(e.credit) * Fraction(e.request.tpot_slo) * scale
                if n.denominator != 1 or n < 0 or n >= 1 << 63:
                    raise ValueError("credit outside the exact fixed-point domain")
                credit[k] = int(n)
                k += 1
        return {
            "w_begin": w_begin, "r_begin": r_begin,
            "w_arrival": np.array([w.request.arrival_time for w in items], np.float64),
            "w_ttft": np.array([w.request.ttft_slo for w in items], np.float64),
            "w_tpot": np.array([w.request.tpot_slo for w in items], np.float64),
            "w_prefill": np.array([w.prefill_s for w in items], np.float64),
            "w_prompt": np.array([w.request.prompt_len for w in items], np.int32),
            "w_pred": np.array([w.predicted_len for w in items], np.int32),
            "w_id": np.array([w.request.id for w in items], np.int64),
            "r_tpot": np.array([e.request.tpot_slo for e in ents], np.float64),
            "r_cur_len": np.array([e.current_len for e in ents], np.int32),
            "r_id": np.array([e.request.id for e in ents], np.int64),
            "r_credit": credit, "now": np.array([s.now for s in states], np.float64),
            "credit_exp": E,
        }

    def set_exclude(self, per_state: list[set[int]]) -> None:
        """Entries (by id()) excluded from the credit phase (select_batch `exclude`)."""
        ex = np.zeros(max(self.R, 1), np.uint8)
        k = 0
        for s, excl in zip(self.states, per_state):
            for e in s.running:
                ex[k] = 1 if excl and id(e) in excl else 0
                k += 1
        self.d["r_exclude"].copy_(self.torch.from_numpy(ex))

    def _cfg(self, flags: int, itl, prefill) -> N.SlPlanConfig:
        a, b, g, d, e = itl
        phi, th, ap, bp = prefill
        if self.exact_walk:
            flags |= N.PLAN_EXACT_WALK
        return N.SlPlanConfig(flags, 0, N.SlCost(a, b, g, d, e, phi, th, ap, bp))

    def _stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def sort(self) -> None:
        rc = N.lib().sl_ttft_sort_batch(C.byref(self.st), self.max_w, C.byref(self.out),
                                       self._stream())
        if rc:
            raise RuntimeError(f"sl_ttft_sort_batch failed ({rc})")

    def guard_admit(self, flags: int, itl, prefill) -> None:
        cfg = self._cfg(flags, itl, prefill)
        rc = N.lib().sl_guard_admit_batch(C.byref(self.st), C.byref(cfg), C.byref(self.out),
                                         self._stream())
        if rc:
            raise RuntimeError(f"sl_guard_admit_batch failed ({rc})")

    def select(self, flags: int, use_seg_min: bool) -> None:
        cfg = self._cfg(flags, (0.0, 0.0, 0.0, 0.0, 1.0), (1.0, 0.0, 0.0, 0.0))
        rc = N.lib().sl_credit_select_batch(C.byref(self.st), C.byref(cfg), C.byref(self.out),
                                           int(use_seg_min), self._stream())
        if rc:
            raise RuntimeError(f"sl_credit_select_batch failed ({rc})")

    def plan(self, flags: int, itl, prefill) -> None:
        cfg = self._cfg(flags, itl, prefill)
        rc = N.lib().sl_plan_step_batch(C.byref(self.st), C.byref(cfg), self.max_w,
                                       C.byref(self.out), self._stream())
        if rc:
            raise RuntimeError(f"sl_plan_step_batch failed ({rc})")

    def results(self) -> list[PlanResult]:
        h = {k: v.cpu().numpy() for k, v in self.o.items()}
        res = []
        for si in range(self.S):
            wb, we = int(self.w_begin[si]), int(self.w_begin[si + 1])
            rb, re = int(self.r_begin[si]), int(self.r_begin[si + 1])
            kept, nadm, nrej, nb = (int(x) for x in h["seg_counts"][4 * si: 4 * si + 4])
            E = int(self.E[si])
            inv_scale = Fraction(2) ** E
            nums = h["r_credit_out"][rb:re].view(np.uint64)
            tp = self.d["r_tpot"][rb:re].cpu().numpy() if self.states is None else \
                [e.request.tpot_slo for e in self.states[si].running]
            credits = [Fraction(int(n)) * inv_scale / Fraction(float(t)) for n, t in zip(nums, tp)]
            ms = float(h["seg_min_slo"][si])
            res.append(PlanResult(
                w_status=h["w_status"][wb:we].copy(), w_pos=h["w_pos"][wb:we].copy(),
                w_rec=h["w_rec"][5 * wb: 5 * we].reshape(-1, 5).copy(),
                adm_order=h["adm_order"][wb: wb + nadm] - wb,
                r_credit=credits, r_batch=h["r_batch"][rb:re].copy(), r_pos=h["r_pos"][rb:re].copy(),
                kept=kept, admitted=nadm, rejected=nrej, batch=nb,
                vbs=float(h["seg_vbs"][si]), min_slo=None if math.isnan(ms) else ms))
        return res


def vbs_batch(tpot_lists: list[list[float]], min_slos: list[float], device=None) -> list[float]:
    """vbs() for many running sets in one launch (sl_vbs_batch)."""
    torch = N.require_cuda()
    dev = torch.device(device if device is not None else "cuda")
    begin = np.zeros(len(tpot_lists) + 1, np.int64)
    np.cumsum([len(t) for t in tpot_lists], out=begin[1:])
    flat = np.array([x for t in tpot_lists for x in t] or [0.0], np.float64)
    b = torch.from_numpy(begin).to(dev)
    f = torch.from_numpy(flat).to(dev)
    m = torch.from_numpy(np.array(min_slos, np.float64)).to(dev)
    out = torch.zeros(max(len(tpot_lists), 1), dtype=torch.float64, device=dev)
    rc = N.lib().sl_vbs_batch(len(tpot_lists), b.data_ptr(), f.data_ptr(), m.data_ptr(),
                              out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    if rc:
        raise RuntimeError(f"sl_vbs_batch failed ({rc})")
    return [float(x) for x in out.cpu().numpy()[: len(tpot_lists)]]
