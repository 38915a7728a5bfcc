"""Scorpio policy API on the device (slosim.sched_scorpio drop-in,
pkg/src/slosim/sched_scorpio.py:37-346).

Same names, signatures, error behaviour and state mutation as the reference;
each decision function marshals the state(s) to the SoA device layout and runs
the sm_100a plan kernels (plan.py): ``ttft_guard`` = LDF sort + TTFT walk,
``admit`` / ``plan_step`` = guard + admission scan + credit phase,
``select_batch`` = credit phase, ``vbs`` = Neumaier TRP sum.  ``plan_step_batch``
is the batched form over many independent states (one launch per kernel).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native as N
from ._family import family
from .core import Request, Status
from .costmodel import ItlParams, PrefillParams, itl_coeffs, prefill_coeffs, prefill_time
from .plan import PlanBatch, vbs_batch
from .predictor import LengthPredictor
from .schedtypes import AdmissionRecord, RunningEntry, SchedulerState, StepPlan, WaitingItem

SCORPIO = "scorpio"
R_PRIME = "r_prime"
R_ONLY = "r_only"

_REJECT_NAME = {N.PLAN_REJECTED_TTFT: "REJECTED_TTFT",
                N.PLAN_REJECTED_ADMISSION: "REJECTED_ADMISSION"}


@dataclass(frozen=True)
class ScorpioConfig:
    """Guard toggles and the admission threshold form (sched_scorpio.py:43-60)."""

    ttft_guard: bool = True
    tpot_guard: bool = True
    admission_min: str = R_PRIME

    def __post_init__(self) -> None:
        if self.admission_min not in (R_PRIME, R_ONLY):
            raise ValueError(f"unknown admission_min {self.admission_min!r}")

    def flags(self) -> int:
        return scorpio_flags(self)


def scorpio_flags(config) -> int:
    """Kernel flag word of any ScorpioConfig-shaped object (sched_scorpio.py:43-60)."""
    if config.admission_min not in (R_PRIME, R_ONLY):
        raise ValueError(f"unknown admission_min {config.admission_min!r}")
    f = N.FLAG_TTFT_GUARD if config.ttft_guard else 0
    f |= N.FLAG_TPOT_GUARD if config.tpot_guard else 0
    f |= N.FLAG_R_ONLY if config.admission_min == R_ONLY else 0
    return f


def trp(tpot_slo: float, running_min_slo: float) -> float:
    """Credit-earning rate relative to the strictest running SLO (:63-67)."""
    if tpot_slo <= 0 or running_min_slo <= 0:
        raise ValueError("TPOT SLOs must be positive")
    return running_min_slo / tpot_slo


def vbs(running: list[RunningEntry], min_slo: float) -> float:
    """Virtual batch size: Neumaier sum of TRPs in running order (:70-74), on device."""
    if not running:
        return 0.0
    for e in running:
        trp(e.request.tpot_slo, min_slo)  # reference validation
    return vbs_batch([[e.request.tpot_slo for e in running]], [min_slo])[0]


def _apply_plan(state: SchedulerState, r, plan: StepPlan | None, records: bool) -> None:
    """Apply one segment's device decisions to the caller's objects (this
    package's or the reference's classes, whichever ``state`` belongs to)."""
    fam = family(state)
    items = state.waiting
    running_before = list(state.running)
    # rejected, in plan order (TTFT walk first, then the admission scan)
    rej = sorted((int(r.w_pos[i]), i) for i in range(len(items))
                 if int(r.w_status[i]) in _REJECT_NAME)
    admitted = []
    for k in r.adm_order:
        it = items[int(k)]
        e = fam.RunningEntry(request=it.request, predicted_len=it.predicted_len,
                             prefill_s=it.prefill_s)
        admitted.append((int(k), e))
    keep = sorted((int(r.w_pos[i]), i) for i in range(len(items))
                  if int(r.w_status[i]) == N.PLAN_WAITING)
    if plan is not None:
        plan.rejected.extend((items[i], getattr(fam.Status, _REJECT_NAME[int(r.w_status[i])]))
                             for _, i in rej)
        if records:
            snap = [(e.request.id, e.request.tpot_slo, e.current_len) for e in running_before]
            for k, e in admitted:
                v = r.w_rec[k]
                plan.admissions.append(fam.AdmissionRecord(
                    now=state.now, candidate_id=e.request.id,
                    candidate_tpot_slo=e.request.tpot_slo, candidate_len=e.request.prompt_len,
                    predicted_len=e.predicted_len, running=tuple(snap), vbs=float(v[0]),
                    l_avg=float(v[1]), min_slo=float(v[2]), estimate=float(v[3]),
                    threshold=float(v[4])))
                snap.append((e.request.id, e.request.tpot_slo, e.current_len))
        plan.admitted.extend(e for _, e in admitted)
    state.running.extend(e for _, e in admitted)
    state.waiting = [items[i] for _, i in keep]


def _apply_select(state_running: list[RunningEntry], r) -> list[RunningEntry]:
    for e, c in zip(state_running, r.r_credit):
        e.credit = c
    order = sorted((int(r.r_pos[j]), j) for j in range(len(state_running)) if r.r_batch[j])
    return [state_running[j] for _, j in order]


def admit(state: SchedulerState, candidate: Request, predicted_len: int, cost: ItlParams,
          admission_min: str = R_PRIME, prefill_s: float = 0.0) -> bool:
    """Admit ``candidate`` if the projected TPOT allows (:127-158)."""
    if predicted_len < 1:
        raise ValueError("predicted_len must be >= 1")
    fam = family(state)
    probe = SchedulerState(waiting=[WaitingItem(candidate, predicted_len, prefill_s)],
                           running=state.running, now=state.now)
    pb = PlanBatch([probe], need_credits=False)
    flags = N.FLAG_TPOT_GUARD | (N.FLAG_R_ONLY if admission_min == R_ONLY else 0)
    pb.guard_admit(flags, itl_coeffs(cost), (1.0, 0.0, 0.0, 0.0))
    r = pb.results()[0]
    ok = int(r.w_status[0]) == N.PLAN_ADMITTED
    if ok:
        state.running.append(fam.RunningEntry(request=candidate, predicted_len=predicted_len,
                                              prefill_s=prefill_s))
    return ok


def select_batch(state: SchedulerState, exclude: set[int] | None = None) -> list[RunningEntry]:
    """Credit phase: earn min/slo, batch at credit >= 1, debit 1 (:161-180)."""
    if not state.running:
        return []
    pb = PlanBatch([state])
    pb.set_exclude([exclude or set()])
    pb.select(N.FLAG_TPOT_GUARD, use_seg_min=False)
    return _apply_select(state.running, pb.results()[0])


def ttft_guard(state: SchedulerState, cost: PrefillParams) -> tuple[list[WaitingItem],
                                                                    list[WaitingItem]]:
    """LDF order + drop TTFT-unattainable requests (:183-207)."""
    pb = PlanBatch([state], need_credits=False)
    if state.waiting:
        pb.sort()
        pb.guard_admit(N.FLAG_TTFT_GUARD | N.PLAN_GUARD_ONLY, (0.0, 0.0, 0.0, 0.0, 1.0),
                       prefill_coeffs(cost))
    r = pb.results()[0]
    items = state.waiting
    rejected = [items[i] for _, i in sorted((int(r.w_pos[i]), i) for i in range(len(items))
                                            if int(r.w_status[i]) == N.PLAN_REJECTED_TTFT)]
    kept = [items[i] for _, i in sorted((int(r.w_pos[i]), i) for i in range(len(items))
                                        if int(r.w_status[i]) == N.PLAN_WAITING)]
    state.waiting = kept
    return kept, rejected


def plan_step_batch(states: list[SchedulerState], itl_params: ItlParams,
                    prefill_params: PrefillParams, config: ScorpioConfig = ScorpioConfig(),
                    records: bool = True) -> list[StepPlan]:
    """plan_step for many independent states: sort + guard/admit + select kernels,
    one launch each, over all states."""
    flags = scorpio_flags(config)
    pb = PlanBatch(states, need_credits=bool(config.tpot_guard))
    pb.plan(flags, itl_coeffs(itl_params), prefill_coeffs(prefill_params))
    plans = []
    for s, r in zip(states, pb.results()):
        plan = family(s).StepPlan()
        running_before = list(s.running)
        _apply_plan(s, r, plan, records and config.tpot_guard)
        # fresh entries are not in the kernel's running arrays, so they never batch
        plan.decode_batch = (_apply_select(running_before, r) if config.tpot_guard
                             else list(running_before))
        if s.running:
            plan.min_slo = r.min_slo
            plan.vbs = r.vbs
        plans.append(plan)
    return plans


def plan_step(state: SchedulerState, predictor: LengthPredictor, itl_params: ItlParams,
              prefill_params: PrefillParams, config: ScorpioConfig = ScorpioConfig()) -> StepPlan:
    """One scheduling iteration: TTFT guard, admission scan, credit phase (:210-316)."""
    return plan_step_batch([state], itl_params, prefill_params, config)[0]


class ScorpioPolicy:
    """Policy adapter (:319-346)."""

    def __init__(self, predictor: LengthPredictor, itl_params: ItlParams,
                 prefill_params: PrefillParams, config: ScorpioConfig = ScorpioConfig()) -> None:
        self.predictor = predictor
        self.itl_params = itl_params
        self.prefill_params = prefill_params
        self.config = config

    def on_arrival(self, state: SchedulerState, req: Request) -> None:
        state.waiting.append(WaitingItem(request=req, predicted_len=self.predictor.predict(req),
                                         prefill_s=prefill_time(self.prefill_params,
                                                                req.prompt_len)))

    def plan(self, state: SchedulerState) -> StepPlan:
        return plan_step(state, self.predictor, self.itl_params, self.prefill_params, self.config)
