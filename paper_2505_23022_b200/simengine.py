"""Discrete-event engine API on the device (slosim.simengine drop-in,
pkg/src/slosim/simengine.py:42-303).

``run(trace, config)`` executes the whole simulation in the sm_100a sweep
engine (``sl_run_batch``: one warp-resident simulation) with the decision log
enabled, then rebuilds the reference's return values -- per-request
``RequestOutcome`` objects and an ``EventLog`` whose ``StepRecord``s,
``AdmissionRecord``s, ``token_emits`` and ``idle_skips`` come from the device
log.  ``run_many`` runs many (trace, config) cells in one launch.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _native as N
from ._family import family
from .batch import BatchEngine, Cell, CellConfig, TraceArrays
from .core import Request, RequestOutcome
from .costmodel import ItlParams, PrefillParams, itl_coeffs, prefill_coeffs
from .predictor import ORACLE, LengthPredictor, predict_many
from .sched_baselines import (EARLY_REJECT, GREEDY, SJF, BaselineConfig, EarlyRejectPolicy,
                              GreedyPolicy, SjfPolicy)
from .sched_scorpio import SCORPIO, ScorpioConfig, ScorpioPolicy
from .schedtypes import AdmissionRecord, Policy


class EngineError(RuntimeError):
    """The policy handed back a plan the engine cannot execute."""


@dataclass(frozen=True)
class SimConfig:
    policy: str
    itl_params: ItlParams
    prefill_params: PrefillParams
    predictor: LengthPredictor
    scorpio: ScorpioConfig = ScorpioConfig()
    baseline: BaselineConfig = BaselineConfig()
    horizon: float | None = None
    log_decisions: bool = False

    def __post_init__(self) -> None:
        if self.horizon is not None and self.horizon <= 0:
            raise ValueError("horizon must be positive when finite")

    def cell_config(self) -> CellConfig:
        return cell_config_of(self)


def cell_config_of(config) -> CellConfig:
    """Flatten any SimConfig-shaped object (this package's or the reference's,
    simengine.py:46-61) into the device cell config; fields only."""
    if config.policy not in (SCORPIO, GREEDY, SJF, EARLY_REJECT):
        raise ValueError(f"unknown policy {config.policy!r}")
    sc, bl = config.scorpio, config.baseline
    return CellConfig(policy=config.policy, itl=itl_coeffs(config.itl_params),
                      prefill=prefill_coeffs(config.prefill_params),
                      ttft_guard=bool(sc.ttft_guard), tpot_guard=bool(sc.tpot_guard),
                      admission_min=sc.admission_min, max_batch_size=int(bl.max_batch_size),
                      prefill_priority=bool(bl.prefill_priority), horizon=config.horizon)


def build_policy(config: SimConfig) -> Policy:
    """Policy objects for step-by-step use (simengine.py:64-77)."""
    if config.policy == SCORPIO:
        return ScorpioPolicy(config.predictor, config.itl_params, config.prefill_params,
                             config.scorpio)
    base = BaselineConfig(policy=config.policy, max_batch_size=config.baseline.max_batch_size,
                          prefill_priority=config.baseline.prefill_priority)
    cls = {GREEDY: GreedyPolicy, SJF: SjfPolicy, EARLY_REJECT: EarlyRejectPolicy}[config.policy]
    return cls(config.predictor, config.prefill_params, base)


@dataclass
class StepRecord:
    step: int
    now_s: float
    end_s: float
    admitted: list[int]
    rejected: list[tuple[int, str]]
    batch: list[int]
    vbs: float
    min_slo_s: float | None
    prefill_s: float
    decode_s: float
    admissions: list[AdmissionRecord] = field(default_factory=list)


@dataclass
class EventLog:
    steps: list[StepRecord] = field(default_factory=list)
    token_emits: dict[int, list[float]] = field(default_factory=dict)
    idle_skips: list[tuple[float, float, int]] = field(default_factory=list)
    policy_wall_s: float = 0.0
    engine_wall_s: float = 0.0
    sim_end_s: float = 0.0

    def to_jsonl(self, path: str | Path) -> None:
        """Per-step decision log (simengine.py:106-137 format)."""
        with open(path, "w", encoding="utf-8") as f:
            for rec in self.steps:
                row = {"step": rec.step, "now_s": rec.now_s, "admitted": rec.admitted,
                       "rejected": [[rid, reason] for rid, reason in rec.rejected],
                       "batch": rec.batch, "vbs": rec.vbs,
                       "min_slo_ms": None if rec.min_slo_s is None else rec.min_slo_s * 1000.0}
                if rec.admissions:
                    row["admissions"] = [{
                        "id": a.candidate_id, "tpot_slo_ms": a.candidate_tpot_slo * 1000.0,
                        "candidate_len": a.candidate_len, "predicted_len": a.predicted_len,
                        "running": [list(t) for t in a.running], "vbs": a.vbs,
                        "l_avg": a.l_avg, "min_slo_ms": a.min_slo * 1000.0,
                        "estimate_ms": a.estimate * 1000.0, "threshold_ms": a.threshold * 1000.0,
                    } for a in rec.admissions]
                f.write(json.dumps(row) + "\n")


@dataclass(frozen=True)
class OverheadReport:
    total_s: float
    schedule_s: float
    policy_s: float
    overhead_pct: float


def measure_overhead(log: EventLog) -> OverheadReport:
    total = log.sim_end_s
    pct = 0.0 if total <= 0 else log.policy_wall_s / total * 100.0
    return OverheadReport(total_s=total, schedule_s=log.engine_wall_s, policy_s=log.policy_wall_s,
                          overhead_pct=pct)


def trace_arrays(trace: list[Request], predictor: LengthPredictor) -> TraceArrays:
    """Marshal a reference-shaped trace (+ device predictions) to SoA."""
    for a, b in zip(trace, trace[1:]):
        if b.arrival_time < a.arrival_time:
            raise ValueError("trace must be sorted by arrival time")
    if len({r.id for r in trace}) != len(trace):
        raise ValueError("trace contains duplicate request ids")
    ids = np.array([r.id for r in trace], np.int64)
    tout = np.array([r.true_output_len for r in trace], np.int32)
    if predictor.mode == ORACLE or not trace:
        pred = tout.copy()
    else:
        pred = predict_many(predictor, ids, tout)
    return TraceArrays(np.array([r.arrival_time for r in trace], np.float64),
                       np.array([r.ttft_slo for r in trace], np.float64),
                       np.array([r.tpot_slo for r in trace], np.float64),
                       np.array([r.prompt_len for r in trace], np.int32), tout, pred, ids,
                       np.array([r.category for r in trace], np.int32))


def _raise_status(status: int) -> None:
    if status & N.SIM_NO_WORK_RUNNING:
        raise EngineError("policy produced no work while requests are running")
    if status & N.SIM_NO_PROGRESS:
        raise EngineError("no progress possible: clock cannot advance")


def run_many(traces: list[list[Request]], configs: list[SimConfig], with_log: bool = True
             ) -> list[tuple[list[RequestOutcome], EventLog]]:
    """Many independent (trace, config) cells in one device launch."""
    if len(traces) != len(configs):
        raise ValueError("one config per trace")
    arrs = [trace_arrays(t, c.predictor) for t, c in zip(traces, configs)]
    cells = [Cell(k, cell_config_of(c)) for k, c in enumerate(configs)]
    tok = [int(a.true_out.sum()) for a in arrs]
    step_cap = max(tok + [1])
    id_cap = max([len(a) + t for a, t in zip(arrs, tok)] + [1])
    skip_cap = max([len(a) + 1 for a in arrs] + [1])
    t0 = time.perf_counter()
    eng = BatchEngine(arrs, cells, outcomes=True,
                      log_cells=list(range(len(cells))) if with_log else None,
                      log_steps=step_cap if with_log else 0, log_ids=id_cap,
                      log_skips=skip_cap)
    eng.launch()
    res = eng.results()
    wall = time.perf_counter() - t0
    out_all = eng.outcomes()
    results = []
    for k, (trace, cfg, arr) in enumerate(zip(traces, configs, arrs)):
        r = res[k]
        _raise_status(int(r["status"]))
        o = eng.sim_outcomes(k, out_all)
        # outcomes / log in the caller's classes (reference Status members keep
        # the reference summarize()'s identity checks true)
        fam = family(trace[0] if trace else None, cfg)
        by_code = (fam.Status.COMPLETED, fam.Status.REJECTED_TTFT,
                   fam.Status.REJECTED_ADMISSION, fam.Status.INCOMPLETE)
        outcomes = []
        for i, req in enumerate(trace):
            st = by_code[int(o["status"][i])]
            done = int(o["status"][i]) == N.COMPLETED
            outcomes.append(fam.RequestOutcome(
                id=req.id, status=st, ttft_slo=req.ttft_slo, tpot_slo=req.tpot_slo,
                category=req.category,
                first_token_time=float(o["first_token_time"][i]) if done else None,
                completion_time=float(o["completion_time"][i]) if done else None,
                ttft=float(o["ttft"][i]) if done else None,
                tpot=float(o["tpot"][i]) if done else None,
                slo_compliant=bool(o["compliant"][i])))
        log = fam.EventLog(sim_end_s=float(r["sim_end"]), engine_wall_s=wall,
                           policy_wall_s=wall)
        if with_log:
            _fill_log(log, eng.log(k), trace, cfg, dict(zip(arr.id.tolist(),
                                                            arr.predicted.tolist())), fam)
        results.append((outcomes, log))
    return results


def _fill_log(log: EventLog, lg: dict, trace: list[Request], cfg: SimConfig,
              pred: dict[int, int], fam) -> None:
    by_id = {r.id: r for r in trace}
    tokens: dict[int, int] = {}
    running: list[int] = []
    ia = ir = ib = 0
    records = cfg.policy == SCORPIO and cfg.scorpio.tpot_guard
    for s in range(len(lg["now"])):
        na, nr, nb = int(lg["n_admitted"][s]), int(lg["n_rejected"][s]), int(lg["n_batch"][s])
        adm = [int(x) for x in lg["adm_ids"][ia:ia + na]]
        rej = [(int(x) // 2, "rejected_admission" if int(x) % 2 else "rejected_ttft")
               for x in lg["rej_ids"][ir:ir + nr]]
        bat = [int(x) for x in lg["batch_ids"][ib:ib + nb]]
        recs = []
        if records:
            snap = [(i, by_id[i].tpot_slo, by_id[i].prompt_len + tokens.get(i, 0)) for i in running]
            for q, rid in enumerate(adm):
                v = lg["adm_rec"][ia + q]
                r = by_id[rid]
                recs.append(fam.AdmissionRecord(
                    now=float(lg["now"][s]), candidate_id=rid, candidate_tpot_slo=r.tpot_slo,
                    candidate_len=r.prompt_len, predicted_len=int(pred[rid]),
                    running=tuple(snap),
                    vbs=float(v[0]), l_avg=float(v[1]), min_slo=float(v[2]),
                    estimate=float(v[3]), threshold=float(v[4])))
                snap.append((rid, r.tpot_slo, r.prompt_len))
        ia, ir, ib = ia + na, ir + nr, ib + nb
        end = float(lg["end"][s])
        ms = float(lg["min_slo"][s])
        log.steps.append(fam.StepRecord(step=s, now_s=float(lg["now"][s]), end_s=end, admitted=adm,
                                    rejected=rej, batch=bat, vbs=float(lg["vbs"][s]),
                                    min_slo_s=None if np.isnan(ms) else ms,
                                    prefill_s=float(lg["prefill_s"][s]),
                                    decode_s=float(lg["decode_s"][s]), admissions=recs))
        for rid in adm:
            log.token_emits[rid] = [end]
            tokens[rid] = 1
            running.append(rid)
        for rid in bat:
            log.token_emits[rid].append(end)
            tokens[rid] += 1
        running = [i for i in running if tokens[i] < by_id[i].true_output_len]
    sn, st, sw = lg["skips"]
    log.idle_skips = [(float(a), float(b), int(c)) for a, b, c in zip(sn, st, sw)]


def run(trace: list[Request], config: SimConfig) -> tuple[list[RequestOutcome], EventLog]:
    """Simulate one trace under one policy on the device (simengine.py:168-303)."""
    return run_many([trace], [config])[0]
