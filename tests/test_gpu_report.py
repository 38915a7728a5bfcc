"""RunReport reductions on the device (sl_report_batch) against the host
restatement of report.summarize (report.py:71-127) on the same outcomes:
nearest-rank p50/p90/p99 of TTFT (s) and TPOT (ms) over completed requests and
per-category totals / compliant counts, exactly."""

import math

import numpy as np
import pytest

from tests._sweepcase import grid

pytestmark = pytest.mark.gpu


def nearest_rank(values, pct):  # report.py:_nearest_rank
    if len(values) == 0:
        return float("nan")
    ordered = sorted(values)
    return ordered[max(1, math.ceil(pct / 100.0 * len(ordered))) - 1]


def test_device_report_matches_summarize():
    from paper_2505_23022_b200.batch import BatchEngine

    traces, cells = grid(n_req=1200)
    eng = BatchEngine(traces, cells, outcomes=True)
    eng.launch()
    rows, counts = eng.report(traces, n_categories=8)
    out = eng.outcomes()
    for k, c in enumerate(cells):
        o = eng.sim_outcomes(k, out)
        done = o["status"] == 0
        ttft = [float(x) for x in o["ttft"][done]]
        tpot_ms = [float(x) * 1000.0 for x in o["tpot"][done]]
        r = rows[k]
        assert r["n_completed"] == int(done.sum())
        for p, f in zip((50, 90, 99), ("p50", "p90", "p99")):
            want_t, want_p = nearest_rank(ttft, p), nearest_rank(tpot_ms, p)
            assert (np.isnan(want_t) and np.isnan(r["ttft_" + f])) or r["ttft_" + f] == want_t, k
            assert (np.isnan(want_p) and np.isnan(r["tpot_ms_" + f])) or r["tpot_ms_" + f] == want_p
        cat = np.asarray(traces[c.trace].category)
        for q in range(8):
            sel = cat == q
            assert counts[k, q, 0] == int(sel.sum())
            assert counts[k, q, 1] == int((o["compliant"][sel] != 0).sum())


def test_summarize_batch_matches_summarize():
    """The batched RunReport equals summarize() on each cell's outcomes, every
    field including the cumulative SLO-met series."""
    from paper_2505_23022_b200 import core
    from paper_2505_23022_b200.batch import BatchEngine
    from paper_2505_23022_b200.report import summarize, summarize_batch

    traces, cells = grid(n_req=600, rates=(4.0, 16.0), scales=[0.5, 1.0, 2.0])
    eng = BatchEngine(traces, cells, outcomes=True)
    eng.launch()
    got = summarize_batch(eng, traces)
    out = eng.outcomes()
    rows = eng.results()
    codes = list(core.Status)  # C ABI status codes 0..3
    for k, c in enumerate(cells):
        o = eng.sim_outcomes(k, out)
        t = traces[c.trace]
        outcomes = []
        for i in range(len(t)):
            st = codes[int(o["status"][i])]
            done = st is core.Status.COMPLETED
            outcomes.append(core.RequestOutcome(
                id=int(t.id[i]), status=st, category=int(t.category[i]),
                ttft_slo=float(t.ttft_slo[i] * c.slo_scale),
                tpot_slo=float(t.tpot_slo[i] * c.slo_scale),
                ttft=float(o["ttft"][i]) if done else None,
                tpot=float(o["tpot"][i]) if done else None,
                completion_time=float(o["completion_time"][i]) if done else None,
                slo_compliant=bool(o["compliant"][i])))
        want = summarize(outcomes, float(rows[k]["horizon"])).to_dict()
        have = got[k].to_dict()
        assert len(have["cumulative_slo_met"]) == rows[k]["compliant"]
        assert json_equal(have, want), k


def json_equal(a, b):
    import json

    return json.dumps(a, sort_keys=True) == json.dumps(b, sort_keys=True)


def test_cumulative_radix_sort_edge_cases():
    """The device series is the sorted multiset of compliant completion times:
    random times (all 8 radix passes live), equal times, an empty series."""
    import torch

    from paper_2505_23022_b200 import _native as N
    from paper_2505_23022_b200.batch import BatchEngine

    traces, cells = grid(n_req=400, rates=(4.0, 32.0), scales=[0.5, 2.0])
    eng = BatchEngine(traces, cells, outcomes=True)
    eng.launch()
    rng = np.random.default_rng(5)
    n = eng.total_slots
    comp = rng.random(n) < 0.7
    times = rng.random(n) * 10.0 ** rng.integers(-3, 4, n)
    times[: n // 3] = 1.25  # ties
    comp[eng.sims_host[0]["out_offset"]: eng.sims_host[0]["out_offset"] + 400] = False
    eng._out["compliant"][:n].copy_(torch.from_numpy(comp.astype(np.int8)))
    eng._out["completion_time"][:n].copy_(torch.from_numpy(times))
    got = eng.cumulative()
    for k, s in enumerate(eng.sims_host):
        b = int(s["out_offset"])
        m = len(traces[s["trace"]])
        want = np.sort(times[b:b + m][comp[b:b + m]])
        assert np.array_equal(got[k], want), k
    assert len(got[0]) == 0


def test_report_with_no_completions():
    """Cells whose SLOs reject everything: NaN percentiles, n_completed 0, an
    empty cumulative series, per-category totals still counted."""
    from paper_2505_23022_b200.batch import BatchEngine
    from paper_2505_23022_b200.report import summarize_batch

    traces, cells = grid(n_req=300, rates=(32.0,), scales=[1e-4, 1.0])
    eng = BatchEngine(traces, cells, outcomes=True)
    eng.launch()
    rows, counts = eng.report(traces)
    series = eng.cumulative()
    rep = summarize_batch(eng, traces)
    res = eng.results()
    for k in range(len(cells)):
        if res[k]["completed"] == 0:
            assert rows[k]["n_completed"] == 0
            assert np.isnan(rows[k]["ttft_p50"]) and np.isnan(rows[k]["tpot_ms_p99"])
            assert len(series[k]) == 0 and rep[k].cumulative == []
        assert counts[k, :, 0].sum() == len(traces[cells[k].trace])
    assert (res["completed"] == 0).any()


def test_report_and_jsonl_match_reference_bytes(golden):
    """Every golden case through the device engine: summarize_batch().to_dict()
    equals the reference's summarize(...).to_dict() (make_golden.py), key order
    included (status_counts in first-occurrence order, report.py:104-106), and
    run()'s EventLog.to_jsonl bytes equal the reference's (simengine.py:106-137)."""
    import json
    import os
    import tempfile

    from paper_2505_23022_b200.batch import BatchEngine, Cell, CellConfig, TraceArrays
    from paper_2505_23022_b200.core import Request
    from paper_2505_23022_b200.predictor import Bucketing, LengthPredictor
    from paper_2505_23022_b200.report import summarize_batch
    from paper_2505_23022_b200.sched_baselines import BaselineConfig
    from paper_2505_23022_b200.sched_scorpio import ScorpioConfig
    from paper_2505_23022_b200.costmodel import ItlParams, PrefillParams
    from paper_2505_23022_b200.simengine import SimConfig, run_many
    from tests._golden import HERE

    want = json.load(open(os.path.join(HERE, "reports.json")))
    jsonl = np.load(os.path.join(HERE, "decisions_jsonl.npz"))
    traces, cells = [], []
    for k, c in enumerate(golden):
        t = c["trace"]
        traces.append(TraceArrays(t["arrival"], t["ttft_slo"], t["tpot_slo"], t["prompt_len"],
                                  t["true_out"], t["predicted"], t["id"], t["category"]))
        cells.append(Cell(k, CellConfig(policy=c["policy"], itl=tuple(c["itl"]),
                                        prefill=tuple(c["prefill"]), ttft_guard=c["ttft_guard"],
                                        tpot_guard=c["tpot_guard"],
                                        admission_min=c["admission_min"],
                                        max_batch_size=c["max_batch_size"],
                                        prefill_priority=c["prefill_priority"],
                                        horizon=c["horizon"])))
    eng = BatchEngine(traces, cells, outcomes=True)
    eng.launch()
    reps = summarize_batch(eng, traces)
    for c, r in zip(golden, reps):
        got = r.to_dict()
        assert json.dumps(got) == json.dumps(want[c["name"]]), c["name"]
    # decision-log bytes through the drop-in run() (device log -> EventLog)
    jcases = [c for c in golden if c["name"] in jsonl.files]
    assert len(jcases) >= 10
    trs, cfgs = [], []
    for c in jcases:
        t = c["trace"]
        trs.append([Request(id=int(t["id"][i]), arrival_time=float(t["arrival"][i]),
                            prompt_len=int(t["prompt_len"][i]),
                            true_output_len=int(t["true_out"][i]),
                            ttft_slo=float(t["ttft_slo"][i]), tpot_slo=float(t["tpot_slo"][i]),
                            category=int(t["category"][i])) for i in range(c["n"])])
        pd = c["predictor"]
        pred = LengthPredictor(mode=pd["mode"],
                               bucketing=Bucketing.equal_width(pd["num_buckets"], pd["max_len"]),
                               error_prob=pd["error_prob"], error_spread=pd["error_spread"],
                               rng_seed=int(pd["rng_seed"]))
        cfgs.append(SimConfig(policy=c["policy"], itl_params=ItlParams(*c["itl"]),
                              prefill_params=PrefillParams(*c["prefill"]), predictor=pred,
                              scorpio=ScorpioConfig(c["ttft_guard"], c["tpot_guard"],
                                                    c["admission_min"]),
                              baseline=BaselineConfig(max_batch_size=c["max_batch_size"],
                                                      prefill_priority=c["prefill_priority"]),
                              horizon=c["horizon"]))
    for c, (outs, log) in zip(jcases, run_many(trs, cfgs)):
        fd, p = tempfile.mkstemp(suffix=".jsonl")
        os.close(fd)
        try:
            log.to_jsonl(p)
            got = open(p, "rb").read()
        finally:
            os.remove(p)
        assert got == jsonl[c["name"]].tobytes(), c["name"]
