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
