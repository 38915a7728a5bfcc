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
    """The batched RunReport equals summarize() on each cell's outcomes (all fields
    but the per-request cumulative series)."""
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
        want.pop("cumulative_slo_met")
        have.pop("cumulative_slo_met")
        assert json_equal(have, want), k


def json_equal(a, b):
    import json

    return json.dumps(a, sort_keys=True) == json.dumps(b, sort_keys=True)
