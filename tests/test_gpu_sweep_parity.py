"""At-scale parity: one batched sl_run_batch launch over a rate x SLO-scale grid
(+ ablations, r_only, horizon, baselines, 128-bit credits) against the C oracle,
per cell: digest, every result-row field and every per-request outcome, bit-exact."""

import numpy as np
import pytest

from tests._golden import same_float
from tests._sweepcase import grid, oracle_job

pytestmark = pytest.mark.gpu

FIELDS = ("n_steps", "n_plans", "n_idle_skips", "request_steps", "completed", "compliant",
          "rejected_ttft", "rejected_admission", "incomplete", "ttft_violations",
          "tpot_violations")


@pytest.mark.parametrize("mode", ["auto", "general"])
def test_sweep_grid_matches_oracle(mode):
    from oracle import oracle as orc
    from paper_2505_23022_b200 import _native as N
    from paper_2505_23022_b200.batch import BatchEngine

    traces, cells = grid()
    eng = BatchEngine(traces, cells, outcomes=True,
                      mode=N.MODE_AUTO if mode == "auto" else N.MODE_GENERAL)
    eng.launch()
    res = eng.results()
    out = eng.outcomes()
    refs = orc.run_many([oracle_job(traces[c.trace], c) for c in cells])
    assert any(int(s["credit_wide"]) for s in eng.sims_host)
    for k, (c, ref) in enumerate(zip(cells, refs)):
        r, sm = res[k], ref["summary"]
        assert ref["rc"] == 0 and r["status"] == 0
        for f in FIELDS:
            assert r[f] == sm[f], (k, f, r[f], sm[f])
        for f in ("sim_end", "goodput", "adherence", "horizon"):
            assert same_float([r[f]], [sm[f]]), (k, f)
        assert int(r["digest"]) == sm["digest"], k
        o = eng.sim_outcomes(k, out)
        for f in ("status", "compliant", "completion_step"):
            assert np.array_equal(o[f].astype(np.int64), ref[f].astype(np.int64)), (k, f)
        for f in ("first_token_time", "completion_time", "ttft", "tpot"):
            assert same_float(o[f], ref[f]), (k, f)


def test_relaunch_is_deterministic():
    from paper_2505_23022_b200.batch import BatchEngine

    traces, cells = grid(n_req=400, rates=(4.0, 16.0), scales=[0.5, 1.0, 2.0])
    eng = BatchEngine(traces, cells)
    eng.launch()
    a = eng.results()
    eng.launch()
    b = eng.results()
    assert a.tobytes() == b.tobytes()
