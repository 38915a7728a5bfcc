"""Parity at BASELINE's full size: the bench workload itself (config 3: 64 rates x
64 SLO scales, 10k requests per sim, one sl_run_batch launch over 4,096 sims).

* every cell: size-independent invariants of simengine.run (conservation of
  requests, compliant <= completed, violation counts <= completed, goodput ==
  compliant / sim_end, adherence == compliant / total, no engine error, request
  steps >= steps);
* every one of the 4,096 cells (and of config 4's 16,384): every result-row
  field and the work-step digest bit-exact against the C oracle on the same
  traces;
* 48 stratified cells (every rate row, scales spread over the axis, the 2 req/s
  critical-path cells included): also every request's outcome (status,
  completion step, first-token and completion times, TTFT, TPOT, compliance).
"""

OUTCOME_FIELDS = ("status", "compliant", "completion_step", "first_token_time",
                  "completion_time", "ttft", "tpot")


def assert_outcomes_equal(got, ref, where):
    for f in OUTCOME_FIELDS:
        a, b = np.asarray(got[f]), np.asarray(ref[f])
        if a.dtype.kind == "f":
            assert same_float(a, b), (where, f)
        else:
            assert np.array_equal(a, b), (where, f, int((a != b).sum()))

import numpy as np
import pytest

from tests._golden import same_float

pytestmark = pytest.mark.gpu

FIELDS = ("n_steps", "n_plans", "n_idle_skips", "request_steps", "completed", "compliant",
          "rejected_ttft", "rejected_admission", "incomplete", "ttft_violations",
          "tpot_violations")


@pytest.fixture(scope="module")
def config3():
    import torch

    from paper_2505_23022_b200.sweep import SweepGrid, build_local

    grid = SweepGrid()  # the bench's config-3 grid
    eng, owned, traces = build_local(grid, outcomes=True, device=torch.device("cuda", 0))
    eng.launch()
    return grid, eng.results(), traces, eng


def test_config3_invariants_every_cell(config3):
    grid, res, _, _ = config3
    assert len(res) == 4096
    assert ((res["status"] & 3) == 0).all()
    n = res["total"]
    assert (n == grid.n_requests).all()
    assert (res["completed"] + res["rejected_ttft"] + res["rejected_admission"] +
            res["incomplete"] == n).all()
    assert (res["incomplete"] == 0).all()  # no horizon: every request resolves
    assert (res["compliant"] <= res["completed"]).all()
    assert (res["ttft_violations"] <= res["completed"]).all()
    assert (res["tpot_violations"] <= res["completed"]).all()
    assert (res["request_steps"] >= res["n_steps"]).all()
    h = np.maximum(res["sim_end"], 1e-12)
    assert np.array_equal(res["goodput"], res["compliant"] / h)
    assert np.array_equal(res["adherence"], res["compliant"] / n)


def test_config3_sampled_cells_match_oracle(config3):
    from oracle import oracle as orc

    grid, res, traces, eng = config3
    ns = len(grid.scales)
    scale_pick = [0, 9, 21, 32, 45, 63]
    rate_pick = list(range(0, 64, 8)) + [1, 63]
    cells = sorted({(ri, si) for ri in rate_pick for si in scale_pick})[:48]
    params = orc.make_params(itl=grid.config.itl, prefill=grid.config.prefill)
    jobs = []
    for ri, si in cells:
        t, s = traces[ri], float(grid.scales[si])
        jobs.append(dict(arrival=t.arrival, ttft_slo=t.ttft_slo * s, tpot_slo=t.tpot_slo * s,
                         prompt_len=t.prompt_len, true_out=t.true_out, ids=t.id,
                         predicted=t.predicted, params=params))
    refs = orc.run_many(jobs)
    for (ri, si), ref in zip(cells, refs):
        r, sm = res[ri * ns + si], ref["summary"]
        assert ref["rc"] == 0
        for f in FIELDS:
            assert r[f] == sm[f], (ri, si, f, r[f], sm[f])
        for f in ("sim_end", "goodput", "adherence"):
            assert same_float([r[f]], [sm[f]]), (ri, si, f)
        assert int(r["digest"]) == sm["digest"], (ri, si)
        assert_outcomes_equal(eng.cell_outcomes(ri * ns + si), ref, (ri, si))


def _all_cells_vs_oracle(res, traces, scales, config, batch=256):
    """Every cell's result row and work-step digest against the C oracle on the
    same traces (outcome arrays are dropped per batch to bound host memory)."""
    from oracle import oracle as orc

    params = orc.make_params(itl=config.itl, prefill=config.prefill)
    ns = len(scales)
    cells = [(ri, si) for ri in range(len(traces)) for si in range(ns)]
    for b in range(0, len(cells), batch):
        chunk = cells[b:b + batch]
        jobs = []
        for ri, si in chunk:
            t, s = traces[ri], float(scales[si])
            jobs.append(dict(arrival=t.arrival, ttft_slo=t.ttft_slo * s, tpot_slo=t.tpot_slo * s,
                             prompt_len=t.prompt_len, true_out=t.true_out, ids=t.id,
                             predicted=t.predicted, params=params))
        for (ri, si), ref in zip(chunk, orc.run_many(jobs)):
            r, sm = res[ri * ns + si], ref["summary"]
            assert ref["rc"] == 0
            for f in FIELDS:
                assert r[f] == sm[f], (ri, si, f, r[f], sm[f])
            for f in ("sim_end", "goodput", "adherence"):
                assert same_float([r[f]], [sm[f]]), (ri, si, f)
            assert int(r["digest"]) == sm["digest"], (ri, si)


def test_config3_every_cell_matches_oracle(config3):
    """All 4,096 cells of the bench workload: every result-row field (counts,
    request-steps, sim_end, goodput, adherence) and the work-step digest --
    every admit / reject / batch decision and step end time -- bit-exact."""
    grid, res, traces, _ = config3
    _all_cells_vs_oracle(res, traces, grid.scales, grid.config)


def test_config4_sampled_cells_match_oracle():
    """Config 4 at full size (16,384 ShareGPT-shaped sims with the device
    noisy-bucket predictor in the loop -- its stream is pinned to numpy's in
    test_predictor.py): engine invariants on every cell and 24 stratified cells
    bit-exact vs the oracle fed the same predicted lengths."""
    import torch

    from oracle import oracle as orc
    from paper_2505_23022_b200.batch import BatchEngine, Cell
    from paper_2505_23022_b200.predictor import Bucketing, LengthPredictor
    from paper_2505_23022_b200.seeds import derive_seed
    from paper_2505_23022_b200.sweep import SweepGrid

    dev = torch.device("cuda", 0)
    grid = SweepGrid(rates=tuple(np.linspace(2.0, 32.0, 128)),
                     scales=tuple(np.geomspace(0.5, 2.0, 128)), prompt=(4.6, 0.9),
                     output=(4.5, 0.9))
    traces = [grid.trace_for_rate(q) for q in grid.rates]
    pred = LengthPredictor("noisy_bucket", Bucketing.equal_width(100, 4096), error_prob=0.73,
                           error_spread=3, rng_seed=derive_seed(0, "predictor"))
    ids = np.concatenate([t.id for t in traces])
    tout = np.concatenate([t.true_out for t in traces])
    out, _ = pred.predict_device(torch.from_numpy(ids).to(dev), torch.from_numpy(tout).to(dev))
    p = out.cpu().numpy()
    k = 0
    for t in traces:
        t.predicted = p[k: k + len(t)].copy()
        k += len(t)
    cells = [Cell(ri, grid.config, slo_scale=float(sc)) for ri in range(128) for sc in grid.scales]
    eng = BatchEngine(traces, cells, outcomes=True, device=dev)
    eng.launch()
    res = eng.results()
    assert ((res["status"] & 3) == 0).all()
    assert (res["completed"] + res["rejected_ttft"] + res["rejected_admission"] +
            res["incomplete"] == res["total"]).all()
    params = orc.make_params(itl=grid.config.itl, prefill=grid.config.prefill)
    pick = [(ri, si) for ri in (0, 1, 17, 45, 90, 127) for si in (0, 40, 85, 127)]
    jobs = []
    for ri, si in pick:
        t, s = traces[ri], float(grid.scales[si])
        jobs.append(dict(arrival=t.arrival, ttft_slo=t.ttft_slo * s, tpot_slo=t.tpot_slo * s,
                         prompt_len=t.prompt_len, true_out=t.true_out, ids=t.id,
                         predicted=t.predicted, params=params))
    for (ri, si), ref in zip(pick, orc.run_many(jobs)):
        r, sm = res[ri * 128 + si], ref["summary"]
        for f in FIELDS:
            assert r[f] == sm[f], (ri, si, f, r[f], sm[f])
        assert same_float([r["goodput"]], [sm["goodput"]]) and int(r["digest"]) == sm["digest"]
        assert_outcomes_equal(eng.cell_outcomes(ri * 128 + si), ref, (ri, si))
    # and every one of the 16,384 cells: result row + work-step digest
    _all_cells_vs_oracle(res, traces, grid.scales, grid.config)
