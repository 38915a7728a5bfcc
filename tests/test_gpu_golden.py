"""GPU parity against the reference-generated fixtures (tests/golden).

Every case is run through the C ABI (sl_run_batch) in ONE batched launch; each
cell must reproduce the reference's per-request outcomes bit for bit, its
EventLog step records (now/end/prefill/decode/vbs/min_slo and the admitted /
rejected / batch id lists), and the work-step digest.
"""

import numpy as np
import pytest

from tests._golden import OUTCOME_FIELDS, load_cases, same_float

pytestmark = pytest.mark.gpu


def _cells(cases):
    from paper_2505_23022_b200.batch import Cell, CellConfig, TraceArrays

    traces, cells = [], []
    for k, c in enumerate(cases):
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
    return traces, cells


@pytest.fixture(scope="module", params=["auto", "general"])
def gpu_run(request):
    from paper_2505_23022_b200 import _native as N
    from paper_2505_23022_b200.batch import BatchEngine

    cases = load_cases()
    traces, cells = _cells(cases)
    max_steps = max(c["n_steps"] for c in cases) + 1
    max_ids = max(len(c["log"]["ids"]) if c["keep_log"] else 0 for c in cases) + 1
    log_cells = [k for k, c in enumerate(cases) if c["keep_log"]]
    mode = N.MODE_AUTO if request.param == "auto" else N.MODE_GENERAL
    eng = BatchEngine(traces, cells, outcomes=True, log_cells=log_cells,
                      log_steps=max_steps, log_ids=max_ids, mode=mode)
    eng.launch()
    res = eng.results()
    out = eng.outcomes()
    return cases, eng, res, out


@pytest.mark.parametrize("k", range(len(load_cases())), ids=[c["name"] for c in load_cases()])
def test_gpu_matches_reference(gpu_run, k):
    cases, eng, res, out = gpu_run
    c = cases[k]
    r = res[k]
    assert r["status"] == 0, r["status"]
    o = eng.sim_outcomes(k, out)
    for f in OUTCOME_FIELDS:
        want = c["outcomes"][f]
        if want.dtype.kind == "f":
            assert same_float(o[f], want), f
        else:
            assert np.array_equal(o[f].astype(want.dtype), want), f
    assert r["n_steps"] == c["n_steps"]
    assert r["n_idle_skips"] == c["n_idle_skips"]
    assert r["sim_end"] == c["sim_end"]
    assert r["compliant"] == c["compliant"]
    assert r["goodput"] == c["goodput"]
    assert r["adherence"] == c["adherence"]
    assert int(r["digest"]) == c["digest"]
    if c["keep_log"]:
        lg = eng.log(k)
        want = c["log"]
        for f in ("now", "end", "prefill_s", "decode_s", "vbs", "min_slo"):
            assert same_float(lg[f], want[f]), f
        counts = np.stack([lg["n_admitted"], lg["n_rejected"], lg["n_batch"]], 1)
        assert np.array_equal(counts, want["counts"].reshape(-1, 3))
        ids = []
        ia = ir = ib = 0
        for na, nr, nb in counts:
            ids += list(lg["adm_ids"][ia:ia + na]) + list(lg["rej_ids"][ir:ir + nr]) + \
                list(lg["batch_ids"][ib:ib + nb])
            ia, ir, ib = ia + na, ir + nr, ib + nb
        assert np.array_equal(np.array(ids, np.int64), want["ids"])
