"""Pin the C restatement (oracle/) to outputs of the real reference.

Every fixture in tests/golden/sims.npz was produced by ``slosim.simengine.run``
(pkg/src/slosim/simengine.py:168) in the build container; here the oracle must
reproduce outcomes bit for bit (fp64 compared as bit patterns), the per-step
decision log, and the work-step digest.
"""

import numpy as np
import pytest

from tests._golden import OUTCOME_FIELDS, load_cases, oracle_params, same_float

CASES = load_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference(case):
    from oracle import oracle as orc

    t = case["trace"]
    log_steps = case["n_steps"] + 1 if case["keep_log"] else 0
    res = orc.run_sim(t["arrival"], t["ttft_slo"], t["tpot_slo"], t["prompt_len"], t["true_out"],
                      t["id"], t["predicted"], oracle_params(case), log_steps=log_steps,
                      log_ids=int(len(case["log"]["ids"])) + 1 if case["keep_log"] else 0)
    assert res["rc"] == 0
    sm = res["summary"]
    for k in OUTCOME_FIELDS:
        want = case["outcomes"][k]
        if want.dtype.kind == "f":
            assert same_float(res[k], want), k
        else:
            assert np.array_equal(res[k], want), k
    assert sm["n_steps"] == case["n_steps"]
    assert sm["n_idle_skips"] == case["n_idle_skips"]
    assert sm["sim_end"] == case["sim_end"]
    assert sm["compliant"] == case["compliant"]
    assert sm["goodput"] == case["goodput"]
    assert sm["adherence"] == case["adherence"]
    assert sm["digest"] == case["digest"]
    if case["keep_log"]:
        lg, want = res["log"], case["log"]
        assert lg["overflow"] == 0
        for k in ("now", "end", "prefill_s", "decode_s", "vbs", "min_slo"):
            assert same_float(lg[k], want[k]), k
        counts = np.stack([lg["n_admitted"], lg["n_rejected"], lg["n_batch"]], 1)
        assert np.array_equal(counts, want["counts"].reshape(-1, 3))
        assert np.array_equal(lg["ids"], want["ids"])
