"""Golden outputs of the UNPATCHED reference for the Level-1 drop-in test
(tests/test_gpu_reference_dropin.py).  Run here, where /root/reference exists:

    python tests/golden/make_dropin_golden.py [--ref /root/reference/pkg/src]

Writes tests/golden/ref_dropin.json:
  * c07: ``slosim.report.sweep`` of the acceptance overload trace at its native
    rate under scorpio and greedy (test_acceptance.py:308-337) -> to_dict();
  * c08: ``slosim.report.ablation`` on the same trace (test_acceptance.py:340-362);
  * plan_only: ``slosim.simengine.run`` of config 1's first 150 requests
    (outcome tuples + decision-log JSONL text), for the patch that replaces only
    the policy functions (plan_step / ttft_guard / select_batch / admit).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    sys.path.insert(0, args.ref)
    from slosim.core import SloCategory, SloCategoryTable
    from slosim.costmodel import ItlParams, PrefillParams
    from slosim.predictor import Bucketing, LengthPredictor
    from slosim.report import ablation, sweep
    from slosim.sched_baselines import BaselineConfig
    from slosim.simengine import SimConfig, run
    from slosim.workload import LogNormalDist, WorkloadSpec, generate

    itl = ItlParams(alpha=1e-6, beta=1e-3, gamma=1e-5, delta=5e-3, epsilon=1.1)
    pre = PrefillParams(phi=0.004, theta=128.0, alpha_p=2e-5, beta_p=1.5e-3)
    pred = LengthPredictor(mode="oracle", bucketing=Bucketing.equal_width(100, 4096))
    ov = WorkloadSpec(qps=25.0, duration=90.0, seed=20240601,
                      prompt_len_dist=LogNormalDist(5.0, 0.7),
                      output_len_dist=LogNormalDist(4.0, 0.7), category_weights=(1.0,) * 6)
    trace = generate(ov)[:2000]
    cfg = SimConfig(policy="scorpio", itl_params=itl, prefill_params=pre, predictor=pred,
                    baseline=BaselineConfig(max_batch_size=256))
    qps = len(trace) / trace[-1].arrival_time
    out = {"qps": qps}
    out["c07"] = sweep(trace, [qps], ["scorpio", "greedy"], cfg, base_seed=1).to_dict()
    out["c08"] = {k: v.to_dict() for k, v in ablation(trace, cfg).items()}
    three = SloCategoryTable(rows=(SloCategory(1, 0.5, 0.030), SloCategory(2, 2.0, 0.050),
                                   SloCategory(3, 7.5, 0.100)))
    c1 = generate(WorkloadSpec(qps=8.0, duration=150.0, seed=7,
                               prompt_len_dist=LogNormalDist(5.0, 0.7),
                               output_len_dist=LogNormalDist(4.0, 0.7),
                               category_weights=(1.0,) * 3, slo_table=three))[:150]
    outcomes, log = run(c1, cfg)
    out["plan_only"] = {
        "outcomes": [[o.id, o.status.value, o.first_token_time, o.completion_time, o.ttft,
                      o.tpot, o.slo_compliant] for o in outcomes],
        "n_steps": len(log.steps),
    }
    jp = os.path.join(HERE, "_tmp_dropin.jsonl")
    log.to_jsonl(jp)
    with open(jp, encoding="utf-8") as f:
        out["plan_only"]["jsonl"] = f.read()
    os.remove(jp)
    with open(os.path.join(HERE, "ref_dropin.json"), "w") as f:
        json.dump(out, f)
    c = out["c07"]["cells"]
    print("c07", {k: (v["goodput_rps"], v["adherence"]) for k, v in c.items()})


if __name__ == "__main__":
    main()
