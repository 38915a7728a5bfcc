"""INTEGRATION.md Level 1 against the UNMODIFIED reference package.

``baseline/_ref`` holds ``slosim`` installed from /root/reference/pkg
(tools/install_reference.sh, run by __graft_entry__.build()).  The tests patch
its module attributes with this package's device implementations, call the
reference's OWN entry points with the reference's OWN objects, and compare
with what the unpatched reference produced in the build container
(tests/golden/ref_dropin.json, tests/golden/make_dropin_golden.py):

* engine swap: ``slosim.simengine.run`` and ``slosim.report.run`` -> device
  engine; ``slosim.report.sweep`` / ``ablation`` then reproduce c07 / c08
  (test_acceptance.py:308-362) -- goodput 11.54 vs 0.063, adherence 0.5005 --
  field for field, through the reference's own ``summarize``;
* policy swap: ``slosim.sched_scorpio.plan_step`` (what ``ScorpioPolicy.plan``
  calls, sched_scorpio.py:343-346) -> device plan kernels, inside the
  reference's own Python engine loop; outcomes and decision-log bytes equal.
"""

import json
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
GOLD = os.path.join(ROOT, "tests", "golden", "ref_dropin.json")


@pytest.fixture(scope="module")
def slosim():
    if not os.path.isdir(os.path.join(REF, "slosim")):
        pytest.fail("baseline/_ref/slosim missing: run tools/install_reference.sh (build())")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import slosim  # noqa: F401
    import slosim.report
    import slosim.sched_scorpio
    import slosim.simengine

    return sys.modules["slosim"]


@pytest.fixture(scope="module")
def gold():
    return json.load(open(GOLD))


def _overload(slosim):
    from slosim.costmodel import ItlParams, PrefillParams
    from slosim.predictor import Bucketing, LengthPredictor
    from slosim.sched_baselines import BaselineConfig
    from slosim.simengine import SimConfig
    from slosim.workload import LogNormalDist, WorkloadSpec, generate

    spec = WorkloadSpec(qps=25.0, duration=90.0, seed=20240601,
                        prompt_len_dist=LogNormalDist(5.0, 0.7),
                        output_len_dist=LogNormalDist(4.0, 0.7), category_weights=(1.0,) * 6)
    trace = generate(spec)[:2000]
    cfg = SimConfig(policy="scorpio",
                    itl_params=ItlParams(alpha=1e-6, beta=1e-3, gamma=1e-5, delta=5e-3,
                                         epsilon=1.1),
                    prefill_params=PrefillParams(phi=0.004, theta=128.0, alpha_p=2e-5,
                                                 beta_p=1.5e-3),
                    predictor=LengthPredictor(mode="oracle",
                                              bucketing=Bucketing.equal_width(100, 4096)),
                    baseline=BaselineConfig(max_batch_size=256))
    return trace, cfg


def test_level1_engine_swap_c07_c08(slosim, gold, monkeypatch):
    import paper_2505_23022_b200.simengine as dev

    monkeypatch.setattr(slosim.simengine, "run", dev.run)
    monkeypatch.setattr(slosim.report, "run", dev.run)  # report.py imports run by name
    trace, cfg = _overload(slosim)
    qps = len(trace) / trace[-1].arrival_time
    assert qps == gold["qps"]
    res = slosim.report.sweep(trace, [qps], ["scorpio", "greedy"], cfg, base_seed=1)
    got = res.to_dict()
    assert got == gold["c07"]
    sc = res.cells[(qps, "scorpio")].report
    gr = res.cells[(qps, "greedy")].report
    assert round(sc.goodput, 2) == 11.54 and sc.adherence == 0.5005
    assert gr.goodput > 0 and sc.goodput >= 1.5 * gr.goodput  # c07 floors
    # the outcomes really are the reference's classes (summarize's `is` checks)
    outs, log = slosim.simengine.run(trace[:50], cfg)
    assert all(type(o) is slosim.core.RequestOutcome for o in outs)
    assert all(isinstance(o.status, slosim.core.Status) for o in outs)
    assert type(log) is slosim.simengine.EventLog
    abl = {k: v.to_dict() for k, v in slosim.report.ablation(trace, cfg).items()}
    assert abl == gold["c08"]


def test_level1_policy_swap_plan_step(slosim, gold, monkeypatch, tmp_path):
    import paper_2505_23022_b200.sched_scorpio as dev
    from slosim.core import SloCategory, SloCategoryTable
    from slosim.workload import LogNormalDist, WorkloadSpec, generate

    for name in ("plan_step", "ttft_guard", "select_batch", "admit", "vbs"):
        monkeypatch.setattr(slosim.sched_scorpio, name, getattr(dev, name))
    _, cfg = _overload(slosim)
    three = SloCategoryTable(rows=(SloCategory(1, 0.5, 0.030), SloCategory(2, 2.0, 0.050),
                                   SloCategory(3, 7.5, 0.100)))
    c1 = generate(WorkloadSpec(qps=8.0, duration=150.0, seed=7,
                               prompt_len_dist=LogNormalDist(5.0, 0.7),
                               output_len_dist=LogNormalDist(4.0, 0.7),
                               category_weights=(1.0,) * 3, slo_table=three))[:150]
    outcomes, log = slosim.simengine.run(c1, cfg)  # the reference's own Python engine loop
    got = [[o.id, o.status.value, o.first_token_time, o.completion_time, o.ttft, o.tpot,
            o.slo_compliant] for o in outcomes]
    assert got == gold["plan_only"]["outcomes"]
    assert len(log.steps) == gold["plan_only"]["n_steps"]
    p = tmp_path / "d.jsonl"
    log.to_jsonl(p)
    assert p.read_text(encoding="utf-8") == gold["plan_only"]["jsonl"]
