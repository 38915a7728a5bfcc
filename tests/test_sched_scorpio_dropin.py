"""The reference's scorpio unit scenarios (pkg/tests/test_sched_scorpio.py) run
against the drop-in API, whose decisions execute in the sm_100a plan kernels."""

from fractions import Fraction

import numpy as np
import pytest

from paper_2505_23022_b200.core import Request, Status
from paper_2505_23022_b200.costmodel import ItlParams, PrefillParams
from paper_2505_23022_b200.predictor import Bucketing, LengthPredictor
from paper_2505_23022_b200.schedtypes import RunningEntry, SchedulerState, WaitingItem
from paper_2505_23022_b200.sched_scorpio import (R_ONLY, ScorpioConfig, admit, plan_step,
                                                 plan_step_batch, select_batch, trp, ttft_guard,
                                                 vbs)

ITL = ItlParams(alpha=1e-6, beta=1e-3, gamma=1e-5, delta=5e-3, epsilon=1.0)
PRE = PrefillParams(phi=0.020, theta=128.0, alpha_p=1e-4, beta_p=7e-3)
PRED = LengthPredictor(mode="oracle", bucketing=Bucketing.equal_width(10, 1000))


def rq(i, tpot=0.030, ttft=1.0, arrival=0.0, prompt=100, output=10):
    return Request(id=i, arrival_time=arrival, prompt_len=prompt, true_output_len=output,
                   ttft_slo=ttft, tpot_slo=tpot)


def run_entry(r, predicted=10, tokens=0):
    e = RunningEntry(request=r, predicted_len=predicted, prefill_s=0.02)
    e.tokens_generated = tokens
    return e


def wait_item(r, predicted=10, prefill_s=0.02):
    return WaitingItem(request=r, predicted_len=predicted, prefill_s=prefill_s)


def test_trp_values_and_guards():
    assert trp(0.030, 0.030) == 1.0
    assert trp(0.050, 0.030) == pytest.approx(0.6)
    with pytest.raises(ValueError):
        trp(0.0, 0.030)


gpu = pytest.mark.gpu


@gpu
def test_vbs_hand_sum_and_homogeneous():
    es = [run_entry(rq(0, 0.030)), run_entry(rq(1, 0.050)), run_entry(rq(2, 0.050))]
    assert vbs(es, 0.030) == pytest.approx(2.2)
    assert vbs([run_entry(rq(i, 0.040)) for i in range(7)], 0.040) == 7.0
    assert vbs([], 0.030) == 0.0


@gpu
def test_admit_worked_example_block_and_switch():
    st = SchedulerState()
    st.running.append(run_entry(rq(0, 0.030)))
    assert admit(st, rq(1, 0.050), 20, ITL) is True
    assert len(st.running) == 2 and st.running[-1].credit == Fraction(0)
    full = SchedulerState(running=[run_entry(rq(i, 0.030)) for i in range(30)])
    assert admit(full, rq(99, 0.030), 20, ITL) is False and len(full.running) == 30
    cost = ItlParams(alpha=0.0, beta=0.012, gamma=0.0, delta=0.0, epsilon=1.0)
    one = SchedulerState(running=[run_entry(rq(0, 0.050))])
    assert admit(one, rq(1, 0.010), 10, cost, admission_min="r_prime") is False
    assert admit(one, rq(1, 0.010), 10, cost, admission_min=R_ONLY) is True
    with pytest.raises(ValueError):
        admit(SchedulerState(), rq(0), 0, ITL)


def credit_run(slos, steps, subject=0):
    st = SchedulerState(running=[run_entry(rq(i, s, output=10_000)) for i, s in enumerate(slos)])
    hits = []
    for k in range(1, steps + 1):
        if any(e.request.id == subject for e in select_batch(st)):
            hits.append(k)
    return hits, st


@gpu
def test_credit_trajectories():
    hits, st = credit_run([0.030, 0.030], 5)
    assert hits == [1, 2, 3, 4, 5] and all(e.credit == 0 for e in st.running)
    hits, st = credit_run([5.0, 3.0], 5)  # rate 0.6 -> steps 2, 4, 5
    assert hits == [2, 4, 5] and st.running[0].credit == Fraction(0)
    assert credit_run([0.060, 0.030], 8)[0] == [2, 4, 6, 8]


@gpu
@pytest.mark.parametrize("pair", [(1.0, 10.0), (1.0, 4.0), (1.0, 2.0), (3.0, 5.0), (9.0, 10.0),
                                  (1.0, 1.0)])
@pytest.mark.parametrize("steps", [10, 100])
def test_credit_rate_convergence(pair, steps):
    anchor, subject = pair
    hits, _ = credit_run([subject, anchor], steps)
    assert abs(len(hits) / steps - anchor / subject) <= 1.0 / steps


@gpu
def test_credit_bounds_churn_and_exclusion():
    rng = np.random.default_rng(5)
    st = SchedulerState(running=[run_entry(rq(i, float(rng.choice([0.03, 0.05, 0.1])),
                                               output=10_000)) for i in range(12)])
    for k in range(60):
        select_batch(st)
        assert all(0 <= e.credit < 2 for e in st.running)
        if k % 17 == 0 and len(st.running) > 2:
            st.running.pop(int(rng.integers(len(st.running))))
    a, b = run_entry(rq(0, 0.030, output=100)), run_entry(rq(1, 0.030, output=100))
    st = SchedulerState(running=[a, b])
    assert [e.request.id for e in select_batch(st, exclude={id(b)})] == [0]
    assert b.credit == 0


@gpu
def test_scale_invariance_of_membership():
    slos = [0.030, 0.050, 0.050, 0.010, 0.120]
    for scale in (2.0, 4.0, 0.5):
        base = SchedulerState(running=[run_entry(rq(i, s, output=10_000))
                                       for i, s in enumerate(slos)])
        scaled = SchedulerState(running=[run_entry(rq(i, s * scale, output=10_000))
                                         for i, s in enumerate(slos)])
        for _ in range(20):
            assert [e.request.id for e in select_batch(base)] == \
                [e.request.id for e in select_batch(scaled)]


@gpu
def test_ttft_guard_scenarios():
    st = SchedulerState(now=0.0, waiting=[wait_item(rq(0, ttft=2.0)), wait_item(rq(1, ttft=0.5))])
    kept, rej = ttft_guard(st, PRE)
    assert [w.request.id for w in kept] == [1, 0] and rej == []
    st = SchedulerState(now=1.0, waiting=[wait_item(rq(0, ttft=0.5))])
    kept, rej = ttft_guard(st, PRE)
    assert kept == [] and [w.request.id for w in rej] == [0]
    params = PrefillParams(phi=1.0, theta=10_000, alpha_p=0.0, beta_p=0.0)
    st = SchedulerState(now=0.0, waiting=[wait_item(rq(i, ttft=t), prefill_s=1.0)
                                          for i, t in enumerate((0.9, 1.5, 2.5))])
    kept, rej = ttft_guard(st, params)
    assert [w.request.id for w in rej] == [0] and [w.request.id for w in kept] == [1, 2]


@gpu
@pytest.mark.parametrize("n", [40, 300, 5000])
def test_ttft_guard_order_and_soundness(n):
    rng = np.random.default_rng(n)
    now = 0.6
    st = SchedulerState(now=now)
    for i in range(n):
        st.waiting.append(wait_item(rq(i, ttft=float(rng.uniform(0.05, 8.0)),
                                       arrival=float(rng.uniform(0, now)),
                                       prompt=int(rng.integers(10, 500))),
                                    prefill_s=float(rng.uniform(0.0, 0.002))))
    items = sorted(st.waiting, key=lambda w: w.sort_key)
    kept, rej = ttft_guard(st, PRE)
    keys = [w.sort_key for w in kept]
    assert keys == sorted(keys)
    prefix, rej_ids, got_rej = 0.0, {w.request.id for w in rej}, []
    for it in items:  # sequential re-walk (sched_scorpio.py:196-205)
        est = (now - it.request.arrival_time) + prefix + it.prefill_s
        if est > it.request.ttft_slo:
            got_rej.append(it.request.id)
        else:
            prefix += it.prefill_s
    assert got_rej == [w.request.id for w in rej] and set(got_rej) == rej_ids


@gpu
def test_plan_step_scenarios():
    assert not plan_step(SchedulerState(), PRED, ITL, PRE).has_work()
    st = SchedulerState(waiting=[wait_item(rq(0, 0.030))])
    p = plan_step(st, PRED, ITL, PRE)
    assert [e.request.id for e in p.admitted] == [0] and p.decode_batch == []
    assert st.waiting == [] and p.vbs == 1.0
    st = SchedulerState(running=[run_entry(rq(i, 0.030, output=1000), tokens=1) for i in range(30)],
                        waiting=[wait_item(rq(99, 0.030, ttft=50.0))])
    p = plan_step(st, PRED, ITL, PRE)
    assert p.admitted == [] and [w.request.id for w in st.waiting] == [99] and not p.rejected
    cost = ItlParams(alpha=0, beta=0, gamma=0, delta=0.1, epsilon=1.0)
    st = SchedulerState(waiting=[wait_item(rq(0, tpot=0.030, ttft=100.0))])
    p = plan_step(st, PRED, cost, PRE)
    assert [(w.request.id, s) for w, s in p.rejected] == [(0, Status.REJECTED_ADMISSION)]
    st = SchedulerState(running=[run_entry(rq(0, 0.030), tokens=3)],
                        waiting=[wait_item(rq(1, 0.050))])
    (rec,) = plan_step(st, PRED, ITL, PRE).admissions
    assert rec.candidate_id == 1 and rec.running == ((0, 0.030, 103),)
    assert rec.estimate <= rec.threshold


@gpu
def test_plan_step_ablation_branches():
    st = SchedulerState(waiting=[wait_item(rq(1, ttft=0.001)), wait_item(rq(0, ttft=5.0))],
                        running=[run_entry(rq(7, 0.030, output=100), tokens=1)])
    p = plan_step(st, PRED, ITL, PRE, ScorpioConfig(ttft_guard=False, tpot_guard=False))
    assert [e.request.id for e in p.admitted] == [1, 0]
    assert [e.request.id for e in p.decode_batch] == [7] and not p.rejected
    st = SchedulerState(now=10.0, waiting=[wait_item(rq(0, ttft=0.5)), wait_item(rq(1, ttft=50.0))])
    p = plan_step(st, PRED, ITL, PRE, ScorpioConfig(ttft_guard=True, tpot_guard=False))
    assert [(w.request.id, s) for w, s in p.rejected] == [(0, Status.REJECTED_TTFT)]
    assert [e.request.id for e in p.admitted] == [1]


@gpu
def test_plan_step_batch_equals_single_states():
    rng = np.random.default_rng(11)

    def make(seed):
        r = np.random.default_rng(seed)
        st = SchedulerState(now=1.0)
        for i in range(int(r.integers(0, 40))):
            st.waiting.append(wait_item(rq(i, tpot=float(r.choice([0.03, 0.05])),
                                           ttft=float(r.choice([0.5, 2.0, 7.5])),
                                           arrival=float(r.uniform(0.6, 1.0)),
                                           prompt=int(r.integers(20, 600))),
                                        predicted=int(r.integers(5, 400)),
                                        prefill_s=float(r.uniform(0.004, 0.02))))
        for i in range(int(r.integers(0, 40))):
            st.running.append(run_entry(rq(1000 + i, tpot=float(r.choice([0.03, 0.05])),
                                           prompt=int(r.integers(20, 600)), output=500),
                                        tokens=int(r.integers(1, 100))))
        return st

    seeds = [int(x) for x in rng.integers(0, 1 << 30, 64)]
    batch = [make(s) for s in seeds]
    plans = plan_step_batch(batch, ITL, PRE)
    for s, st, p in zip(seeds, batch, plans):
        one = make(s)
        q = plan_step(one, PRED, ITL, PRE)
        assert [e.request.id for e in p.admitted] == [e.request.id for e in q.admitted]
        assert [e.request.id for e in p.decode_batch] == [e.request.id for e in q.decode_batch]
        assert [(w.request.id, x) for w, x in p.rejected] == [(w.request.id, x) for w, x in q.rejected]
        assert p.vbs == q.vbs and p.min_slo == q.min_slo
