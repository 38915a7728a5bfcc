"""Generate golden fixtures by running the REAL reference (slosim) in the build container.

Run here (not on the GPU box, where /root/reference does not exist):

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Writes ``tests/golden/sims.npz`` (traces + reference outcomes/step logs/digests per
case), ``tests/golden/predictor_kat.npz`` (numpy default_rng noisy-bucket
predictions), ``tests/golden/seed_kat.json`` and ``tests/golden/workload_kat.npz``.
Everything here reads the reference through its public API only; the digest is
restated in pure Python from ``EventLog.steps`` (definition: DESIGN.md "digest").
"""

from __future__ import annotations

import argparse
import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
M64 = (1 << 64) - 1


def digest_item(step: int, tag: int, pos: int, val: int) -> int:
    """Work-step digest item: mix(val ^ (step*K_STEP + tag*K_TAG + pos*K_POS))."""
    key = (step * 0x9E3779B97F4A7C15 + tag * 0xC2B2AE3D27D4EB4F + pos * 0x165667B19E3779F9) & M64
    y = (((val & M64) ^ key) * 0xD6E8FEB86659FD93) & M64
    return y ^ (y >> 32)


def dbits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def log_digest(log) -> int:
    h = 0
    for s_idx, rec in enumerate(log.steps):
        assert rec.step == s_idx
        for pos, rid in enumerate(rec.admitted):
            h += digest_item(s_idx, 0, pos, rid)
        for pos, (rid, reason) in enumerate(rec.rejected):
            h += digest_item(s_idx, 1, pos, rid * 2 + (reason == "rejected_admission"))
        bh = 0  # the batch: one item over sum(batch_hid) mod 2^32
        for rid in rec.batch:
            y = ((rid & M64) * 0xD6E8FEB86659FD93) & M64
            bh += (y ^ (y >> 32)) & 0xFFFFFFFF
        h += digest_item(s_idx, 2, len(rec.batch), bh & 0xFFFFFFFF)
        h += digest_item(s_idx, 3, 0, dbits(rec.end_s))
    return h & M64


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.dont_write_bytecode = True
    import logging
    logging.disable(logging.WARNING)
    sys.path.insert(0, args.ref)
    from slosim.core import Request, SloCategory, SloCategoryTable, relaxed_slo_table
    from slosim.costmodel import ItlParams, PrefillParams
    from slosim.predictor import Bucketing, LengthPredictor
    from slosim.sched_baselines import BaselineConfig
    from slosim.sched_scorpio import ScorpioConfig
    from slosim.seeds import derive_seed
    from slosim.report import report_horizon, summarize
    from slosim.simengine import SimConfig, run
    from slosim.workload import LogNormalDist, UniformDist, WorkloadSpec, generate, rescale_arrivals

    acc_itl = ItlParams(1e-6, 1e-3, 1e-5, 5e-3, 1.1)
    acc_pre = PrefillParams(0.004, 128.0, 2e-5, 1.5e-3)
    ex_itl = ItlParams(1e-6, 1e-3, 1e-5, 5e-3, 1.0)
    ex_pre = PrefillParams(0.020, 128.0, 1e-4, 7e-3)
    three_tier = SloCategoryTable(rows=(SloCategory(1, 0.5, 0.030), SloCategory(2, 2.0, 0.050),
                                        SloCategory(3, 7.5, 0.100)))
    oracle_pred = LengthPredictor(mode="oracle", bucketing=Bucketing.equal_width(100, 4096))

    def spec(qps, duration, seed, p=(5.0, 0.7), o=(4.0, 0.7), table=None, ncat=6, uni=None):
        pd = LogNormalDist(*p) if uni is None else UniformDist(*uni[0])
        od = LogNormalDist(*o) if uni is None else UniformDist(*uni[1])
        return WorkloadSpec(qps=qps, duration=duration, seed=seed, prompt_len_dist=pd,
                            output_len_dist=od, category_weights=(1.0,) * ncat, slo_table=table)

    def scaled(trace, s):
        return [Request(id=r.id, arrival_time=r.arrival_time, prompt_len=r.prompt_len,
                        true_output_len=r.true_output_len, ttft_slo=r.ttft_slo * s,
                        tpot_slo=r.tpot_slo * s, category=r.category) for r in trace]

    cases = []

    def add(name, trace, policy="scorpio", itl=acc_itl, pre=acc_pre, pred=oracle_pred,
            scorpio=ScorpioConfig(), cap=256, horizon=None, keep_log=True, prefill_priority=False):
        cases.append(dict(name=name, trace=trace, policy=policy, itl=itl, pre=pre, pred=pred,
                          scorpio=scorpio, cap=cap, horizon=horizon, keep_log=keep_log,
                          prefill_priority=prefill_priority))

    # config 1: 1,000 requests, 8 req/s, 3 tiers
    c1 = generate(spec(8.0, 150.0, 7, table=three_tier, ncat=3))[:1000]
    add("config1", c1, keep_log=False)
    # pinned overload of the acceptance suite (test_acceptance.py:40-59)
    ov = generate(spec(25.0, 90.0, 20240601))[:2000]
    add("overload_scorpio", ov, keep_log=False)
    add("overload_greedy", ov, policy="greedy", keep_log=False)
    for nm, cfg in (("neither", ScorpioConfig(False, False)), ("ttft_only", ScorpioConfig(True, False)),
                    ("tpot_only", ScorpioConfig(False, True))):
        add(f"overload_{nm}", ov[:800], scorpio=cfg, keep_log=False)
    add("overload_r_only", ov[:800], scorpio=ScorpioConfig(admission_min="r_only"), keep_log=False)
    # SLO-scale and rate axes
    mid = generate(spec(12.0, 80.0, 11))[:600]
    for s in (0.5, float(np.geomspace(0.5, 2.0, 64)[23]), 2.0):
        add(f"slo_scale_{s:.6f}", scaled(mid, s))
    span = mid[-1].arrival_time
    native = len(mid) / span
    for q in (4.0, 20.0, 32.0):
        add(f"rate_{q:g}", rescale_arrivals(mid, q / native))
    # noisy predictor in the loop (config 4 style)
    noisy = LengthPredictor(mode="noisy_bucket", bucketing=Bucketing.equal_width(100, 4096),
                            error_prob=0.73, error_spread=3, rng_seed=derive_seed(5, "predictor"))
    sg = generate(spec(14.0, 60.0, 3, p=(4.6, 0.9), o=(4.5, 0.9)))[:700]
    add("sharegpt_noisy", sg, pred=noisy)
    add("sharegpt_oracle", sg)
    # horizon, baselines, example cost params, relaxed table
    add("horizon", mid, horizon=20.0)
    add("sjf", mid[:300], policy="sjf", cap=8)
    add("early_reject", mid[:300], policy="early_reject", cap=8)
    add("greedy_pp", mid[:300], policy="greedy", cap=8, prefill_priority=True)
    add("example_params", generate(spec(6.0, 30.0, 2, uni=((10, 300), (1, 40)))), itl=ex_itl,
        pre=ex_pre)
    add("relaxed_table", generate(spec(10.0, 30.0, 4, table=relaxed_slo_table())))
    # ties: identical arrivals and deadlines exercise the (deadline, arrival, id) order
    tie = []
    rng = np.random.default_rng(17)
    t = 0.0
    for i in range(400):
        if i % 3 == 0:
            t += float(rng.exponential(0.05))
        tie.append(Request(id=int(1000 - i) if i % 7 == 0 else i + 5000, arrival_time=t,
                           prompt_len=int(rng.integers(1, 600)),
                           true_output_len=int(rng.integers(1, 60)),
                           ttft_slo=[0.5, 1.0, 0.25][i % 3], tpot_slo=[0.03, 0.05, 0.02][i % 3]))
    add("ties", tie)
    # c04 six-request scenario (test_acceptance.py:170-222)
    six_itl = ItlParams(0.0, 0.25, 0.0, 0.0, 1.0)
    six_pre = PrefillParams(1.0, 10**6, 0.0, 0.0)
    six = [Request(id=i, arrival_time=0.0, prompt_len=1, true_output_len=5, ttft_slo=tt,
                   tpot_slo=tp) for i, (tp, tt) in enumerate(
        [(1.0, 10.0), (1.0, 10.0), (2.0, 10.0), (1.0, 10.0), (2.0, 10.0), (0.2, 3.0)])]
    add("c04_six_scorpio", six, itl=six_itl, pre=six_pre)
    add("c04_six_greedy", six, policy="greedy", itl=six_itl, pre=six_pre)
    # golden single request (test_simengine.py:48-63)
    add("single", [Request(id=0, arrival_time=0.0, prompt_len=100, true_output_len=3,
                           ttft_slo=0.5, tpot_slo=0.030, category=1)], itl=ex_itl, pre=ex_pre)
    add("empty", [], itl=ex_itl, pre=ex_pre)
    # round 2: cost models the reference accepts but the fast kernel's monotone
    # shortcuts do not cover -- negative ITL coefficients (fit_itl's lstsq may
    # return them, costmodel.py:205; only epsilon is validated, :45-47) and a
    # negative prefill slope (legal while alpha_p*theta + beta_p >= 0, :59-65;
    # prompts past 500 tokens then get a negative prefill_time)
    add("neg_gamma", ov[:900], itl=ItlParams(1e-6, 1e-3, -2e-6, 5e-3, 1.1))
    add("neg_alpha", ov[:900], itl=ItlParams(-2e-8, 1e-3, 1e-5, 5e-3, 1.1))
    add("neg_alpha_p", ov[:900], pre=PrefillParams(0.004, 128.0, -2e-6, 1e-3))
    add("neg_alpha_p_early_reject", mid[:300], policy="early_reject", cap=8,
        pre=PrefillParams(0.004, 128.0, -2e-6, 1e-3))
    # dyadic everything: arrivals on a 1/64 s grid, power-of-two SLOs and cost
    # coefficients, so walk and admission tests land exactly on their thresholds
    dy_itl = ItlParams(2.0**-20, 2.0**-10, 2.0**-17, 2.0**-8, 1.0)
    dy_pre = PrefillParams(2.0**-8, 128.0, 2.0**-16, 2.0**-9)
    dy = []
    rng = np.random.default_rng(23)
    t = 0.0
    for i in range(500):
        t += float(rng.integers(0, 5)) / 64.0
        dy.append(Request(id=i, arrival_time=t, prompt_len=int(rng.integers(1, 5)) * 64,
                          true_output_len=int(rng.integers(1, 40)),
                          ttft_slo=[0.25, 0.5, 1.0][i % 3], tpot_slo=[2.0**-5, 2.0**-4][i % 2],
                          category=i % 3))
    add("dyadic_ties", dy, itl=dy_itl, pre=dy_pre)
    add("dyadic_ties_r_only", dy, itl=dy_itl, pre=dy_pre,
        scorpio=ScorpioConfig(admission_min="r_only"))

    blobs = {}
    meta = []
    reports = {}
    jsonl = {}
    for ci, c in enumerate(cases):
        tr = c["trace"]
        cfg = SimConfig(policy=c["policy"], itl_params=c["itl"], prefill_params=c["pre"],
                        predictor=c["pred"], scorpio=c["scorpio"],
                        baseline=BaselineConfig(max_batch_size=c["cap"],
                                                prefill_priority=c["prefill_priority"]),
                        horizon=c["horizon"])
        outcomes, log = run(tr, cfg)
        ends = {s.end_s: s.step for s in log.steps}
        p = f"c{ci}_"
        blobs[p + "arrival"] = np.array([r.arrival_time for r in tr], np.float64)
        blobs[p + "ttft_slo"] = np.array([r.ttft_slo for r in tr], np.float64)
        blobs[p + "tpot_slo"] = np.array([r.tpot_slo for r in tr], np.float64)
        blobs[p + "prompt_len"] = np.array([r.prompt_len for r in tr], np.int32)
        blobs[p + "true_out"] = np.array([r.true_output_len for r in tr], np.int32)
        blobs[p + "id"] = np.array([r.id for r in tr], np.int64)
        blobs[p + "category"] = np.array([r.category for r in tr], np.int32)
        blobs[p + "predicted"] = np.array([c["pred"].predict(r) for r in tr], np.int32)
        st = {"completed": 0, "rejected_ttft": 1, "rejected_admission": 2, "incomplete": 3}
        blobs[p + "status"] = np.array([st[o.status.value] for o in outcomes], np.int8)
        blobs[p + "compliant"] = np.array([o.slo_compliant for o in outcomes], np.int8)
        nan = float("nan")
        for f in ("first_token_time", "completion_time", "ttft", "tpot"):
            blobs[p + f] = np.array([nan if getattr(o, f) is None else getattr(o, f)
                                     for o in outcomes], np.float64)
        blobs[p + "completion_step"] = np.array(
            [ends[o.completion_time] if o.completion_time is not None else -1 for o in outcomes],
            np.int32)
        if c["keep_log"]:
            S = log.steps
            blobs[p + "log_now"] = np.array([s.now_s for s in S], np.float64)
            blobs[p + "log_end"] = np.array([s.end_s for s in S], np.float64)
            blobs[p + "log_prefill_s"] = np.array([s.prefill_s for s in S], np.float64)
            blobs[p + "log_decode_s"] = np.array([s.decode_s for s in S], np.float64)
            blobs[p + "log_vbs"] = np.array([s.vbs for s in S], np.float64)
            blobs[p + "log_min_slo"] = np.array(
                [nan if s.min_slo_s is None else s.min_slo_s for s in S], np.float64)
            blobs[p + "log_counts"] = np.array(
                [[len(s.admitted), len(s.rejected), len(s.batch)] for s in S], np.int32).reshape(-1, 3)
            ids = []
            for s in S:
                ids += list(s.admitted)
                ids += [rid * 2 + (rs == "rejected_admission") for rid, rs in s.rejected]
                ids += list(s.batch)
            blobs[p + "log_ids"] = np.array(ids, np.int64)
        compliant = sum(o.slo_compliant for o in outcomes)
        horizon = c["horizon"] if c["horizon"] is not None else max(log.sim_end_s, 1e-12)
        pd = c["pred"]
        meta.append(dict(
            name=c["name"], policy=c["policy"], n=len(tr),
            itl=[c["itl"].alpha, c["itl"].beta, c["itl"].gamma, c["itl"].delta, c["itl"].epsilon],
            prefill=[c["pre"].phi, c["pre"].theta, c["pre"].alpha_p, c["pre"].beta_p],
            ttft_guard=c["scorpio"].ttft_guard, tpot_guard=c["scorpio"].tpot_guard,
            admission_min=c["scorpio"].admission_min, max_batch_size=c["cap"],
            prefill_priority=c["prefill_priority"], horizon=c["horizon"],
            predictor=dict(mode=pd.mode, num_buckets=pd.bucketing.num_buckets,
                           max_len=pd.bucketing.max_len, error_prob=pd.error_prob,
                           error_spread=pd.error_spread, rng_seed=str(pd.rng_seed)),
            n_steps=len(log.steps), n_idle_skips=len(log.idle_skips), sim_end=log.sim_end_s,
            digest=str(log_digest(log)), compliant=int(compliant), goodput=compliant / horizon,
            adherence=(compliant / len(outcomes)) if outcomes else 0.0, keep_log=c["keep_log"]))
        # the reference's own RunReport and decision-log bytes (report.py:71-134,
        # simengine.py:106-137) for the device report / log parity tests
        reports[c["name"]] = summarize(outcomes, report_horizon(cfg.horizon, log)).to_dict()
        if c["keep_log"] and len(tr) <= 1000:
            jp = os.path.join(HERE, "_tmp.jsonl")
            log.to_jsonl(jp)
            with open(jp, "rb") as f:
                jsonl[c["name"]] = np.frombuffer(f.read(), np.uint8)
            os.remove(jp)
        print(f"{c['name']:>24}: n={len(tr)} steps={len(log.steps)} compliant={compliant}")
    np.savez_compressed(os.path.join(HERE, "sims.npz"), **blobs)
    with open(os.path.join(HERE, "sims.json"), "w") as f:
        json.dump(meta, f, indent=1)
    with open(os.path.join(HERE, "reports.json"), "w") as f:
        json.dump(reports, f)
    np.savez_compressed(os.path.join(HERE, "decisions_jsonl.npz"), **jsonl)

    # ---- predictor KATs: numpy default_rng([seed, id]) stream (predictor.py:115-126)
    kat = {"seed": [], "id": [], "true_out": [], "num_buckets": [], "max_len": [],
           "error_prob": [], "spread": [], "pred": []}
    rng = np.random.default_rng(99)
    configs = [(100, 4096, 0.73, 3), (10, 1000, 1.0, 1), (4, 100, 1.0, 10), (25, 1500, 0.6, 3),
               (100, 4096, 0.5, 2), (7, 50, 0.9, 4), (1, 1, 1.0, 5)]
    for nb, ml, ep, sp in configs:
        for seed in (0, 5, 17, derive_seed(5, "predictor"), derive_seed(123, "predictor"), 2**63 + 7):
            pred = LengthPredictor(mode="noisy_bucket", bucketing=Bucketing.equal_width(nb, ml),
                                   error_prob=ep, error_spread=sp, rng_seed=seed)
            ids = list(range(0, 300)) + [int(x) for x in rng.integers(0, 2**40, 100)] + [2**32 - 1, 2**32, 2**33 + 5]
            for rid in ids:
                tout = int(rng.integers(1, ml * 2 + 2))
                r = Request(id=rid, arrival_time=0.0, prompt_len=1, true_output_len=tout,
                            ttft_slo=1.0, tpot_slo=1.0)
                kat["seed"].append(seed)
                kat["id"].append(rid)
                kat["true_out"].append(tout)
                kat["num_buckets"].append(nb)
                kat["max_len"].append(ml)
                kat["error_prob"].append(ep)
                kat["spread"].append(sp)
                kat["pred"].append(pred.predict(r))
    np.savez_compressed(os.path.join(HERE, "predictor_kat.npz"),
                        seed=np.array(kat["seed"], np.uint64), id=np.array(kat["id"], np.int64),
                        true_out=np.array(kat["true_out"], np.int32),
                        num_buckets=np.array(kat["num_buckets"], np.int32),
                        max_len=np.array(kat["max_len"], np.int32),
                        error_prob=np.array(kat["error_prob"]), spread=np.array(kat["spread"], np.int32),
                        pred=np.array(kat["pred"], np.int32))
    print("predictor KATs:", len(kat["pred"]))

    # ---- derive_seed KATs (seeds.py:14-17)
    seeds = [[b, parts, str(derive_seed(b, *parts))] for b, parts in (
        (0, ["predictor"]), (5, ["predictor"]), (1, ["trace", 4.0]), (1, ["trace", 12.5]),
        (77, ["admission-audit", 3]), (20240601, ["trace", 25.0]), (-3, ["x", "y", 1]))]
    with open(os.path.join(HERE, "seed_kat.json"), "w") as f:
        json.dump(seeds, f)

    # ---- workload.generate KATs (workload.py:107-137)
    wl = {}
    for k, sp in enumerate((spec(8.0, 40.0, 7, table=three_tier, ncat=3), spec(25.0, 10.0, 20240601),
                            spec(5.0, 20.0, 2, uni=((10, 300), (1, 40))),
                            spec(14.0, 10.0, 3, p=(4.6, 0.9), o=(4.5, 0.9)))):
        tr = generate(sp)
        wl[f"w{k}_arrival"] = np.array([r.arrival_time for r in tr])
        wl[f"w{k}_prompt_len"] = np.array([r.prompt_len for r in tr], np.int32)
        wl[f"w{k}_true_out"] = np.array([r.true_output_len for r in tr], np.int32)
        wl[f"w{k}_category"] = np.array([r.category for r in tr], np.int32)
        wl[f"w{k}_ttft_slo"] = np.array([r.ttft_slo for r in tr])
        wl[f"w{k}_tpot_slo"] = np.array([r.tpot_slo for r in tr])
    np.savez_compressed(os.path.join(HERE, "workload_kat.npz"), **wl)
    print("done")


if __name__ == "__main__":
    main()
