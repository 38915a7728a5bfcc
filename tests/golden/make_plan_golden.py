"""Reference plan_step outputs on seeded config-2 snapshots (run in the build
container, where /root/reference exists).  Inputs are regenerated from seeds by
paper_2505_23022_b200.snapshot on the GPU box; only outputs are stored.

    python tests/golden/make_plan_golden.py
"""

from __future__ import annotations

import json
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CASES = [  # (name, segments, W, R, seed, flags)
    ("primary_32x32", 64, 32, 32, 1, "both"),
    ("small_mixed", 96, 7, 5, 2, "both"),
    ("mid_300x60", 8, 300, 60, 3, "both"),
    ("r_only", 32, 32, 32, 4, "r_only"),
    ("ttft_only", 32, 32, 32, 5, "ttft_only"),
    ("tpot_only", 32, 32, 32, 6, "tpot_only"),
    ("neither", 16, 32, 32, 7, "neither"),
    ("tile_merge_5000", 1, 5000, 300, 8, "both"),
    ("stress_32768", 1, 32768, 32768, 9, "both"),
    # the shapes bench.py times (config 2): the primary batch exactly ...
    ("bench_primary_1024", 1024, 32, 32, 11, "both"),
    # few large segments (the one-CTA-per-segment kernels): multi-tile walks with
    # admissions, the guard ablations, and admissions that lower the running
    # minimum (R = 3: vbs refolded with the new minimum)
    ("large_adm_3000x40", 4, 3000, 40, 12, "both"),
    ("large_r_only", 2, 2500, 2000, 13, "r_only"),
    ("large_tpot_only", 2, 3000, 3000, 14, "tpot_only"),
    ("large_ttft_only", 2, 3000, 3000, 15, "ttft_only"),
    ("large_neither", 1, 2000, 5000, 16, "neither"),
    ("large_min_drop", 8, 2000, 3, 17, "both"),
    # ragged batch: empty, short, exactly-32 and over-32 queues and running sets
    # side by side (the group kernel's staged and unstaged segments in one warp)
    ("ragged_mixed", 48, [0, 1, 5, 31, 32, 33, 40, 64, 17, 2, 32, 0] * 4,
     [3, 0, 32, 33, 16, 1, 64, 0, 8, 40, 2, 31] * 4, 20, "both"),
    ("ragged_long", 24, [0, 300, 33, 7, 250, 32] * 4, [60, 0, 5, 64, 32, 1] * 4, 21, "both"),
]
# deadline ties (arrivals on a 2^-4 s grid, ids reversed): the LDF sort's
# tie-breaks on every route -- warp network (<= 32), one cluster per segment
TIES = [("ties_small", 16, 32, 8, 18, "both", 0.0625),
        ("ties_large", 2, 5000, 50, 19, "both", 0.0625)]
# negative prefill times (alpha_p < 0 is legal: PrefillParams checks only the
# value at theta, costmodel.py:45-47): prompts past -beta_p/alpha_p get negative
# prefills, so the walk's prefix can shrink -- the kernels drop their
# prefix-monotone shortcuts (PLAN_EXACT_WALK) on every route
NEG_PREFILL = (0.004, 128.0, -1e-5, 4.5e-3)
NEG = [("neg_prefill_small", 32, 40, 16, 22, "both"),
       ("neg_prefill_large", 2, 3000, 50, 23, "both")]
# ... and 256 segments spread over the bench's 262,144-segment scaled batch
# (config2_plan_arrays_fast, seed 11): the test runs the whole batch through the
# same kernels the bench times and compares the sampled segments
SAMPLED = [("bench_scaled_262144", 262144, 32, 32, 11, "both", 256)]


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, ROOT)
    from slosim import core, schedtypes
    from slosim.costmodel import ItlParams, PrefillParams
    from slosim.predictor import Bucketing, LengthPredictor
    from slosim.sched_scorpio import ScorpioConfig, plan_step

    from paper_2505_23022_b200.snapshot import (config2_arrays, config2_plan_arrays_fast,
                                                 states_from_arrays, states_from_plan_arrays)

    T = types.SimpleNamespace(Request=core.Request, WaitingItem=schedtypes.WaitingItem,
                              RunningEntry=schedtypes.RunningEntry,
                              SchedulerState=schedtypes.SchedulerState)
    itl = ItlParams(1e-6, 1e-3, 1e-5, 5e-3, 1.1)
    pre = PrefillParams(0.004, 128.0, 2e-5, 1.5e-3)
    pred = LengthPredictor(mode="oracle", bucketing=Bucketing.equal_width(100, 4096))
    cfgs = {"both": ScorpioConfig(), "r_only": ScorpioConfig(admission_min="r_only"),
            "ttft_only": ScorpioConfig(tpot_guard=False), "tpot_only": ScorpioConfig(ttft_guard=False),
            "neither": ScorpioConfig(False, False)}
    blobs, meta = {}, []
    jobs = ([(name, S, W, R, seed, fl, None, None, None) for name, S, W, R, seed, fl in CASES]
            + [(name, S, W, R, seed, fl, None, tg, None) for name, S, W, R, seed, fl, tg in TIES]
            + [j + (None, None) for j in SAMPLED]
            + [(name, S, W, R, seed, fl, None, None, NEG_PREFILL)
               for name, S, W, R, seed, fl in NEG])
    for name, S, W, R, seed, fl, n_sample, tg, pf in jobs:
        pre_c = PrefillParams(*pf) if pf else pre
        if n_sample is None:
            a = config2_arrays(S, W, R, seed, tie_grid=tg, **({"prefill": pf} if pf else {}))
            states = states_from_arrays(a, T)
            segs = None
        else:
            a = config2_plan_arrays_fast(S, W, R, seed)
            segs = [int(x) for x in np.linspace(0, S - 1, n_sample).round()]
            states = states_from_plan_arrays(a, T, segs)
        adm, rej, bat, wait, vbs, mins, cred = [], [], [], [], [], [], []
        for st in states:
            p = plan_step(st, pred, itl, pre_c, cfgs[fl])
            adm.append([e.request.id for e in p.admitted])
            rej.append([w.request.id * 2 + (s.value == "rejected_admission") for w, s in p.rejected])
            bat.append([e.request.id for e in p.decode_batch])
            wait.append([w.request.id for w in st.waiting])
            vbs.append(p.vbs)
            mins.append(float("nan") if p.min_slo is None else p.min_slo)
            E = int(a["credit_exp"][0])
            from fractions import Fraction
            for e in st.running[: len(st.running) - len(p.admitted)]:
                n = e.credit * Fraction(e.request.tpot_slo) / Fraction(2) ** E
                assert n.denominator == 1
                cred.append(int(n))
        k = f"{name}_"
        for key, lists in (("adm", adm), ("rej", rej), ("bat", bat), ("wait", wait)):
            blobs[k + key] = np.array([x for l in lists for x in l], np.int64)
            blobs[k + key + "_n"] = np.array([len(l) for l in lists], np.int64)
        blobs[k + "vbs"] = np.array(vbs)
        blobs[k + "min_slo"] = np.array(mins)
        blobs[k + "credit"] = np.array(cred, np.uint64)
        meta.append(dict(name=name, segments=S, w=W, r=R, seed=seed, flags=fl, sample=segs,
                         tie_grid=tg, **({"prefill": list(pf)} if pf else {})))
        print(name, "admitted", sum(map(len, adm)), "rejected", sum(map(len, rej)),
              "batch", sum(map(len, bat)))
    np.savez_compressed(os.path.join(HERE, "plan.npz"), **blobs)
    json.dump(meta, open(os.path.join(HERE, "plan.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
