"""Baseline-policy sweeps: fast-kernel vs general-kernel time and handoff counts."""
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2505_23022_b200 import _native as N  # noqa: E402
from paper_2505_23022_b200.batch import BatchEngine, Cell  # noqa: E402
from paper_2505_23022_b200.sweep import SweepGrid  # noqa: E402

g = SweepGrid()
tr = [g.trace_for_rate(q) for q in g.rates]
for pol in ("greedy", "early_reject"):
    cfg = replace(g.config, policy=pol)
    cells = [Cell(ri, cfg, slo_scale=float(sc)) for ri in range(len(g.rates)) for sc in g.scales]
    for mode in (N.MODE_AUTO, N.MODE_GENERAL):
        eng = BatchEngine(tr, cells, device="cuda:0", mode=mode)
        eng.launch()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.launch()
        b.record()
        torch.cuda.synchronize()
        r = eng.results()
        print(pol, "mode", mode, "ms %.1f" % a.elapsed_time(b))
    # running-set peak per sim from a log-free proxy: cells whose max running exceeded 64
