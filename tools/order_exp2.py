"""Sweep time without the lowest-rate row(s) (critical-path floor experiment)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200.sweep import SweepGrid, build_local  # noqa: E402

z = np.load("scratch/cost_data.npz")
d = (z["t1"].astype(np.int64) - z["t0"].astype(np.int64)).astype(float)
full = np.linspace(2.0, 32.0, 64)
for drop in (0, 1, 2, 4):
    grid = SweepGrid(rates=tuple(full[drop:]))
    eng, owned, _ = build_local(grid, device=torch.device("cuda", 0))
    dd = d[drop * 64:]
    for name, o in (("current", eng._order.cpu().numpy().copy()), ("lpt", np.argsort(-dd, kind="stable"))):
        eng._order.copy_(torch.from_numpy(np.ascontiguousarray(o, np.int32)))
        eng.launch()
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            eng.launch()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"drop {drop} sims {eng.n_sims} {name:8s} {np.median(ts):7.2f} ms  work-share {dd.sum() / d.sum():.3f}")
