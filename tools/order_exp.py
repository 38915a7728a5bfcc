"""Sweep time under different schedule orders (work-queue order of sl_run_batch)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200.sweep import SweepGrid, build_local  # noqa: E402

grid = SweepGrid()
eng, owned, traces = build_local(grid, device=torch.device("cuda", 0))
z = np.load(sys.argv[1]) if len(sys.argv) > 1 else None
orders = {"current": eng._order.cpu().numpy().copy()}
if z is not None:
    d = (z["t1"].astype(np.int64) - z["t0"].astype(np.int64)).astype(float)
    orders["lpt_measured"] = np.argsort(-d, kind="stable")
    X = np.stack([z["n_steps"], z["req"], z["plans"]], 1).astype(float)
    c, *_ = np.linalg.lstsq(X, d, rcond=None)
    orders["lpt_countfit"] = np.argsort(-(X @ c), kind="stable")
    for k in list(z.keys()):
        if k.startswith("order_"):
            orders[k] = z[k]
if len(sys.argv) > 2:
    z2 = np.load(sys.argv[2])
    for k in z2.keys():
        orders[k] = z2[k]
rng = np.random.default_rng(0)
orders["random"] = rng.permutation(eng.n_sims)
orders["rate_desc"] = orders["current"][::-1].copy()
res0 = None
for name, o in orders.items():
    eng._order.copy_(torch.from_numpy(np.ascontiguousarray(o, np.int32)))
    eng.launch()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.launch()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    r = eng.results()
    if res0 is None:
        res0 = r["digest"].copy()
    assert np.array_equal(r["digest"], res0)
    print(f"{name:16s} {np.median(ts):7.2f} ms  {[round(t, 1) for t in ts]}")
