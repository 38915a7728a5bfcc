import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from dataclasses import replace
from paper_2505_23022_b200.batch import BatchEngine, Cell
from paper_2505_23022_b200.sweep import SweepGrid
g = SweepGrid()
tr = [g.trace_for_rate(q) for q in g.rates]
for pol in ("scorpio", "greedy", "sjf", "early_reject"):
    cfg = replace(g.config, policy=pol)
    cells = [Cell(ri, cfg, slo_scale=float(sc)) for ri in range(len(g.rates)) for sc in g.scales]
    eng = BatchEngine(tr, cells, device="cuda:0")
    eng.launch(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); eng.launch(); b.record(); torch.cuda.synchronize()
    r = eng.results()
    print(pol, "ms %.1f" % a.elapsed_time(b), "req-steps %.3e" % r["request_steps"].sum(), "goodput %.3f" % r["goodput"].mean(), "status", np.unique(r["status"] & 0xff, return_counts=True))
