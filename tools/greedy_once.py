"""One config-3 sweep under the greedy policy (for launch-list profiling)."""
import sys
from dataclasses import replace

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2505_23022_b200.batch import BatchEngine, Cell  # noqa: E402
from paper_2505_23022_b200.sweep import SweepGrid  # noqa: E402

g = SweepGrid()
tr = [g.trace_for_rate(q) for q in g.rates]
cfg = replace(g.config, policy=sys.argv[1] if len(sys.argv) > 1 else "greedy")
cells = [Cell(ri, cfg, slo_scale=float(sc)) for ri in range(len(g.rates)) for sc in g.scales]
eng = BatchEngine(tr, cells, device="cuda:0")
eng.launch()
torch.cuda.synchronize()
r = eng.results()
print("handed off (general kernel):", int(((r["status"] & 0) == 0).sum()))
