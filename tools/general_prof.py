import sys
from dataclasses import replace
import torch
sys.path.insert(0, '/root/repo')
from paper_2505_23022_b200 import _native as N
from paper_2505_23022_b200.batch import BatchEngine, Cell
from paper_2505_23022_b200.sweep import SweepGrid
import numpy as np
g = SweepGrid(rates=tuple(np.linspace(2.0, 32.0, 16)), scales=tuple(np.geomspace(0.5, 2.0, 16)))
tr = [g.trace_for_rate(q) for q in g.rates]
cfg = replace(g.config, policy="greedy")
cells = [Cell(ri, cfg, slo_scale=float(sc)) for ri in range(len(g.rates)) for sc in g.scales]
eng = BatchEngine(tr, cells, device="cuda:0", mode=N.MODE_GENERAL)
eng.launch(); torch.cuda.synchronize()
