"""Where the e2e step's time goes beyond the sweep kernel (config 3, one GPU):
cell packing, BatchEngine construction (uploads, allocations), launch to
completion, result read-back -- wall clock per part, mean of 5 after 3 warm-up."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_23022_b200.batch import BatchEngine, CellColumns, TraceTable, pack_cells  # noqa: E402
from paper_2505_23022_b200.sweep import build_local  # noqa: E402

import types
args = types.SimpleNamespace(rates=64, scales=64, n_requests=10_000)
dev = torch.device("cuda", 0)
grid = bench.make_grid(args, 1)
eng, owned, traces = build_local(grid, 0, 1, device=dev)
del eng
table = TraceTable(traces)
cl = bench.build_cells(grid, owned, traces)
cells = CellColumns(np.array([c.trace for c in cl], np.int64), np.array([c.slo_scale for c in cl]),
                    grid.config)
l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
parts = {k: [] for k in ("pack", "engine", "launch", "results", "total")}
for it in range(8):
    l2.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pack_cells(table, cells)
    t1 = time.perf_counter()
    e = BatchEngine(table, cells, device=dev)
    t2 = time.perf_counter()
    e.launch(torch.cuda.current_stream(dev))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    e.results()
    t4 = time.perf_counter()
    if it >= 3:
        for k, v in zip(parts, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t1)):
            parts[k].append(v * 1e3)
    del e
print({k: round(float(np.mean(v)), 3) for k, v in parts.items()}, "ms (engine includes its own pack)")
