"""Per-sim cost data for schedule-order modelling: full-sweep durations (profiling
build's globaltimer stamps, SL_LIB_PATH=libvar_prof.so) + result counts, and the
counts of pilot sweeps over truncated traces (first m requests)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200 import _native as N  # noqa: E402
from paper_2505_23022_b200.batch import BatchEngine, Cell, TraceArrays  # noqa: E402
from paper_2505_23022_b200.sweep import SweepGrid, build_local  # noqa: E402

grid = SweepGrid()
dev = torch.device("cuda", 0)
eng, owned, traces = build_local(grid, device=dev)
eng.launch()
torch.cuda.synchronize()
res = eng.results()
lib = N.lib()
out = np.zeros((eng.n_sims, 16), np.uint64)
lib.sl_phase_prof_read.argtypes = [C.c_void_p, C.c_int32]
lib.sl_phase_prof_read(out.ctypes.data, eng.n_sims)
save = {"t0": out[:, 14], "t1": out[:, 15], "n_steps": res["n_steps"], "req": res["request_steps"],
        "plans": res["n_plans"], "phase": out[:, :14]}
tr = traces
cells = [Cell(int(c) // len(grid.scales), grid.config, slo_scale=float(grid.scales[int(c) % len(grid.scales)]))
         for c in owned]
for m in (100, 250, 500, 1000):
    cut = [TraceArrays(*[getattr(t, f)[:m] for f in ("arrival", "ttft_slo", "tpot_slo", "prompt_len",
                                                        "true_out", "predicted", "id", "category")])
           for t in tr]
    e2 = BatchEngine(cut, cells, device=dev)
    e2.launch()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        e2.launch()
    torch.cuda.synchronize()
    r2 = e2.results()
    save[f"p{m}_steps"] = r2["n_steps"]
    save[f"p{m}_req"] = r2["request_steps"]
    save[f"p{m}_plans"] = r2["n_plans"]
    p2 = np.zeros((eng.n_sims, 16), np.uint64)
    lib.sl_phase_prof_read(p2.ctypes.data, eng.n_sims)
    save[f"p{m}_dur"] = p2[:, 15] - p2[:, 14]
    print(m, "pilot ms", (time.perf_counter() - t) / 3 * 1e3)
np.savez("gpurun_out/cost_data.npz", **save)
