"""Per-sim start / end times of the config-3 sweep (timeline build:
tools/build_variant.sh tl -DSL_TIMELINE; SL_LIB_PATH=.../libvar_tl.so) -> slot
occupancy over time, and what a perfect packing of the same per-sim durations
onto the warp slots would give."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200 import _native as N  # noqa: E402
from paper_2505_23022_b200.sweep import SweepGrid, build_local  # noqa: E402

grid = SweepGrid()
eng, owned, _ = build_local(grid, device=torch.device("cuda", 0))
for _ in range(2):
    eng.launch()
torch.cuda.synchronize()
lib = N.lib()
lib.sl_phase_prof_read.argtypes = [C.c_void_p, C.c_int32]
out = np.zeros((eng.n_sims, 26), np.uint64)
assert lib.sl_phase_prof_read(out.ctypes.data, eng.n_sims) == eng.n_sims
t0, t1 = out[:, 14].astype(np.int64), out[:, 15].astype(np.int64)
base = t0.min()
t0, t1 = (t0 - base) / 1e6, (t1 - base) / 1e6
span = t1.max()
dur = t1 - t0
slots = 148 * 16
print("makespan %.1f ms; busy / (slots x makespan) = %.3f; sum of durations / slots = %.1f ms"
      % (span, dur.sum() / (slots * span), dur.sum() / slots))
for q in np.linspace(0, span, 11)[1:]:
    print("  t=%6.1f ms  sims running %4d" % (q, int(((t0 <= q) & (t1 > q)).sum())))
nr, ns = len(grid.rates), len(grid.scales)
d = dur.reshape(nr, ns)
print("duration by rate row (ms): min/median/max per 8th row:")
for r in range(0, nr, 8):
    print("  rate %5.2f: %.1f / %.1f / %.1f; start %.1f" % (grid.rates[r], d[r].min(), np.median(d[r]), d[r].max(), t0.reshape(nr, ns)[r].min()))
np.save("gpurun_out/timeline_real.npy", np.stack([t0, t1]))
