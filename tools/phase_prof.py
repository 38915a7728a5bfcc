"""Per-phase cycle accounting of the fast sweep kernel (profiling build, -DSL_PHASE_PROF).

usage: SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_prof.so python tools/phase_prof.py [rates scales]
Prints per-phase cycle totals over all sims and for the longest sim."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200 import _native as N  # noqa: E402
from paper_2505_23022_b200.sweep import SweepGrid, build_local  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 64
grid = SweepGrid(rates=tuple(np.linspace(2.0, 32.0, nr)), scales=tuple(np.geomspace(0.5, 2.0, ns)))
eng, owned, _ = build_local(grid, device=torch.device("cuda", 0))
eng.launch()
torch.cuda.synchronize()
res = eng.results()
lib = N.lib()
lib.sl_phase_prof_read.argtypes = [C.c_void_p, C.c_int32]
out = np.zeros((eng.n_sims, 26), np.uint64)
assert lib.sl_phase_prof_read(out.ctypes.data, eng.n_sims) == eng.n_sims
k4 = out[:, 22:26].sum(axis=0)
print('general steps: R>32 & W==0 %d, R>32 & blocked & walk ahead %d, R>32 %d, W>0 & not blocked %d' % tuple(int(x) for x in k4))
names = ["arrivals+top", "quiet", "walk", "inv_sum", "admit", "decode", "tail", "retire",
         "gen_steps", "quiet_blocks", "quiet_steps", "gen_blocked", "maxW", "maxR"]
cyc = out[:, :8].astype(np.float64)
tot = cyc.sum(axis=0)
print("all sims: total cycles %.3e (%d sims); per-phase share:" % (tot.sum(), eng.n_sims))
for k in range(8):
    print(f"  {names[k]:14s} {100 * tot[k] / tot.sum():5.1f}%   {tot[k] / max(1, out[:, 8].sum()):8.1f} cyc/gen-step")
cnt = out[:, 8:12].sum(axis=0)
mw, mr = out[:, 12].astype(np.int64), out[:, 13].astype(np.int64)
print("max waiting per sim: quantiles", np.percentile(mw, [50, 90, 99, 100]).tolist(),
      "sims with maxW > 32:", int((mw > 32).sum()), "> 64:", int((mw > 64).sum()),
      "| max running: quantiles", np.percentile(mr, [50, 90, 99, 100]).tolist())
print("counts:", dict(zip(names[8:12], cnt.tolist())), "sim steps", int(res["n_steps"].sum()),
      "request_steps", int(res["request_steps"].sum()))
print("quiet: %.1f cyc/quiet-step, %.2f steps/block" % (tot[1] / max(1, cnt[2]), cnt[2] / max(1, cnt[1])))
tot_s = cyc.sum(axis=1)
order = np.argsort(-tot_s)
print("top-8 sims by cycles (ms at 1.965 GHz):", [(int(k), round(tot_s[k] / 1.965e6, 1), int(res["n_steps"][k])) for k in order[:8]])
i = int(order[0])
print(f"longest sim {i}: {cyc[i].sum():.3e} cycles, steps {int(res['n_steps'][i])}")
for k in range(8):
    print(f"  {names[k]:14s} {100 * cyc[i, k] / cyc[i].sum():5.1f}%")
print("  counts", out[i, 8:].tolist())

wk = out[:, 16:20].sum(axis=0).astype(np.float64)
print("walks %d (exact %d), mean W at walk %.1f; admission scans: sum W %d (mean W %.1f over gen steps)" % (
    wk[0], wk[1], wk[2] / max(1, wk[0]), wk[3], wk[3] / max(1, out[:, 8].sum())))
ce, cc = out[:, 20].sum(), out[:, 21].sum()
print("walk cycles: exact walks %.3e (%.0f per walk), certified-only %.3e (%.0f per walk)" % (
    ce, ce / max(1, wk[1]), cc, cc / max(1, wk[0] - wk[1])))
# occupancy timeline from the per-sim globaltimer stamps
t0, t1 = out[:, 14].astype(np.int64), out[:, 15].astype(np.int64)
base = t0.min()
t0, t1 = (t0 - base) / 1e6, (t1 - base) / 1e6
span = t1.max()
print("timeline: makespan %.1f ms; sim-busy sum / (slots x makespan) = %.3f" % (
    span, (t1 - t0).sum() / (148 * 16 * span)))
for q in np.linspace(0, span, 13)[1:]:
    print("  t=%6.1f ms  sims running %4d" % (q, int(((t0 <= q) & (t1 > q)).sum())))
rate_idx = np.arange(eng.n_sims) // ns if eng.n_sims == nr * ns else None
if rate_idx is not None:
    for r in range(0, nr, max(1, nr // 8)):
        sel = rate_idx == r
        print("  rate %5.2f: dur %.1f-%.1f ms, start %.1f-%.1f" % (
            grid.rates[r], (t1 - t0)[sel].min(), (t1 - t0)[sel].max(), t0[sel].min(), t0[sel].max()))
np.save("gpurun_out/timeline.npy", np.stack([t0, t1]))
