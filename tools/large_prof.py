"""Phase timeline of the one-CTA-per-segment guard kernel at the stress shape
(profiling build: SL_LIB_PATH=.../libvar_lprof.so, built with -DSL_LARGE_PROF)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200 import _native as N  # noqa: E402
from paper_2505_23022_b200.plan import PlanBatch  # noqa: E402
from paper_2505_23022_b200.snapshot import config2_arrays, plan_arrays  # noqa: E402

S, W, R = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1, 32768, 32768)
pb = PlanBatch(arrays=plan_arrays(config2_arrays(S, W, R, seed=11)), device="cuda")
itl, pre = (1e-6, 1e-3, 1e-5, 5e-3, 1.1), (0.004, 128.0, 2e-5, 1.5e-3)
pb.sort()
lib = N.lib()
lib.sl_large_prof_read.argtypes = [C.c_void_p]
l2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    l2.zero_()  # cold L2, as bench.py times it
    torch.cuda.synchronize()
    pb.guard_admit(3, itl, pre)
    torch.cuda.synchronize()
    t = np.zeros(16, np.uint64)
    lib.sl_large_prof_read(t.ctypes.data)
    c = t[8:13].astype(np.int64)
    t = (t[:8].astype(np.int64) - int(t[0])) / 1e3
    print("walk tile phases (us at 1.965 GHz): loads+outright %.1f compact %.1f chain %.1f bookkeeping %.1f; survivors %d"
          % (c[0] / 1965, c[1] / 1965, c[2] / 1965, c[3] / 1965, c[4]))
    print("us: walk %.1f inv %.1f minlens %.1f vbs_run %.1f admission %.1f end %.1f; kernel entry %.1f" % tuple(list(t[1:7]) + [t[7]]))
