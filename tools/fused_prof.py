"""clock64 stamps of the fused plan step, segment 0 (profiling build: tools/build_variant.sh
lprof -DSL_LARGE_PROF; SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_lprof.so), primary shape:
start, inputs issued, sorted, fields gathered, walk done, aggregates + inv fold, admission, vbs, end."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200 import _native as N  # noqa: E402
from paper_2505_23022_b200.plan import PlanBatch  # noqa: E402
from paper_2505_23022_b200.snapshot import config2_arrays, plan_arrays  # noqa: E402

lib = N.lib()
lib.sl_fused_prof_read.argtypes = [C.c_void_p]
pb = PlanBatch(arrays=plan_arrays(config2_arrays(1024, 32, 32, seed=11)))
itl, pre = (1e-6, 1e-3, 1e-5, 5e-3, 1.1), (0.004, 128.0, 2e-5, 1.5e-3)
l2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(4):
    t = np.zeros(16, np.uint64)
    lib.sl_fused_prof_read(t.ctypes.data)
    l2.zero_()
    torch.cuda.synchronize()
    pb.plan(3, itl, pre)
    torch.cuda.synchronize()
    lib.sl_fused_prof_read(t.ctypes.data)
    k = int(t[0])
    st = t[1:k + 1].astype(np.int64)
    print("stamps", k, "cycles between:", np.diff(st).tolist(), "total", st[-1] - st[0])
