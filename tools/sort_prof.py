"""clock64 stamps of sort_cluster_kernel, CTA 0 (profiling build: tools/build_variant.sh lprof
-DSL_LARGE_PROF; SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_lprof.so).  usage: sort_prof.py W"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200 import _native as N  # noqa: E402
from paper_2505_23022_b200.plan import PlanBatch  # noqa: E402
from paper_2505_23022_b200.snapshot import config2_plan_arrays_fast  # noqa: E402

lib = N.lib()
lib.sl_sort_prof_read.argtypes = [C.c_void_p]
for w in (int(x) for x in sys.argv[1:]):
    pb = PlanBatch(arrays=config2_plan_arrays_fast(1, w, 1, seed=11))
    for _ in range(3):
        t = np.zeros(96, np.uint64)
        lib.sl_sort_prof_read(t.ctypes.data)
        pb.sort()
        torch.cuda.synchronize()
        lib.sl_sort_prof_read(t.ctypes.data)
        k = int(t[0])
        st = t[1:k + 1].astype(np.int64)
        print("W=%d stamps %d, cycles between:" % (w, k), np.diff(st).tolist(), "total", st[-1] - st[0])
        c = t[32:96].reshape(16, 4).astype(np.int64)
        if c[0, 0]:
            print("  per CTA: local-sort ns", (c[:, 1] - c[:, 0]).tolist(), "after-scatter skew ns",
                  (c[:, 0] - c[:, 0].min()).tolist(), "big", c[:, 2].tolist(), "n", c[:, 3].tolist())
