"""Run the config-2 plan kernels once at a given size (for ncu captures).
usage: python tools/plan_only.py S W R [fused]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200.plan import PlanBatch  # noqa: E402
from paper_2505_23022_b200.snapshot import (config2_arrays, config2_plan_arrays_fast,  # noqa: E402
                                            plan_arrays)

S, W, R = (int(x) for x in sys.argv[1:4])
arrays = config2_plan_arrays_fast(S, W, R, seed=11) if S > 4096 else \
    plan_arrays(config2_arrays(S, W, R, seed=11))
pb = PlanBatch(arrays=arrays, device="cuda")
itl, pre = (1e-6, 1e-3, 1e-5, 5e-3, 1.1), (0.004, 128.0, 2e-5, 1.5e-3)
for _ in range(2):
    pb.sort()
    pb.guard_admit(3, itl, pre)
    pb.select(3, True)
    if len(sys.argv) > 4:
        pb.plan(3, itl, pre)
torch.cuda.synchronize()
print("ok")
