"""Run the credit-select kernels (cluster route) on a few shapes (for compute-sanitizer)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200.plan import PlanBatch  # noqa: E402
from paper_2505_23022_b200.snapshot import config2_arrays, plan_arrays  # noqa: E402

itl, pre = (1e-6, 1e-3, 1e-5, 5e-3, 1.1), (0.004, 128.0, 2e-5, 1.5e-3)
for S, W, R in ((1, 64, 4096), (4, 30, 300), (2, 10, 0), (3, 5, 7)):
    pb = PlanBatch(arrays=plan_arrays(config2_arrays(S, W, R, seed=5)))
    for flags in (3, 1):
        for seg_min in (True, False):
            pb.select(flags, seg_min)
    torch.cuda.synchronize()
    print(S, W, R, "ok", flush=True)
