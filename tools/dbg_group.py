"""The many-segment guard kernel (guard_admit_group_kernel, cp.async staging)
once on a ragged 4,096-segment batch, for compute-sanitizer:
    compute-sanitizer --tool racecheck python tools/dbg_group.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SL_PLAN_FUSED", "0")
os.environ.setdefault("SL_PLAN_CTA_MAX", "0")
os.environ.setdefault("SL_PLAN_GROUP_MIN", "1")
import torch  # noqa: E402

from paper_2505_23022_b200.plan import PlanBatch  # noqa: E402
from paper_2505_23022_b200.snapshot import config2_arrays, plan_arrays  # noqa: E402

S = 4096
ws = list(np.resize([0, 1, 5, 31, 32, 33, 40, 64, 17, 2, 32, 0], S))
rs = list(np.resize([3, 0, 32, 33, 16, 1, 64, 0, 8, 40, 2, 31], S))
pb = PlanBatch(arrays=plan_arrays(config2_arrays(S, ws, rs, 20)), device="cuda")
pb.sort()
pb.guard_admit(3, (1e-6, 1e-3, 1e-5, 5e-3, 1.1), (0.004, 128.0, 2e-5, 1.5e-3))
torch.cuda.synchronize()
print("ok", int(pb.o["seg_counts"].view(-1, 4)[:, 1].sum().item()), "admitted")
