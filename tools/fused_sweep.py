"""Fused plan step time (CUDA events, L2 flushed, behind a GPU sleep) at several
segment counts of the primary shape (32 waiting + 32 running), for the routing
threshold between the warp-pair and the one-warp fused kernels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200.plan import PlanBatch  # noqa: E402
from paper_2505_23022_b200.snapshot import config2_plan_arrays_fast  # noqa: E402

itl, pre = (1e-6, 1e-3, 1e-5, 5e-3, 1.1), (0.004, 128.0, 2e-5, 1.5e-3)
l2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for S in (512, 1024, 2048, 4096, 8191):
    pb = PlanBatch(arrays=config2_plan_arrays_fast(S, 32, 32, seed=11))
    ts = []
    for it in range(7):
        l2.zero_()
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        pb.plan(3, itl, pre)
        e1.record(st)
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print("S=%5d fused %.2f us" % (S, np.mean(ts)))
