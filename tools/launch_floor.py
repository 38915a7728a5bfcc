"""Event-timed floor of one tiny launch in bench.py's config-2 harness (behind a GPU
sleep, L2 flushed): an empty-ish torch kernel vs the fused plan step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200.plan import PlanBatch  # noqa: E402
from paper_2505_23022_b200.snapshot import config2_arrays, plan_arrays  # noqa: E402

dev = torch.device("cuda", 0)
l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
x = torch.zeros(1, device=dev)
pb = PlanBatch(arrays=plan_arrays(config2_arrays(1024, 32, 32, seed=11)), device=dev)
itl, pre = (1e-6, 1e-3, 1e-5, 5e-3, 1.1), (0.004, 128.0, 2e-5, 1.5e-3)
stream = torch.cuda.current_stream(dev)
for name, fn in (("tiny torch kernel", lambda: x.add_(1.0)), ("fused plan step", lambda: pb.plan(3, itl, pre))):
    ts = []
    for it in range(12):
        l2.zero_()
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print("%-20s %.2f us (min %.2f)" % (name, np.mean(ts), np.min(ts)))
