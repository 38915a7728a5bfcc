"""Time sl_ttft_sort_batch alone for one segment of W waiting (CUDA events, mean of 20).
usage: python tools/sort_bench.py W [W ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200.plan import PlanBatch  # noqa: E402
from paper_2505_23022_b200.snapshot import config2_plan_arrays_fast  # noqa: E402

for w in (int(x) for x in sys.argv[1:]):
    pb = PlanBatch(arrays=config2_plan_arrays_fast(1, w, 1, seed=11))
    for _ in range(3):
        pb.sort()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        pb.sort()
    e1.record()
    torch.cuda.synchronize()
    print("W=%6d sort %.2f us" % (w, e0.elapsed_time(e1) * 1000 / 20))
