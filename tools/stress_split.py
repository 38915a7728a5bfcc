"""Time the config-2 stress segment's guard kernel split: walk only vs walk+admission."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_23022_b200 import _native as N
from paper_2505_23022_b200.plan import PlanBatch
from paper_2505_23022_b200.snapshot import config2_arrays, plan_arrays
pb = PlanBatch(arrays=plan_arrays(config2_arrays(1, 32768, 32768, seed=11)), device="cuda")
itl, pre = (1e-6, 1e-3, 1e-5, 5e-3, 1.1), (0.004, 128.0, 2e-5, 1.5e-3)
pb.sort()
for name, flags in (("walk only", 3 | 64), ("walk+admission", 3), ("admission only (no walk)", 2)):
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pb.guard_admit(flags, itl, pre); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    r = pb.results()[0]
    print(name, "ms", [round(t, 3) for t in ts], "kept", r.kept, "adm", r.admitted, "rej", r.rejected)
