"""Config-2 plan kernels alone (bench.py's plan_microbench): per-shape, per-kernel us and HBM fraction."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

peak, _ = bench.peaks()
r = bench.plan_microbench(torch.device("cuda", 0), peak)
for k, v in r.items():
    if not isinstance(v, dict):
        print(k, round(v, 2))
        continue
    print(k, round(v["us_per_step"], 2), {kk: (round(vv["us"], 2), round(vv["frac"], 3))
                                            for kk, vv in v["kernels"].items()})
if len(sys.argv) > 1:
    json.dump(r, open(sys.argv[1], "w"))
