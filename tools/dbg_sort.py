import sys, numpy as np, torch
sys.path.insert(0, '.')
from tests.test_gpu_sort import _arrays
from paper_2505_23022_b200.plan import PlanBatch
for ws in ([9000], [20000], [20000, 9000]):
    a = _arrays(ws, seed=5, ties=False, cluster=19990)
    pb = PlanBatch(arrays=a)
    pb.sort()
    torch.cuda.synchronize()
    perm = pb.o["perm"].cpu().numpy()
    dl = a["w_arrival"] + a["w_ttft"]
    ok = True
    for s in range(len(ws)):
        b, e = int(a["w_begin"][s]), int(a["w_begin"][s + 1])
        want = b + np.lexsort((a["w_id"][b:e], a["w_arrival"][b:e], dl[b:e]))
        ok &= np.array_equal(perm[b:e], want)
    print(ws, "ok" if ok else "MISMATCH", flush=True)
