"""LDF sort kernels (sl_ttft_sort_batch) against numpy's lexsort of the reference
sort key (deadline, arrival_time, id) -- sched_scorpio.py:193, schedtypes.py:28-32,
deadline = arrival + ttft (core.py:50-53) -- for every route: warp bitonic
(<= 32 waiting), the cluster sort for few large segments (one CTA, and 2, 4 and 8
CTAs merging through distributed shared memory), and tile sort + merge passes
for many large segments.  Keys include exact deadline ties and near-ties (equal
top 49 bits), which the packed-key networks must send to the full comparison."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _arrays(ws, seed, ties, cluster=None):
    rng = np.random.default_rng(seed)
    W = int(sum(ws))
    S = len(ws)
    arr = 10.0 - rng.uniform(0.0, 0.4, W)
    ttft = np.array([0.5, 2.0, 7.5])[rng.integers(0, 3, W)]
    if cluster:
        # `cluster` keys of each segment with distinct deadlines 1e-8 s apart (far
        # above the packed keys' 2^-34 s resolution: no near-ties), in random order
        for b, e in zip(np.cumsum([0] + ws[:-1]), np.cumsum(ws)):
            k = min(cluster, e - b)
            sel = b + rng.permutation(e - b)[:k]
            arr[sel] = 10.0 - 1e-8 * rng.permutation(k)
            ttft[sel] = 2.0
    if ties:
        # arrivals on a coarse grid -> many equal deadlines (ties on arrival too),
        # plus near-ties: deadlines one ulp apart
        arr = 10.0 - np.round(rng.uniform(0.0, 0.4, W) * 16) / 16
        k = rng.random(W) < 0.2
        arr[k] = np.nextafter(arr[k], 20.0)
    ids = rng.permutation(W).astype(np.int64)  # ids out of input order
    return {
        "w_begin": np.concatenate([[0], np.cumsum(ws)]).astype(np.int64),
        "r_begin": np.zeros(S + 1, np.int64),
        "w_arrival": arr, "w_ttft": ttft, "w_tpot": np.full(W, 0.05),
        "w_prefill": np.full(W, 0.004), "w_prompt": np.full(W, 64, np.int32),
        "w_pred": np.full(W, 16, np.int32), "w_id": ids,
        "r_tpot": np.zeros(0), "r_cur_len": np.zeros(0, np.int32), "r_id": np.zeros(0, np.int64),
        "r_credit": np.zeros(0, np.uint64), "now": np.full(S, 10.0),
        "credit_exp": np.full(S, -60, np.int32),
    }


CASES = {
    "warp": [32, 7, 1, 0, 31, 32] * 8,
    "cluster_1cta": [3000, 129, 4096],
    "cluster_2cta": [5000, 4097, 8192],
    "cluster_4cta": [16384, 9000],
    "cluster_8cta": [32768, 20000, 16385],
    "tiles": [3000] * 70,  # more than 64 segments: tile sort + merge passes
}


# clustered deadlines: 1,000 keys in one MSD bucket (the local sub-bucket pass
# overflows -> LSD passes in that CTA), and almost every key in one bucket (the
# distribution overflows a CTA -> cluster-wide LSD passes)
CLUSTERED = {"dense_cluster": ([32768], 1000), "one_bucket": ([20000, 9000], 19990)}


@pytest.mark.parametrize("case", list(CLUSTERED))
def test_ldf_sort_clustered_deadlines(case):
    from paper_2505_23022_b200.plan import PlanBatch

    ws, k = CLUSTERED[case]
    a = _arrays(ws, seed=5, ties=False, cluster=k)
    pb = PlanBatch(arrays=a)
    pb.sort()
    perm = pb.o["perm"].cpu().numpy()
    dl = a["w_arrival"] + a["w_ttft"]
    for s in range(len(ws)):
        b, e = int(a["w_begin"][s]), int(a["w_begin"][s + 1])
        want = b + np.lexsort((a["w_id"][b:e], a["w_arrival"][b:e], dl[b:e]))
        assert np.array_equal(perm[b:e], want), (case, s)


@pytest.mark.parametrize("ties", [False, True], ids=["random", "ties"])
@pytest.mark.parametrize("case", list(CASES))
def test_ldf_sort_matches_lexsort(case, ties):
    from paper_2505_23022_b200.plan import PlanBatch

    ws = CASES[case]
    a = _arrays(ws, seed=len(ws) * 7 + ties, ties=ties)
    pb = PlanBatch(arrays=a)
    pb.sort()
    perm = pb.o["perm"].cpu().numpy()
    dl = a["w_arrival"] + a["w_ttft"]
    for s in range(len(ws)):
        b, e = int(a["w_begin"][s]), int(a["w_begin"][s + 1])
        if e == b:
            continue
        want = b + np.lexsort((a["w_id"][b:e], a["w_arrival"][b:e], dl[b:e]))
        assert np.array_equal(perm[b:e], want), (case, s)
