"""Native trace synthesis (csrc_host/tracegen.c) against the Python restatement of
the reference's per-request draw loop (workload._draw_rows, which the golden
tests pin to slosim.workload.generate): identical arrivals, categories and
lengths, draw for draw, including zero category weights and the horizon stop."""

import numpy as np
import pytest

from paper_2505_23022_b200 import workload as W
from paper_2505_23022_b200.seeds import derive_seed


@pytest.mark.parametrize("qps", [0.7, 8.0, 31.5])
@pytest.mark.parametrize("dists", [((5.0, 0.7), (4.0, 0.7)), ((4.6, 0.9), (4.5, 0.9)),
                                   ((0.5, 2.5), (0.1, 3.0))])
@pytest.mark.parametrize("limit", [None, 1500])
def test_native_generator_matches_draw_loop(qps, dists, limit):
    if W._tracegen() is None:
        pytest.skip("native trace generator not built")
    spec = W.WorkloadSpec(qps=qps, duration=1.1 * 1500 / qps, seed=derive_seed(3, "trace", qps),
                          prompt_len_dist=W.LogNormalDist(*dists[0]),
                          output_len_dist=W.LogNormalDist(*dists[1]),
                          category_weights=(1.0, 2.0, 0.0, 1.0, 1.0, 3.0))
    got = W.generate_arrays(spec, limit)
    table, rows = W._draw_rows(spec, limit)
    r = np.array(rows, dtype=np.float64).reshape(-1, 4)
    assert len(r) == len(got["arrival"]) > 0
    assert np.array_equal(r[:, 0], got["arrival"])
    assert np.array_equal(r[:, 2].astype(np.int32), got["prompt_len"])
    assert np.array_equal(r[:, 3].astype(np.int32), got["true_out"])
    cid = np.array([row.category for row in table.rows], np.int32)
    assert np.array_equal(cid[r[:, 1].astype(np.int64)], got["category"])


def test_generate_objects_match_arrays():
    spec = W.WorkloadSpec(qps=4.0, duration=200.0, seed=11,
                          prompt_len_dist=W.LogNormalDist(5.0, 0.7),
                          output_len_dist=W.LogNormalDist(4.0, 0.7), category_weights=(1.0,) * 6)
    objs = W.generate(spec)
    arr = W.generate_arrays(spec)
    assert len(objs) == len(arr["arrival"])
    assert [q.arrival_time for q in objs] == arr["arrival"].tolist()
    assert [q.true_output_len for q in objs] == arr["true_out"].tolist()


def test_non_lognormal_lengths_use_the_draw_loop():
    """Uniform / empirical length distributions are not on the native path: the
    arrays come from the Python draw loop and still equal generate()."""
    spec = W.WorkloadSpec(qps=6.0, duration=60.0, seed=5,
                          prompt_len_dist=W.UniformDist(10, 500),
                          output_len_dist=W.EmpiricalDist((3, 7, 50, 200)),
                          category_weights=(1.0,) * 6)
    assert W._draw_native(spec, None) is None
    objs = W.generate(spec)
    arr = W.generate_arrays(spec)
    assert [q.prompt_len for q in objs] == arr["prompt_len"].tolist()
    assert [q.true_output_len for q in objs] == arr["true_out"].tolist()
    assert [q.arrival_time for q in objs] == arr["arrival"].tolist()
