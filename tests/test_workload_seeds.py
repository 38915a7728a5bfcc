"""Host-side input preparation matches the reference streams exactly
(fixtures from tests/golden/make_golden.py)."""

import json
import os

import numpy as np
import pytest

from paper_2505_23022_b200.core import SloCategory, SloCategoryTable, relaxed_slo_table
from paper_2505_23022_b200.seeds import derive_seed
from paper_2505_23022_b200.workload import (LogNormalDist, UniformDist, WorkloadSpec, generate,
                                            generate_arrays, load_trace, rescale_arrivals,
                                            save_trace)

G = os.path.join(os.path.dirname(__file__), "golden")
THREE = SloCategoryTable(rows=(SloCategory(1, 0.5, 0.030), SloCategory(2, 2.0, 0.050),
                               SloCategory(3, 7.5, 0.100)))


def _spec(qps, duration, seed, p=(5.0, 0.7), o=(4.0, 0.7), table=None, ncat=6, uni=None):
    pd = LogNormalDist(*p) if uni is None else UniformDist(*uni[0])
    od = LogNormalDist(*o) if uni is None else UniformDist(*uni[1])
    return WorkloadSpec(qps=qps, duration=duration, seed=seed, prompt_len_dist=pd,
                        output_len_dist=od, category_weights=(1.0,) * ncat, slo_table=table)


SPECS = [_spec(8.0, 40.0, 7, table=THREE, ncat=3), _spec(25.0, 10.0, 20240601),
         _spec(5.0, 20.0, 2, uni=((10, 300), (1, 40))),
         _spec(14.0, 10.0, 3, p=(4.6, 0.9), o=(4.5, 0.9))]


@pytest.mark.parametrize("k", range(len(SPECS)))
def test_generate_matches_reference_stream(k):
    kat = np.load(os.path.join(G, "workload_kat.npz"))
    tr = generate(SPECS[k])
    assert np.array_equal(np.array([r.arrival_time for r in tr]), kat[f"w{k}_arrival"])
    assert np.array_equal(np.array([r.prompt_len for r in tr]), kat[f"w{k}_prompt_len"])
    assert np.array_equal(np.array([r.true_output_len for r in tr]), kat[f"w{k}_true_out"])
    assert np.array_equal(np.array([r.category for r in tr]), kat[f"w{k}_category"])
    assert np.array_equal(np.array([r.tpot_slo for r in tr]), kat[f"w{k}_tpot_slo"])
    a = generate_arrays(SPECS[k])
    assert np.array_equal(a["arrival"], kat[f"w{k}_arrival"])
    assert np.array_equal(a["ttft_slo"], kat[f"w{k}_ttft_slo"])
    b = generate_arrays(SPECS[k], limit=7)
    assert np.array_equal(b["arrival"], kat[f"w{k}_arrival"][:7])


def test_golden_sim_traces_regenerate():
    """The config1 / overload fixture traces are generate(spec)[:n]."""
    meta = json.load(open(os.path.join(G, "sims.json")))
    blobs = np.load(os.path.join(G, "sims.npz"))
    ci = [m["name"] for m in meta].index("overload_scorpio")
    a = generate_arrays(_spec(25.0, 90.0, 20240601), limit=2000)
    assert np.array_equal(a["arrival"], blobs[f"c{ci}_arrival"])
    assert np.array_equal(a["prompt_len"], blobs[f"c{ci}_prompt_len"])


def test_derive_seed_kat():
    for base, parts, want in json.load(open(os.path.join(G, "seed_kat.json"))):
        assert derive_seed(base, *parts) == int(want)


def test_trace_io_roundtrip(tmp_path):
    tr = generate(_spec(5.0, 5.0, 1, table=relaxed_slo_table()))
    p = tmp_path / "t.jsonl"
    save_trace(tr, p)
    back = load_trace(p)
    assert [r.id for r in back] == [r.id for r in tr]
    assert all(abs(a.tpot_slo - b.tpot_slo) < 1e-15 for a, b in zip(tr, back))
    r2 = rescale_arrivals(tr, 2.0)
    assert all(x.arrival_time == y.arrival_time / 2.0 for x, y in zip(r2, tr))
    with pytest.raises(ValueError):
        rescale_arrivals(tr, 0.0)
