"""Shared sweep-parity case builder: traces + cells for GPU and the oracle."""

from __future__ import annotations

import numpy as np

from paper_2505_23022_b200.batch import Cell, CellConfig, TraceArrays
from paper_2505_23022_b200.seeds import derive_seed
from paper_2505_23022_b200.workload import LogNormalDist, WorkloadSpec, generate_arrays

ACC_ITL = (1e-6, 1e-3, 1e-5, 5e-3, 1.1)
ACC_PRE = (0.004, 128.0, 2e-5, 1.5e-3)


def make_trace(qps: float, n: int, base_seed: int = 11, p=(5.0, 0.7), o=(4.0, 0.7)) -> TraceArrays:
    spec = WorkloadSpec(qps=qps, duration=1.2 * n / qps, seed=derive_seed(base_seed, "trace", qps),
                        prompt_len_dist=LogNormalDist(*p), output_len_dist=LogNormalDist(*o),
                        category_weights=(1.0,) * 6)
    a = generate_arrays(spec, limit=n)
    return TraceArrays(a["arrival"], a["ttft_slo"], a["tpot_slo"], a["prompt_len"], a["true_out"],
                       a["true_out"].copy(), a["id"], a["category"])


def oracle_job(t: TraceArrays, cell: Cell) -> dict:
    """Oracle inputs for one cell: the host applies the same single IEEE ops
    (arrival / rate_factor, slo * slo_scale) the device applies on the fly."""
    from oracle import oracle as orc

    c = cell.config
    return dict(arrival=t.arrival / cell.rate_factor, ttft_slo=t.ttft_slo * cell.slo_scale,
                tpot_slo=t.tpot_slo * cell.slo_scale, prompt_len=t.prompt_len,
                true_out=t.true_out, ids=t.id, predicted=t.predicted,
                params=orc.make_params(policy=c.policy, ttft_guard=c.ttft_guard,
                                       tpot_guard=c.tpot_guard, admission_min=c.admission_min,
                                       horizon=c.horizon, max_batch_size=c.max_batch_size,
                                       prefill_priority=c.prefill_priority, itl=c.itl,
                                       prefill=c.prefill))


def grid(n_req: int = 1500, rates=(2.0, 8.0, 16.0, 32.0), scales=None):
    scales = np.geomspace(0.5, 2.0, 6) if scales is None else scales
    base = make_trace(8.0, n_req)
    native = len(base) / base.arrival[-1]
    traces = [base] + [make_trace(q, n_req) for q in rates[2:]]
    cells = []
    cfg = CellConfig(itl=ACC_ITL, prefill=ACC_PRE)
    for q in rates:  # rate axis by rescaling the base trace (report._trace_for_qps)
        for s in scales:
            cells.append(Cell(0, cfg, slo_scale=float(s), rate_factor=float(q / native)))
    for ti in range(1, len(traces)):  # rate axis by regeneration
        for s in scales[::2]:
            cells.append(Cell(ti, cfg, slo_scale=float(s)))
    variants = [CellConfig(itl=ACC_ITL, prefill=ACC_PRE, ttft_guard=False),
                CellConfig(itl=ACC_ITL, prefill=ACC_PRE, tpot_guard=False),
                CellConfig(itl=ACC_ITL, prefill=ACC_PRE, ttft_guard=False, tpot_guard=False),
                CellConfig(itl=ACC_ITL, prefill=ACC_PRE, admission_min="r_only"),
                CellConfig(itl=ACC_ITL, prefill=ACC_PRE, horizon=60.0),
                CellConfig(policy="greedy", itl=ACC_ITL, prefill=ACC_PRE, max_batch_size=64),
                CellConfig(policy="sjf", itl=ACC_ITL, prefill=ACC_PRE, max_batch_size=16),
                CellConfig(policy="early_reject", itl=ACC_ITL, prefill=ACC_PRE,
                           max_batch_size=16),
                CellConfig(policy="greedy", itl=ACC_ITL, prefill=ACC_PRE, max_batch_size=16,
                           prefill_priority=True)]
    for v in variants:
        cells.append(Cell(len(traces) - 1, v, slo_scale=1.0))
    # wide (128-bit) credits: SLO span > 2^10 within one sim
    wide = make_trace(16.0, 600)
    wide.tpot_slo[::5] = 8.0
    wide.tpot_slo[1::7] = 0.002
    traces.append(wide)
    cells.append(Cell(len(traces) - 1, cfg, slo_scale=1.0))
    return traces, cells
