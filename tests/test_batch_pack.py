"""Cell packing from columns and a pinned trace table (the e2e input form) equals
packing from Cell objects and per-trace arrays, byte for byte; on the GPU the
two engines give identical result rows."""

import numpy as np
import pytest

from tests._sweepcase import make_trace


def _inputs():
    from paper_2505_23022_b200.batch import Cell, CellColumns, CellConfig

    traces = [make_trace(q, 300) for q in (4.0, 12.0, 24.0)]
    cfg = CellConfig()
    scales = np.geomspace(0.5, 2.0, 5)
    cells = [Cell(t, cfg, slo_scale=float(s)) for t in (2, 0, 1) for s in scales]
    cols = CellColumns(np.array([c.trace for c in cells]), np.array([c.slo_scale for c in cells]),
                       cfg)
    return traces, cells, cols


def test_pack_from_columns_and_table_matches_cells():
    from paper_2505_23022_b200.batch import TraceTable, default_order, pack_cells

    traces, cells, cols = _inputs()
    table = TraceTable(traces, pin=False)
    a = pack_cells(traces, cells)
    b = pack_cells(table, cols)
    assert a.tobytes() == b.tobytes()
    assert np.array_equal(default_order(traces, a), default_order(table, b))
    assert np.array_equal(table.begin, np.cumsum([0] + [len(t) for t in traces]))
    for k in ("arrival", "ttft_slo", "id"):
        assert np.array_equal(table.host[k].numpy(), np.concatenate([getattr(t, k) for t in traces]))


def test_columns_validate():
    from paper_2505_23022_b200.batch import CellColumns, TraceTable, pack_cells

    traces, _, _ = _inputs()
    with pytest.raises(ValueError):
        pack_cells(TraceTable(traces, pin=False), CellColumns(np.array([0, 3]), np.ones(2)))
    with pytest.raises(ValueError):
        pack_cells(traces, CellColumns(np.array([0]), np.array([-1.0])))
    with pytest.raises(ValueError):
        CellColumns(np.array([0, 1]), np.ones(3))


@pytest.mark.gpu
def test_engine_from_table_matches_engine_from_traces():
    from paper_2505_23022_b200.batch import BatchEngine, TraceTable

    traces, cells, cols = _inputs()
    e1 = BatchEngine(traces, cells, device="cuda:0")
    e1.launch()
    e2 = BatchEngine(TraceTable(traces), cols, device="cuda:0")
    e2.launch()
    assert e1.results().tobytes() == e2.results().tobytes()
