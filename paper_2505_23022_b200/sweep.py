"""Rate x SLO-scale goodput sweeps over many independent simulations.

A sweep is the batched form of ``slosim.report.sweep`` (report.py:180-221):
one trace per request rate, regenerated with ``derive_seed(base, "trace", qps)``
(``_trace_for_qps``, report.py:167-177), crossed with an SLO-scale axis that
multiplies both thresholds.  Cells are independent, so
multi-GPU runs shard cells across ranks (rate-strided for balance) with no
data-path collective; the only collective is one NCCL all_gather of the
fixed-width result rows at the end.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .batch import BatchEngine, Cell, CellConfig, TraceArrays
from .seeds import derive_seed
from .workload import LogNormalDist, WorkloadSpec, generate_arrays

ACCEPTANCE_ITL = (1e-6, 1e-3, 1e-5, 5e-3, 1.1)  # tests/test_acceptance.py:48
ACCEPTANCE_PREFILL = (0.004, 128.0, 2e-5, 1.5e-3)  # tests/test_acceptance.py:49


@dataclass
class SweepGrid:
    """Config-3 style grid: rates x SLO scales, n_requests per trace."""

    rates: tuple[float, ...] = tuple(np.linspace(2.0, 32.0, 64))
    scales: tuple[float, ...] = tuple(np.geomspace(0.5, 2.0, 64))
    n_requests: int = 10_000
    base_seed: int = 0
    prompt: tuple[float, float] = (5.0, 0.7)
    output: tuple[float, float] = (4.0, 0.7)
    category_weights: tuple[float, ...] = (1.0,) * 6
    config: CellConfig = field(default_factory=lambda: CellConfig(
        itl=ACCEPTANCE_ITL, prefill=ACCEPTANCE_PREFILL))

    @property
    def n_cells(self) -> int:
        return len(self.rates) * len(self.scales)

    def trace_for_rate(self, qps: float) -> TraceArrays:
        spec = WorkloadSpec(qps=float(qps), duration=1.1 * self.n_requests / float(qps),
                            seed=derive_seed(self.base_seed, "trace", float(qps)),
                            prompt_len_dist=LogNormalDist(*self.prompt),
                            output_len_dist=LogNormalDist(*self.output),
                            category_weights=self.category_weights)
        a = generate_arrays(spec, limit=self.n_requests)
        # oracle predictor: predicted == true output length (predictor.py:116-117)
        return TraceArrays(a["arrival"], a["ttft_slo"], a["tpot_slo"], a["prompt_len"],
                           a["true_out"], a["true_out"].copy(), a["id"], a["category"])

    def cell_index(self, ri: int, si: int) -> int:
        return ri * len(self.scales) + si


def shard_cells(n_cells: int, n_scales: int, rank: int, world: int) -> np.ndarray:
    """Global cell ids owned by `rank`: cells are ordered rate-major; rank r takes
    the SLO scales s with s % world == r at EVERY rate, so every rank gets the
    same rate mix and hence the same expected work."""
    ids = np.arange(n_cells)
    return ids[(ids % n_scales) % world == rank]


def build_local(grid: SweepGrid, rank: int = 0, world: int = 1, outcomes: bool = False,
                device=None) -> tuple[BatchEngine, np.ndarray, list[TraceArrays]]:
    """Traces this rank needs + a BatchEngine over its cells."""
    owned = shard_cells(grid.n_cells, len(grid.scales), rank, world)
    need = sorted({int(c) // len(grid.scales) for c in owned})
    tix = {ri: k for k, ri in enumerate(need)}
    traces = [grid.trace_for_rate(grid.rates[ri]) for ri in need]
    cells = [Cell(tix[int(c) // len(grid.scales)], grid.config,
                  slo_scale=float(grid.scales[int(c) % len(grid.scales)])) for c in owned]
    eng = BatchEngine(traces, cells, outcomes=outcomes, device=device)
    return eng, owned, traces


def gather_rows(rows_dev, owned: np.ndarray, n_cells: int, group=None) -> np.ndarray:
    """All-gather fixed-width result rows (uint8 tensors) from every rank and
    place them by global cell id.  Works with NCCL (GPU tensors) and gloo (CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    item = N.RESULT_DTYPE.itemsize
    n_local = torch.tensor([len(owned)], dtype=torch.int64, device=rows_dev.device)
    all_n = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(all_n, n_local, group=group)
    maxn = int(max(int(x.item()) for x in all_n))
    pad_rows = torch.zeros(maxn * item, dtype=torch.uint8, device=rows_dev.device)
    pad_rows[: rows_dev.numel()] = rows_dev
    ids = torch.full((maxn,), -1, dtype=torch.int64, device=rows_dev.device)
    ids[: len(owned)] = torch.from_numpy(owned.astype(np.int64)).to(rows_dev.device)
    out_rows = torch.zeros(world * maxn * item, dtype=torch.uint8, device=rows_dev.device)
    out_ids = torch.zeros(world * maxn, dtype=torch.int64, device=rows_dev.device)
    dist.all_gather_into_tensor(out_rows, pad_rows, group=group)
    dist.all_gather_into_tensor(out_ids, ids, group=group)
    rows = out_rows.cpu().numpy().view(N.RESULT_DTYPE)
    gid = out_ids.cpu().numpy()
    full = np.zeros(n_cells, N.RESULT_DTYPE)
    sel = gid >= 0
    full[gid[sel]] = rows[sel]
    return full


def surface(grid: SweepGrid, rows: np.ndarray) -> dict[str, np.ndarray]:
    """Goodput / attainment surfaces [rate, scale] from gathered rows (host, fixed order)."""
    shape = (len(grid.rates), len(grid.scales))
    return {"goodput": rows["goodput"].reshape(shape), "adherence": rows["adherence"].reshape(shape),
            "request_steps": rows["request_steps"].reshape(shape)}
