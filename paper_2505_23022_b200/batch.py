"""Batched device execution of many independent simulations (the sweep hot path).

``BatchEngine`` owns the device buffers for one batch of simulation cells:
the packed trace table (SoA over requests), the ``sl_sim`` cell table, the
workspace, the per-sim result rows and optional per-request outcomes and
decision log.  ``launch()`` is one asynchronous ``sl_run_batch`` call on the
current torch stream; nothing on this path runs on the CPU except packing.

Reference: one cell == ``slosim.simengine.run(trace, SimConfig)``
(pkg/src/slosim/simengine.py:168-303); a batch == the cells of
``report.sweep`` (report.py:180-221) run concurrently.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

TRACE_FIELDS = ("arrival", "ttft_slo", "tpot_slo", "prompt_len", "true_out", "predicted", "id")
_TRACE_DTYPES = {"arrival": np.float64, "ttft_slo": np.float64, "tpot_slo": np.float64,
                 "prompt_len": np.int32, "true_out": np.int32, "predicted": np.int32,
                 "id": np.int64}


@dataclass
class TraceArrays:
    """One trace as host SoA (request order == arrival order, trace.py semantics)."""

    arrival: np.ndarray
    ttft_slo: np.ndarray
    tpot_slo: np.ndarray
    prompt_len: np.ndarray
    true_out: np.ndarray
    predicted: np.ndarray
    id: np.ndarray
    category: np.ndarray | None = None

    def __post_init__(self) -> None:
        for k in TRACE_FIELDS:
            setattr(self, k, np.ascontiguousarray(getattr(self, k), _TRACE_DTYPES[k]))
        n = len(self.arrival)
        if any(len(getattr(self, k)) != n for k in TRACE_FIELDS):
            raise ValueError("trace arrays must have equal length")
        if self.category is None:
            self.category = np.zeros(n, np.int32)
        validate_trace(self)

    def __len__(self) -> int:
        return len(self.arrival)


def validate_trace(t: TraceArrays) -> None:
    """Host-side checks that the reference raises as ValueError
    (core.py:40-48 Request.__post_init__, simengine.py:170-178 run)."""
    n = len(t.arrival)
    if n == 0:
        return
    if np.any(t.prompt_len < 1):
        raise ValueError("prompt_len must be >= 1")
    if np.any(t.true_out < 1):
        raise ValueError("true_output_len must be >= 1")
    if np.any(~(t.ttft_slo > 0)) or np.any(~(t.tpot_slo > 0)):
        raise ValueError("SLO thresholds must be positive")
    if np.any(t.arrival < 0):
        raise ValueError("arrival_time must be >= 0")
    if np.any(np.diff(t.arrival) < 0):
        raise ValueError("trace must be sorted by arrival time")
    if len(np.unique(t.id)) != n:
        raise ValueError("trace contains duplicate request ids")
    if np.any(t.predicted < 1):
        raise ValueError("predicted_len must be >= 1")


@dataclass
class CellConfig:
    """The SimConfig of one cell (simengine.py:46-61), flattened."""

    policy: str = "scorpio"
    itl: tuple = (1e-6, 1e-3, 1e-5, 5e-3, 1.1)  # alpha, beta, gamma, delta, epsilon
    prefill: tuple = (0.004, 128.0, 2e-5, 1.5e-3)  # phi, theta, alpha_p, beta_p
    ttft_guard: bool = True
    tpot_guard: bool = True
    admission_min: str = "r_prime"
    max_batch_size: int = 256
    prefill_priority: bool = False
    horizon: float | None = None

    def flags(self) -> int:
        f = 0
        if self.ttft_guard:
            f |= N.FLAG_TTFT_GUARD
        if self.tpot_guard:
            f |= N.FLAG_TPOT_GUARD
        if self.admission_min == "r_only":
            f |= N.FLAG_R_ONLY
        elif self.admission_min != "r_prime":
            raise ValueError(f"unknown admission_min {self.admission_min!r}")
        if self.horizon is not None:
            if not self.horizon > 0:
                raise ValueError("horizon must be positive when finite")
            f |= N.FLAG_HAS_HORIZON
        if self.prefill_priority:
            f |= N.FLAG_PREFILL_PRIORITY
        return f


@dataclass
class Cell:
    """One simulation: trace index, config, and the sweep axes."""

    trace: int
    config: CellConfig = field(default_factory=CellConfig)
    slo_scale: float = 1.0
    rate_factor: float = 1.0


@dataclass
class CellColumns:
    """Many cells sharing one config, as columns (the sweep's form): trace index,
    SLO scale and rate factor per cell.  pack_cells handles it without a
    per-cell Python loop."""
    trace: np.ndarray
    slo_scale: np.ndarray
    config: CellConfig = field(default_factory=CellConfig)
    rate_factor: np.ndarray | None = None

    def __post_init__(self) -> None:
        self.trace = np.ascontiguousarray(self.trace, np.int64)
        self.slo_scale = np.ascontiguousarray(self.slo_scale, np.float64)
        self.rate_factor = (np.ones(len(self.trace)) if self.rate_factor is None else
                            np.ascontiguousarray(self.rate_factor, np.float64))
        if not (len(self.slo_scale) == len(self.trace) == len(self.rate_factor)):
            raise ValueError("cell columns must have equal length")

    def __len__(self) -> int:
        return len(self.trace)


class _TraceMeta:
    """Per-trace facts pack_cells / default_order need: lengths, last arrival,
    distinct TPOT SLOs, longest prompt, longest prompt + output."""

    def __init__(self, traces) -> None:
        self.lens = np.array([len(t) for t in traces], np.int64)
        self.last = np.array([float(t.arrival[-1]) if len(t) else 0.0 for t in traces])
        self.uniq_tpot = [np.unique(t.tpot_slo) for t in traces]
        self.max_prompt = np.array([int(t.prompt_len.max()) if len(t) else 0 for t in traces],
                                   np.int64)
        self.max_total = np.array(
            [int((t.prompt_len.astype(np.int64) + t.true_out).max()) if len(t) else 0
             for t in traces], np.int64)


class TraceTable:
    """Many traces as ONE host SoA (concatenated, `begin` offsets), in pinned
    memory when CUDA is available -- the form BatchEngine uploads with async
    copies -- plus the per-trace facts cell packing needs.  Build it once per
    set of traces; every BatchEngine over it then copies from pinned memory."""

    def __init__(self, traces: list[TraceArrays], pin: bool = True) -> None:
        import torch

        self.meta = _TraceMeta(traces)
        self.n = len(traces)
        self.begin = np.zeros(self.n + 1, np.int64)
        np.cumsum(self.meta.lens, out=self.begin[1:])
        self.categories = [t.category for t in traces]
        pin = pin and torch.cuda.is_available()
        self.host = {}
        for k in TRACE_FIELDS:
            a = (np.concatenate([getattr(t, k) for t in traces]) if traces else
                 np.zeros(0, _TRACE_DTYPES[k]))
            ht = torch.from_numpy(np.ascontiguousarray(a))
            self.host[k] = ht.pin_memory() if pin else ht
        bt = torch.from_numpy(self.begin.copy())
        self.host["begin"] = bt.pin_memory() if pin else bt

    def __len__(self) -> int:
        return self.n


def _meta(traces) -> _TraceMeta:
    return traces.meta if isinstance(traces, TraceTable) else _TraceMeta(traces)


_MIN_NORMAL = 2.2250738585072014e-308


def credit_params_many(uniq_tpot: np.ndarray, scales: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(E, wide) of the fixed-point credits for many cells sharing one trace
    (vectorised ``sl_credit_params``): E = min frexp exponent of the scaled TPOT
    SLOs - 53; wide when 2 * S_max needs more than 64 bits."""
    n = len(scales)
    if len(uniq_tpot) == 0:
        return np.zeros(n, np.int32), np.zeros(n, np.int32)
    prod = uniq_tpot[None, :] * scales[:, None]  # one IEEE multiply each, as on device
    if not (np.isfinite(prod).all() and (prod >= _MIN_NORMAL).all()):
        raise ValueError("TPOT SLOs must be positive normal doubles within the credit range")
    ex = np.frexp(prod)[1]
    emin, emax = ex.min(axis=1), ex.max(axis=1)
    E = emin - 53
    span = emax - emin
    if (E < -1022).any() or (53 + span + 1 > 128).any():
        raise ValueError("TPOT SLOs must be positive normal doubles within the credit range")
    return E.astype(np.int32), (53 + span + 1 > 64).astype(np.int32)


def _config_row(cfg: CellConfig) -> tuple:
    """Validated (policy code, flags, cap, horizon, 9 cost coefficients) of one config."""
    if cfg.policy not in N.POLICY:
        raise ValueError(f"unknown policy {cfg.policy!r}")
    a, b, g, d, e = (float(x) for x in cfg.itl)
    if e < 1.0:
        raise ValueError("epsilon must be >= 1.0")
    phi, th, ap, bp = (float(x) for x in cfg.prefill)
    if phi <= 0 or th < 0 or ap * th + bp < 0:
        raise ValueError("invalid PrefillParams")
    if cfg.max_batch_size < 1:
        raise ValueError("max_batch_size must be >= 1")
    return (N.POLICY[cfg.policy], cfg.flags(), int(cfg.max_batch_size),
            float(cfg.horizon) if cfg.horizon is not None else 0.0, a, b, g, d, e, phi, th, ap, bp)


def pack_cells(traces, cells, outcomes: bool = False,
               log_cells: list[int] | None = None) -> np.ndarray:
    """Build the sl_sim table (host), column-wise: per-config rows are validated
    once per distinct config object, credit exponents per trace for all its
    cells at once, workspace/outcome offsets by prefix sum.  `traces`: a list of
    TraceArrays or a TraceTable; `cells`: a list of Cell or a CellColumns (one
    config, no per-cell Python work)."""
    n = len(cells)
    sims = np.zeros(n, N.SIM_DTYPE)
    if n == 0:
        return sims
    meta = _meta(traces)
    if isinstance(cells, CellColumns):
        tr_idx, scale, factor = cells.trace, cells.slo_scale, cells.rate_factor
        keys = np.zeros(n, np.int64)
        table = [_config_row(cells.config)]
    else:
        tr_idx = np.fromiter((c.trace for c in cells), np.int64, n)
        scale = np.fromiter((c.slo_scale for c in cells), np.float64, n)
        factor = np.fromiter((c.rate_factor for c in cells), np.float64, n)
        rows: dict[int, tuple] = {}
        keys = np.empty(n, np.int64)
        table = []
        for k, c in enumerate(cells):
            key = id(c.config)
            r = rows.get(key)
            if r is None:
                r = rows[key] = (len(table), c.config)
                table.append(_config_row(c.config))
            keys[k] = r[0]
    if not ((scale > 0).all() and (factor > 0).all()):
        raise ValueError("slo_scale and rate_factor must be positive")
    if ((tr_idx < 0) | (tr_idx >= len(meta.lens))).any():
        raise ValueError("cell trace index out of range")
    cols = {name: np.array([row[j] for row in table])[keys]
            for j, name in enumerate(("policy", "flags", "max_batch_size", "horizon")
                                     + N.COST_FIELDS)}
    lens = meta.lens
    flags = cols["flags"].astype(np.int32)
    E = np.zeros(n, np.int32)
    wide = np.zeros(n, np.int32)
    # credit exponents: one vectorised call per distinct set of TPOT SLOs (a sweep's
    # traces share one SLO table), over every cell of the traces that have it
    groups: dict[bytes, list[int]] = {}
    for t in np.unique(tr_idx):
        groups.setdefault(meta.uniq_tpot[int(t)].tobytes(), []).append(int(t))
    for tlist in groups.values():
        sel = np.nonzero(np.isin(tr_idx, tlist))[0]
        E[sel], wide[sel] = credit_params_many(meta.uniq_tpot[tlist[0]], scale[sel])
    nonempty = lens[tr_idx] > 0
    # the fast kernel sums up to 64 current lengths in 32 bits
    flags[nonempty & (meta.max_total[tr_idx] >= 1 << 26)] |= N.FLAG_GENERAL_ONLY
    # a negative prefill_time (alpha_p < 0 past -beta_p/alpha_p) breaks the fast
    # kernel's monotone-prefix walk shortcuts: exact general kernel
    big = meta.max_prompt[tr_idx].astype(np.float64)
    ap, bp, th = cols["alpha_p"], cols["beta_p"], cols["theta"]
    flags[nonempty & (ap < 0) & (big > th) & (ap * big + bp < 0)] |= N.FLAG_GENERAL_ONLY
    ws = np.zeros(n, np.int64)
    np.cumsum(lens[tr_idx][:-1], out=ws[1:])
    log_slot = np.full(n, -1, np.int32)
    if log_cells:
        log_slot[np.asarray(log_cells, np.int64)] = np.arange(len(log_cells), dtype=np.int32)
    sims["trace"] = tr_idx
    sims["policy"] = cols["policy"]
    sims["flags"] = flags
    sims["max_batch_size"] = cols["max_batch_size"]
    sims["slo_scale"] = scale
    sims["rate_factor"] = factor
    sims["horizon"] = cols["horizon"]
    sims["credit_exp"] = E
    sims["credit_wide"] = wide
    sims["ws_offset"] = ws
    sims["out_offset"] = ws if outcomes else -1
    sims["log_slot"] = log_slot
    for name in N.COST_FIELDS:
        sims[name] = cols[name].astype(np.float64)
    return sims


class BatchEngine:
    """Device buffers + launch for one batch of cells (reusable across launches)."""

    def __init__(self, traces: "list[TraceArrays] | TraceTable",
                 cells: "list[Cell] | CellColumns | np.ndarray",
                 outcomes: bool = False, log_cells: list[int] | None = None,
                 log_steps: int = 0, log_ids: int = 0, order: np.ndarray | None = None,
                 device=None, mode: int = N.MODE_AUTO, log_skips: int = 0):
        torch = N.require_cuda()
        self.torch = torch
        self.device = torch.device(device if device is not None else "cuda")
        dev = self.device
        if isinstance(traces, TraceTable):
            # async copies from pinned host memory, enqueued first so that the
            # cell packing below runs on the host while they are in flight
            self._tr = {k: v.to(dev, non_blocking=True) for k, v in traces.host.items()}
        if isinstance(cells, np.ndarray):
            sims = cells
        else:
            sims = pack_cells(traces, cells, outcomes, log_cells)
        self.n_sims = len(sims)
        self.sims_host = sims
        self.mode = mode

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        if isinstance(traces, TraceTable):
            lens = traces.meta.lens
            self.trace_begin = traces.begin
        else:
            lens = np.array([len(t) for t in traces], np.int64)
            begin = np.zeros(len(traces) + 1, np.int64)
            np.cumsum(lens, out=begin[1:])
            self.trace_begin = begin
            self._tr = {k: up(np.concatenate([getattr(t, k) for t in traces]) if traces else
                              np.zeros(0, _TRACE_DTYPES[k])) for k in TRACE_FIELDS}
            self._tr["begin"] = up(begin)
        if order is None:
            order = default_order(traces, sims)
        self._sims = up(sims.view(np.uint8))
        self.total_slots = int(lens[sims["trace"].astype(np.int64)].sum()) if len(sims) else 0
        wsb = N.lib().sl_workspace_bytes(self.total_slots, self.n_sims)
        self._ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        self._res = torch.zeros(self.n_sims * N.RESULT_DTYPE.itemsize, dtype=torch.uint8,
                                device=dev)
        self._order = up(np.ascontiguousarray(order, np.int32))
        self.st = N.SlTraces(len(traces), 0, *[self._tr[k].data_ptr() for k in (
            "begin", "arrival", "ttft_slo", "tpot_slo", "prompt_len", "true_out", "predicted",
            "id")])
        self.has_outcomes = bool(outcomes)
        self.oc = None
        if outcomes:
            m = max(self.total_slots, 1)
            self._out = {
                "status": torch.empty(m, dtype=torch.int8, device=dev),
                "compliant": torch.empty(m, dtype=torch.int8, device=dev),
                "completion_step": torch.empty(m, dtype=torch.int32, device=dev),
                "first_token_time": torch.empty(m, dtype=torch.float64, device=dev),
                "completion_time": torch.empty(m, dtype=torch.float64, device=dev),
                "ttft": torch.empty(m, dtype=torch.float64, device=dev),
                "tpot": torch.empty(m, dtype=torch.float64, device=dev),
            }
            self.oc = N.SlOutcomes(*[self._out[k].data_ptr() for k in (
                "status", "compliant", "completion_step", "first_token_time", "completion_time",
                "ttft", "tpot")])
        self.lg = None
        rows = int((sims["log_slot"] >= 0).sum()) if len(sims) else 0
        if rows and log_steps > 0:
            sc, ic = int(log_steps), int(max(log_ids, 1))
            f64 = dict(dtype=torch.float64, device=dev)
            i32 = dict(dtype=torch.int32, device=dev)
            i64 = dict(dtype=torch.int64, device=dev)
            self._log = {k: torch.zeros(rows * sc, **f64) for k in (
                "now", "end", "prefill_s", "decode_s", "vbs", "min_slo")}
            for k in ("n_admitted", "n_rejected", "n_batch"):
                self._log[k] = torch.zeros(rows * sc, **i32)
            for k in ("adm_ids", "rej_ids", "batch_ids"):
                self._log[k] = torch.zeros(rows * ic, **i64)
            self._log["n_steps"] = torch.zeros(rows, **i64)
            self._log["adm_rec"] = torch.zeros(rows * ic * 5, **f64)
            kc = int(max(log_skips, 1))
            self._log["skip_now"] = torch.zeros(rows * kc, **f64)
            self._log["skip_target"] = torch.zeros(rows * kc, **f64)
            self._log["skip_waiting"] = torch.zeros(rows * kc, **i32)
            self._log["n_skips"] = torch.zeros(rows, **i64)
            self.log_shape = (rows, sc, ic, kc)
            self.lg = N.SlLog(sc, ic, *[self._log[k].data_ptr() for k in (
                "now", "end", "prefill_s", "decode_s", "vbs", "min_slo", "n_admitted",
                "n_rejected", "n_batch", "adm_ids", "rej_ids", "batch_ids", "n_steps",
                "adm_rec")], kc, *[self._log[k].data_ptr() for k in (
                "skip_now", "skip_target", "skip_waiting", "n_skips")])

    def launch(self, stream=None) -> None:
        """One sl_run_batch on `stream` (default: torch's current stream)."""
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = N.lib().sl_run_batch_ex(
            C.byref(self.st), self._sims.data_ptr(), self._order.data_ptr(), self.n_sims,
            self._ws.data_ptr(), self.total_slots, self._res.data_ptr(),
            C.byref(self.oc) if self.oc is not None else None,
            C.byref(self.lg) if self.lg is not None else None, self.mode, s.cuda_stream)
        if rc != 0:
            raise RuntimeError(f"sl_run_batch failed with code {rc}")

    def results(self) -> np.ndarray:
        """Per-sim result rows (host, sl_result dtype); synchronizes."""
        torch = self.torch
        # through a pinned staging buffer (torch's caching host allocator): one
        # DMA on the current stream instead of a pageable copy
        host = torch.empty(self._res.numel(), dtype=torch.uint8, pin_memory=True)
        host.copy_(self._res, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return host.numpy().view(N.RESULT_DTYPE).copy()

    def results_device(self):
        return self._res

    def report(self, traces: list[TraceArrays] | None = None, n_categories: int | None = None):
        """RunReport reductions per cell on the device (sl_report_batch, one launch):
        returns (rows, cat_counts) -- rows: REPORT_DTYPE (nearest-rank p50/p90/p99
        of TTFT in s and TPOT in ms over completed requests, first index of each
        status); cat_counts: [n_sims, n_categories, 2] (total, compliant) per
        request category, the categories taken from `traces`
        (TraceArrays.category), else all 0.  `n_categories` defaults to
        max(category) + 1; a category outside [0, n_categories) or above 127
        raises (nothing is dropped silently)."""
        if not self.has_outcomes:
            raise RuntimeError("engine built without outcomes")
        torch = self.torch
        cat = None
        hi = 0
        if traces is not None:
            c = np.concatenate([np.asarray(t.category) for t in traces]) if traces else \
                np.zeros(0, np.int8)
            if len(c) and (c.min() < 0 or c.max() > 127):
                raise ValueError("request categories must lie in [0, 127] for the device report")
            hi = int(c.max()) + 1 if len(c) else 0
            cat = torch.from_numpy(np.ascontiguousarray(c, np.int8)).to(self.device)
        if n_categories is None:
            n_categories = max(hi, 1)
        elif hi > n_categories:
            raise ValueError(f"category {hi - 1} outside [0, {n_categories})")
        rows = torch.empty(max(self.n_sims, 1) * N.REPORT_DTYPE.itemsize, dtype=torch.uint8,
                           device=self.device)
        counts = torch.zeros(max(self.n_sims * n_categories * 2, 1), dtype=torch.int64,
                             device=self.device)
        rc = N.lib().sl_report_batch(
            C.byref(self.st), self._sims.data_ptr(), self.n_sims, C.byref(self.oc),
            cat.data_ptr() if cat is not None else None, n_categories, rows.data_ptr(),
            counts.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream)
        if rc != 0:
            raise RuntimeError(f"sl_report_batch failed with code {rc}")
        r = rows.cpu().numpy().view(N.REPORT_DTYPE)[: self.n_sims].copy()
        return r, counts.cpu().numpy()[: self.n_sims * n_categories * 2].reshape(
            self.n_sims, n_categories, 2)

    def cumulative(self) -> list[np.ndarray]:
        """Cumulative SLO-met series per cell on the device (sl_cumulative_batch):
        the ascending completion times of the compliant requests; point i of the
        reference series (report.py:92) is (times[i], i + 1)."""
        if not self.has_outcomes:
            raise RuntimeError("engine built without outcomes")
        torch = self.torch
        slots = max(self.total_slots, 1)
        times = torch.empty(slots, dtype=torch.float64, device=self.device)
        scratch = torch.empty(slots, dtype=torch.int64, device=self.device)
        n_out = torch.empty(max(self.n_sims, 1), dtype=torch.int64, device=self.device)
        rc = N.lib().sl_cumulative_batch(
            C.byref(self.st), self._sims.data_ptr(), self.n_sims, C.byref(self.oc),
            times.data_ptr(), scratch.data_ptr(), n_out.data_ptr(),
            torch.cuda.current_stream(self.device).cuda_stream)
        if rc != 0:
            raise RuntimeError(f"sl_cumulative_batch failed with code {rc}")
        t, cnt = times.cpu().numpy(), n_out.cpu().numpy()
        return [t[int(s["out_offset"]):int(s["out_offset"]) + int(cnt[k])].copy()
                if cnt[k] >= 0 else np.zeros(0) for k, s in enumerate(self.sims_host)]

    def outcomes(self) -> dict[str, np.ndarray]:
        if not self.has_outcomes:
            raise RuntimeError("engine built without outcomes")
        return {k: v[: self.total_slots].cpu().numpy() for k, v in self._out.items()}

    def cell_outcomes(self, k: int) -> dict[str, np.ndarray]:
        """Outcome arrays of cell k, copied from the device slice alone."""
        if not self.has_outcomes:
            raise RuntimeError("engine built without outcomes")
        s = self.sims_host[k]
        b = int(s["out_offset"])
        n = int(self.trace_begin[s["trace"] + 1] - self.trace_begin[s["trace"]])
        return {f: v[b:b + n].cpu().numpy() for f, v in self._out.items()}

    def sim_outcomes(self, k: int, all_out: dict | None = None) -> dict[str, np.ndarray]:
        """Outcome arrays of cell k (slices of outcomes())."""
        all_out = all_out if all_out is not None else self.outcomes()
        s = self.sims_host[k]
        b = int(s["out_offset"])
        n = int(self.trace_begin[s["trace"] + 1] - self.trace_begin[s["trace"]])
        return {f: v[b:b + n] for f, v in all_out.items()}

    def log(self, k: int) -> dict:
        """Decision log of cell k (must have a log slot)."""
        row = int(self.sims_host[k]["log_slot"])
        if row < 0 or self.lg is None:
            raise RuntimeError("cell has no log slot")
        rows, sc, ic, kc = self.log_shape
        ns = int(self._log["n_steps"][row].item())
        out = {f: self._log[f][row * sc: row * sc + ns].cpu().numpy() for f in (
            "now", "end", "prefill_s", "decode_s", "vbs", "min_slo", "n_admitted", "n_rejected",
            "n_batch")}
        na, nr, nb = (int(out[f].sum()) for f in ("n_admitted", "n_rejected", "n_batch"))
        out["adm_ids"] = self._log["adm_ids"][row * ic: row * ic + na].cpu().numpy()
        out["rej_ids"] = self._log["rej_ids"][row * ic: row * ic + nr].cpu().numpy()
        out["batch_ids"] = self._log["batch_ids"][row * ic: row * ic + nb].cpu().numpy()
        out["adm_rec"] = self._log["adm_rec"][5 * row * ic: 5 * (row * ic + na)].cpu().numpy(
        ).reshape(-1, 5)
        nk = int(self._log["n_skips"][row].item())
        out["skips"] = (self._log["skip_now"][row * kc: row * kc + nk].cpu().numpy(),
                        self._log["skip_target"][row * kc: row * kc + nk].cpu().numpy(),
                        self._log["skip_waiting"][row * kc: row * kc + nk].cpu().numpy())
        return out


def default_order(traces: list[TraceArrays], sims: np.ndarray) -> np.ndarray:
    """Longest-expected-first schedule: sims with the lowest arrival rate have the
    longest step chains, so they start first."""
    if len(sims) == 0:
        return np.zeros(0, np.int32)
    meta = _meta(traces)
    n_tr = meta.lens.astype(np.float64)
    last = meta.last
    ti = sims["trace"].astype(np.int64)
    span = last[ti] / sims["rate_factor"]
    with np.errstate(divide="ignore", invalid="ignore"):
        rate = np.where(span > 0, n_tr[ti] / np.where(span > 0, span, 1.0), np.inf)
    # low rate first; ties by larger trace first
    key = np.lexsort((-n_tr[ti], rate))
    return key.astype(np.int32)


def run_batch(traces: list[TraceArrays], cells: list[Cell], outcomes: bool = False,
              log_cells: list[int] | None = None, log_steps: int = 0, log_ids: int = 0,
              mode: int = N.MODE_AUTO):
    """Convenience: build, launch, and return (results, engine)."""
    eng = BatchEngine(traces, cells, outcomes=outcomes, log_cells=log_cells,
                      log_steps=log_steps, log_ids=log_ids, mode=mode)
    eng.launch()
    return eng.results(), eng
