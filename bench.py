"""Benchmark: Scorpio scheduler request-steps/s on B200 (config 3 / config 5 sweep).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` (N > 1) without torchrun re-launches itself under
`torch.distributed.run` with N ranks (one per GPU, NCCL) and fails loudly when
fewer than N GPUs are visible; under torchrun WORLD_SIZE must equal N.

One "step" = one pass of the hot path over one batch: every simulation cell of
the rank's shard of the config-3 grid (64 request rates x 64 SLO scales of 10k
requests each = 4,096 sims per GPU; N GPUs sweep 4,096*N cells = config 5 at
N=8, weak scaling) run to completion by one sl_run_batch launch, followed by
the NCCL all_gather of the per-sim result rows when N > 1.

metric: request-steps/s, where one request-step = one waiting or running
request at plan_step entry processed by one scheduler iteration of one sim
(SURVEY 8(d)); the device counts them exactly per sim.

`e2e` is the same metric through the public API from host arrays: each step
packs the cell table (pack_cells over the cells' columns), uploads the traces
from a pinned host TraceTable and the cells (BatchEngine), runs the sweep and
reads the result rows back (plus the NCCL gather when N > 1), wall-clock timed
with the device synchronised on both sides.

`--impl reference` times the UNMODIFIED reference (`slosim`, pure Python,
installed in baseline/_ref by tools/install_reference.sh) through its own
`simengine.run` on every host core (multiprocessing.Pool), over a stratified
sample of the same grid's cells with traces from the reference's own
generator; request-steps per cell are counted by the C restatement (oracle/,
parity-pinned) outside the timed region.  Without baseline/_ref it falls back
to the C restatement itself (`kind: port`).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_REQUEST_STEP = 56  # algorithmic bytes per request-step
METRIC = "scheduler request-steps/sec"
UNIT = "request-steps/s"


def peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi style clock/throttle sampling during the timed region (NVML)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self) -> dict:
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def make_grid(args, world: int):
    from paper_2505_23022_b200.sweep import SweepGrid

    rates = tuple(np.linspace(2.0, 32.0, args.rates))
    scales = tuple(np.geomspace(0.5, 2.0, args.scales * world))
    return SweepGrid(rates=rates, scales=scales, n_requests=args.n_requests)


def sample_cells(grid, n_sample: int) -> list[tuple[int, int]]:
    """Stratified (rate, scale) sample across the grid for the CPU baselines."""
    nr, ns = len(grid.rates), len(grid.scales)
    side = max(1, int(round(np.sqrt(n_sample))))
    ri = np.unique(np.linspace(0, nr - 1, side).round().astype(int))
    si = np.unique(np.linspace(0, ns - 1, max(1, n_sample // len(ri))).round().astype(int))
    return [(int(a), int(b)) for a in ri for b in si]


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_label(grid, world: int) -> dict:
    """The workload the metric is quoted on -- identical in both arms."""
    return {"workload": f"config{'5' if world > 1 else '3'}: {len(grid.rates)} rates x "
                        f"{len(grid.scales)} SLO scales sweep, {grid.n_requests} requests/sim",
            "sims": grid.n_cells, "n_requests": grid.n_requests,
            "parallelism": f"sim-sharded x{world}", "l2": "flushed between steps"}


def port_counts(grid, pairs, traces=None) -> dict:
    """Request-steps of each sampled cell, from the C restatement (oracle/,
    parity-pinned to the reference): the reference itself counts nothing."""
    from oracle import oracle as orc

    cfg = grid.config
    params = orc.make_params(itl=cfg.itl, prefill=cfg.prefill)
    traces = traces or {}
    out = {}
    for ri, si in pairs:
        t = traces.get(ri) or grid.trace_for_rate(grid.rates[ri])
        traces[ri] = t
        sc = float(grid.scales[si])
        r = orc.run_sim(t.arrival, t.ttft_slo * sc, t.tpot_slo * sc, t.prompt_len, t.true_out,
                        t.id, t.predicted, params)
        out[(ri, si)] = int(r["summary"]["request_steps"])
    return out


def cpu_port(grid, n_sample: int, budget_s: float, threads: int):
    """Time the C restatement (oracle/) on all host threads over a sample of the
    grid's cells (stratified rate x scale; every cell when n_sample >= cells),
    scheduled longest-first on a thread pool (ctypes drops the GIL per sim).
    Stops submitting new cells once `budget_s` has elapsed.

    Returns (request_steps, seconds, n_cells, cells_desc)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as orc

    if n_sample >= grid.n_cells:
        pairs = [(ri, si) for ri in range(len(grid.rates)) for si in range(len(grid.scales))]
    else:
        pairs = sample_cells(grid, n_sample)
    pairs.sort(key=lambda p: grid.rates[p[0]])  # low rate = most steps first
    cfg = grid.config
    traces = {ri: grid.trace_for_rate(grid.rates[ri]) for ri in sorted({p[0] for p in pairs})}
    params = orc.make_params(itl=cfg.itl, prefill=cfg.prefill)
    orc.lib()
    t0 = time.perf_counter()

    def one(p):
        if time.perf_counter() - t0 > budget_s:
            return None
        t, sc = traces[p[0]], float(grid.scales[p[1]])
        r = orc.run_sim(t.arrival, t.ttft_slo * sc, t.tpot_slo * sc, t.prompt_len, t.true_out,
                        t.id, t.predicted, params)
        return r["summary"]["request_steps"]

    with ThreadPoolExecutor(max_workers=threads) as ex:
        out = [x for x in ex.map(one, pairs) if x is not None]
    dt = time.perf_counter() - t0
    return sum(out), dt, len(out), f"{len(out)} of {grid.n_cells} cells " \
                                   f"(rate x scale), {grid.n_requests} requests each"


# ---- the unmodified reference (slosim, pure Python) in worker processes
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_REF_TRACES: dict = {}


def _ref_init(ref_dir: str, rates: list, n_requests: int) -> None:
    """Worker start-up (outside the timed region): import slosim from
    baseline/_ref and draw the sampled rates' traces with the reference's own
    generator (report.py:167-177 seeds)."""
    sys.path.insert(0, ref_dir)
    import logging

    logging.disable(logging.WARNING)
    from slosim.seeds import derive_seed
    from slosim.workload import LogNormalDist, WorkloadSpec, generate

    for q in rates:
        spec = WorkloadSpec(qps=float(q), duration=1.1 * n_requests / float(q),
                            seed=derive_seed(0, "trace", float(q)),
                            prompt_len_dist=LogNormalDist(5.0, 0.7),
                            output_len_dist=LogNormalDist(4.0, 0.7),
                            category_weights=(1.0,) * 6)
        _REF_TRACES[float(q)] = generate(spec)[:n_requests]


def _ref_ready(_) -> int:
    time.sleep(0.05)
    return os.getpid()


def _ref_cell(task) -> tuple[int, int]:
    """One cell through slosim.simengine.run: the SLO scale multiplies both
    thresholds of every request."""
    q, sc, itl, pre = task
    from slosim.core import Request
    from slosim.costmodel import ItlParams, PrefillParams
    from slosim.predictor import Bucketing, LengthPredictor
    from slosim.sched_baselines import BaselineConfig
    from slosim.simengine import SimConfig, run

    tr = [Request(id=r.id, arrival_time=r.arrival_time, prompt_len=r.prompt_len,
                  true_output_len=r.true_output_len, ttft_slo=r.ttft_slo * sc,
                  tpot_slo=r.tpot_slo * sc, category=r.category) for r in _REF_TRACES[q]]
    cfg = SimConfig(policy="scorpio", itl_params=ItlParams(*itl), prefill_params=PrefillParams(*pre),
                    predictor=LengthPredictor(mode="oracle",
                                              bucketing=Bucketing.equal_width(100, 4096)),
                    baseline=BaselineConfig(max_batch_size=256))
    outcomes, _ = run(tr, cfg)
    return len(outcomes), sum(1 for o in outcomes if o.slo_compliant)


class PythonReference:
    """A process pool (one worker per host core) running the reference over a
    stratified sample of the grid; each `step()` runs the whole sample, cells
    handed out one at a time, lowest rate (longest step chain) first."""

    def __init__(self, grid, cores: int, n_sample: int = 64):
        import multiprocessing as mp

        self.grid, self.cores = grid, cores
        self.pairs = sorted(sample_cells(grid, n_sample), key=lambda p: (p[0], p[1]))
        rates = sorted({float(grid.rates[ri]) for ri, _ in self.pairs})
        self.counts = port_counts(grid, self.pairs)
        self.pool = mp.get_context("spawn").Pool(cores, initializer=_ref_init,
                                                 initargs=(REF_DIR, rates, grid.n_requests))
        # every worker initialised (traces drawn) before any timing: a worker runs
        # tasks only after its initializer, so seeing every pid proves it
        pids: set = set()
        for _ in range(200):
            pids |= set(self.pool.map(_ref_ready, range(4 * cores), chunksize=1))
            if len(pids) >= cores:
                break

    def step(self) -> tuple[int, float]:
        cfg = self.grid.config
        tasks = [(float(self.grid.rates[ri]), float(self.grid.scales[si]), tuple(cfg.itl),
                  tuple(cfg.prefill)) for ri, si in self.pairs]
        t0 = time.perf_counter()
        self.pool.map(_ref_cell, tasks, chunksize=1)
        dt = time.perf_counter() - t0
        return sum(self.counts.values()), dt

    def close(self) -> None:
        self.pool.terminate()
        self.pool.join()


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    world = args.gpus
    grid = make_grid(args, world)
    have_ref = os.path.isdir(os.path.join(REF_DIR, "slosim"))
    steps_rs, steps_dt = [], []
    if have_ref:
        ref = PythonReference(grid, cores, args.ref_sample)
        for it in range(args.warmup + args.steps):
            rs, dt = ref.step()
            if it >= args.warmup:
                steps_rs.append(rs)
                steps_dt.append(dt)
        ref.close()
        kind = "reference"
        desc = (f"slosim.simengine.run (unmodified, baseline/_ref) on {cores} processes: each "
                f"step runs a stratified {len(ref.pairs)}-cell sample of the {grid.n_cells}-cell "
                f"grid (lowest rate first, one cell per task), {grid.n_requests} requests each; "
                f"request-steps per cell counted by the parity-pinned C restatement outside "
                f"the timed region")
    else:  # no reference install: the C restatement (oracle/)
        for it in range(args.warmup + args.steps):
            rs, dt, n, desc = cpu_port(grid, args.cpu_sample, args.ref_budget, cores)
            if it >= args.warmup:
                steps_rs.append(rs)
                steps_dt.append(dt)
        kind = "port"
    value = sum(steps_rs) / sum(steps_dt)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(steps_dt) / len(steps_dt), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64+int64",
            "data": "synthetic (reference workload generator, seeded)",
            "config": config_label(grid, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": desc, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def plan_microbench(dev, peak: float, reps: int = 5) -> dict:
    """Config 2: one batched plan_step over 64k active requests:
    1,024 segments x (32 waiting + 32 running), the 1 x (32,768 + 32,768) stress
    segment, and the primary shape scaled to 4M and 16.8M requests (65,536 and
    262,144 segments), where the kernels are bandwidth- rather than
    launch/latency-bound.  The LDF sort,
    guard+admission scan and credit select kernels are timed separately, and the
    fused single-launch plan step (segments <= 32 waiting) as a whole; each launch
    alone on the stream (enqueued behind a GPU sleep so no host launch overhead
    is timed), L2 flushed before each.  Compulsory bytes (each input read once,
    each output written once): sort 16 B read (arrival, ttft: the deadline key;
    the id is read only on deadline ties) + 4 B written (perm) per waiting item;
    scan 44 B read (perm, arrival, prefill, ttft, tpot, prompt, predicted) + 8 B
    written (status, position) per waiting item, 12 B read (tpot, current
    length) per running item, 40 B written per admitted item (its
    AdmissionRecord inputs) and per segment (counts, vbs, min_slo, fixed-point
    minimum); select 17 B read (tpot, credit, exclude) + 13 B written (credit,
    batch flag, position) per running item; fused = the union without the perm
    round trip (48 + 12 B per waiting item, 21 + 13 B per running item)."""
    import torch

    from paper_2505_23022_b200.plan import PlanBatch
    from paper_2505_23022_b200.snapshot import config2_arrays, config2_plan_arrays_fast, plan_arrays

    itl, pre = (1e-6, 1e-3, 1e-5, 5e-3, 1.1), (0.004, 128.0, 2e-5, 1.5e-3)
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    out = {}
    for name, (S, W, R) in (("primary_1024x(32+32)", (1024, 32, 32)),
                            ("stress_1x(32768+32768)", (1, 32768, 32768)),
                            ("scaled_65536x(32+32)", (65536, 32, 32)),
                            ("scaled_262144x(32+32)", (262144, 32, 32))):
        arrays = (config2_plan_arrays_fast(S, W, R, seed=11) if S > 4096 else
                  plan_arrays(config2_arrays(S, W, R, seed=11)))
        pb = PlanBatch(arrays=arrays, device=dev)
        Wt, Rt = S * W, S * R
        phases = {"sort": lambda: pb.sort(), "scan": lambda: pb.guard_admit(3, itl, pre),
                  "select": lambda: pb.select(3, True)}
        if W <= 32:
            phases["fused"] = lambda: pb.plan(3, itl, pre)
        times = {k: [] for k in phases}
        for it in range(reps + 2):
            for k, fn in phases.items():
                l2.zero_()
                torch.cuda.synchronize()
                torch.cuda._sleep(200_000)  # the launch below is enqueued while this runs
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                torch.cuda.synchronize()
                if it >= 2:
                    times[k].append(e0.elapsed_time(e1) / 1e3)
        # admitted items also write their AdmissionRecord inputs (5 doubles:
        # V, L, min', estimate, threshold -- sched_scorpio.py:254-271)
        n_adm = int(pb.o["seg_counts"].view(-1, 4)[:, 1].sum().item())
        # + 40 B of per-segment results (counts, vbs, min_slo, fixed-point min)
        bytes_ = {"sort": 20 * Wt, "scan": 52 * Wt + 12 * Rt + 40 * n_adm + 40 * S,
                  "select": 30 * Rt, "fused": 60 * Wt + 34 * Rt + 40 * n_adm + 40 * S}
        rows = {}
        for k in phases:
            t = float(np.mean(times[k]))
            rows[k] = {"us": 1e6 * t, "achieved_gbs": bytes_[k] / t / 1e9,
                       "frac": bytes_[k] / t / 1e9 / peak}
        sep = sum(float(np.mean(times[k])) for k in ("sort", "scan", "select"))
        best = min(sep, float(np.mean(times["fused"]))) if "fused" in times else sep
        out[name] = {"request_steps": Wt + Rt, "us_per_step": 1e6 * best,
                     "request_steps_per_s": (Wt + Rt) / best, "kernels": rows}
        del pb
    # the harness floor: a one-element torch kernel timed the same way (behind the
    # sleep, L2 flushed) -- what any single launch costs here before its own work
    x = torch.zeros(1, device=dev)
    floor = []
    for it in range(reps + 2):
        l2.zero_()
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        x.add_(1.0)
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= 2:
            floor.append(e0.elapsed_time(e1) * 1e3)
    out["launch_floor_us"] = float(np.mean(floor))
    return out


def config4_sweep(dev, reps: int = 2) -> dict:
    """Config 4: 16,384 sims = 128 rates (2-32 req/s) x 128 SLO scales
    (0.5-2.0), 10k requests each, ShareGPT-shaped lengths (prompt LogNormal(4.6, 0.9),
    output LogNormal(4.5, 0.9)), with the noisy-bucket length predictor in the loop
    (equal_width(100, 4096), error 0.73, spread 3, seed derive_seed(0, "predictor")):
    the batched predictor kernel (sl_predict_batch, numpy-stream exact) fills every
    trace's predicted lengths on the device, then one sl_run_batch sweeps all cells."""
    import torch

    from paper_2505_23022_b200.batch import BatchEngine, Cell
    from paper_2505_23022_b200.predictor import Bucketing, LengthPredictor
    from paper_2505_23022_b200.seeds import derive_seed
    from paper_2505_23022_b200.sweep import SweepGrid

    grid = SweepGrid(rates=tuple(np.linspace(2.0, 32.0, 128)),
                     scales=tuple(np.geomspace(0.5, 2.0, 128)), prompt=(4.6, 0.9),
                     output=(4.5, 0.9))
    t0 = time.perf_counter()
    traces = [grid.trace_for_rate(q) for q in grid.rates]
    gen_s = time.perf_counter() - t0
    pred = LengthPredictor("noisy_bucket", Bucketing.equal_width(100, 4096), error_prob=0.73,
                           error_spread=3, rng_seed=derive_seed(0, "predictor"))
    ids = torch.from_numpy(np.concatenate([t.id for t in traces])).to(dev)
    tout = torch.from_numpy(np.concatenate([t.true_out for t in traces])).to(dev)
    stream = torch.cuda.current_stream(dev)
    ptimes = []
    for it in range(reps + 1):
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out, _ = pred.predict_device(ids, tout, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        if it:
            ptimes.append(e0.elapsed_time(e1) / 1e3)
    predicted = out.cpu().numpy()
    k = 0
    for t in traces:
        t.predicted = predicted[k: k + len(t)].copy()
        k += len(t)
    cells = [Cell(ri, grid.config, slo_scale=float(sc)) for ri in range(len(grid.rates))
             for sc in grid.scales]
    eng = BatchEngine(traces, cells, device=dev)
    eng.launch(stream)
    torch.cuda.synchronize()
    res = eng.results()
    assert ((res["status"] & 3) == 0).all(), "engine error in a config-4 sim"
    rs = int(res["request_steps"].sum())
    times = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.launch(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t = float(np.mean(times))
    return {"sims": len(cells), "n_requests": grid.n_requests, "request_steps": rs,
            "ms_per_sweep": 1e3 * t, "request_steps_per_s": rs / t,
            "predictor": {"requests": int(len(ids)), "us": 1e6 * float(np.mean(ptimes)),
                          "predictions_per_s": len(ids) / float(np.mean(ptimes))},
            "mean_goodput": float(res["goodput"].mean()), "trace_gen_s": round(gen_s, 2)}


def report_bench(grid, dev, reps: int = 3) -> dict:
    """RunReport on the device for every cell of the config-3 sweep: the sweep with
    per-request outcomes (41M requests), then sl_report_batch (nearest-rank
    percentiles, per-category counts) and sl_cumulative_batch (sorted compliant
    completion times), each timed with CUDA events."""
    import ctypes as C

    import torch

    from paper_2505_23022_b200 import _native as N
    from paper_2505_23022_b200.batch import BatchEngine, Cell

    traces = [grid.trace_for_rate(q) for q in grid.rates]
    cells = [Cell(ri, grid.config, slo_scale=float(sc)) for ri in range(len(grid.rates))
             for sc in grid.scales]
    eng = BatchEngine(traces, cells, outcomes=True, device=dev)
    stream = torch.cuda.current_stream(dev)

    def timed(fn):
        ts = []
        for it in range(reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            if it:
                ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    sweep_ms = timed(lambda: eng.launch(stream))
    cat = torch.from_numpy(np.concatenate([t.category for t in traces]).astype(np.int8)).to(dev)
    rows = torch.empty(len(cells) * N.REPORT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    counts = torch.zeros(len(cells) * 8 * 2, dtype=torch.int64, device=dev)
    times = torch.empty(eng.total_slots, dtype=torch.float64, device=dev)
    scratch = torch.empty(eng.total_slots, dtype=torch.int64, device=dev)
    n_out = torch.empty(len(cells), dtype=torch.int64, device=dev)
    lib = N.lib()

    def rep():
        assert lib.sl_report_batch(C.byref(eng.st), eng._sims.data_ptr(), eng.n_sims,
                                   C.byref(eng.oc), cat.data_ptr(), 8, rows.data_ptr(),
                                   counts.data_ptr(), stream.cuda_stream) == 0

    def cum():
        assert lib.sl_cumulative_batch(C.byref(eng.st), eng._sims.data_ptr(), eng.n_sims,
                                       C.byref(eng.oc), times.data_ptr(), scratch.data_ptr(),
                                       n_out.data_ptr(), stream.cuda_stream) == 0

    rep_ms, cum_ms = timed(rep), timed(cum)
    n_req = int(eng.total_slots)
    return {"sims": len(cells), "requests": n_req, "sweep_with_outcomes_ms": sweep_ms,
            "report_batch_ms": rep_ms, "cumulative_batch_ms": cum_ms,
            "outcome_bytes_read_GBps": {
                # report: status + compliant (2 B) + ttft/tpot (16 B, up to 8 select
                # passes each) + category (1 B); cumulative: compliant + completion time
                "report_1pass": n_req * 19 / (rep_ms * 1e6),
                "cumulative_1pass": n_req * 9 / (cum_ms * 1e6)}}


def baselines_bench(grid, dev) -> dict:
    """the config-3 grid under each reference policy
    (sched_baselines.py greedy / sjf / early_reject and scorpio) on the same
    traces and engine: sweep time, request-steps/s, mean goodput, and the
    per-cell goodput ratio scorpio / baseline (the paper's Fig-4 quantity)."""
    from dataclasses import replace

    import torch

    from paper_2505_23022_b200.batch import BatchEngine, Cell

    traces = [grid.trace_for_rate(q) for q in grid.rates]
    stream = torch.cuda.current_stream(dev)
    out, good = {}, {}
    for pol in ("scorpio", "greedy", "sjf", "early_reject"):
        cfg = replace(grid.config, policy=pol)
        cells = [Cell(ri, cfg, slo_scale=float(sc)) for ri in range(len(grid.rates))
                 for sc in grid.scales]
        eng = BatchEngine(traces, cells, device=dev)
        eng.launch(stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.launch(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        r = eng.results()
        ms = e0.elapsed_time(e1)
        rs = int(r["request_steps"].sum())
        good[pol] = r["goodput"].astype(np.float64)
        out[pol] = {"ms": ms, "request_steps": rs, "request_steps_per_s": rs / (ms / 1e3),
                    "mean_goodput": float(good[pol].mean())}
    for pol in ("greedy", "sjf", "early_reject"):
        ok = good[pol] > 0
        out[pol]["median_goodput_ratio_scorpio_over_this"] = (
            float(np.median(good["scorpio"][ok] / good[pol][ok])) if ok.any() else None)
    return out


def sim_kernel_profile(n_requests: int, cells: int) -> dict | None:
    """The committed ncu capture of the hot sweep kernel for this workload
    (profiles/sim_kernel_ncu.json: DRAM bytes, warp instructions, duration, SM
    clock of one `ncu --set full --clock-control none` launch)."""
    prof = os.path.join(ROOT, "profiles", "sim_kernel_ncu.json")
    if not os.path.exists(prof):
        return None
    p = json.load(open(prof))
    if p.get("n_requests") != n_requests or p.get("cells") != cells:
        return None
    return p


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2505_23022_b200 import _native as N
    from paper_2505_23022_b200.batch import BatchEngine
    from paper_2505_23022_b200.sweep import build_local, gather_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < world:
        sys.exit(f"bench.py: {world} ranks need {world} GPUs, "
                 f"{torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    grid = make_grid(args, world)
    t_setup = time.perf_counter()
    eng, owned, traces = build_local(grid, rank, world, device=dev)
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream(dev)
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def one_step():
        eng.launch(stream)
        if world > 1:
            gather_rows(eng.results_device(), owned, grid.n_cells)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    res = eng.results()
    assert ((res["status"] & 3) == 0).all(), "engine error in a sim"
    local_rs = int(res["request_steps"].sum())

    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            l2.zero_()  # flush L2 between timed iterations
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one_step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    # kernel-only time (for the roofline): the launch alone, same stream
    ktimes = []
    for _ in range(max(1, min(args.steps, 3))):
        l2.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.launch(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ktimes.append(e0.elapsed_time(e1) / 1e3)

    # e2e: the public API from host arrays, every step: pack the cell table,
    # upload traces + cells (BatchEngine), sweep, read the result rows back
    # (+ gather when N > 1); wall clock with the device synchronised both sides
    # inputs as a user holds them: the rank's traces in one pinned host table
    # (TraceTable) and its cells as columns sharing the grid's config
    from paper_2505_23022_b200.batch import CellColumns, TraceTable

    table = TraceTable(traces)
    cl = build_cells(grid, owned, traces)
    cells = CellColumns(np.array([c.trace for c in cl], np.int64),
                        np.array([c.slo_scale for c in cl]), grid.config)
    h2d = sum(getattr(t, k).nbytes for t in traces for k in
              ("arrival", "ttft_slo", "tpot_slo", "prompt_len", "true_out", "predicted", "id"))
    h2d += 8 * (len(traces) + 1) + len(cells) * (N.SIM_DTYPE.itemsize + 4)  # + begin, order
    d2h = len(cells) * N.RESULT_DTYPE.itemsize
    etimes = []
    for it in range(args.warmup + args.steps):
        l2.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e = BatchEngine(table, cells, device=dev)
        e.launch(stream)
        rows = e.results()  # D2H of the result rows (synchronises)
        if world > 1:
            gather_rows(e.results_device(), owned, grid.n_cells)
        torch.cuda.synchronize()
        if it >= args.warmup:
            etimes.append(time.perf_counter() - t0)
        assert int(rows["request_steps"].sum()) == local_rs
        del e

    t_step = float(np.mean(times))
    t_kernel = float(np.mean(ktimes))
    t_e2e = float(np.mean(etimes))
    if world > 1:
        v = torch.tensor([t_step, t_kernel, t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        t_step, t_kernel, t_e2e = (float(x) for x in v.tolist())
        n = torch.tensor([local_rs], dtype=torch.int64, device=dev)
        dist.all_reduce(n)
        total_rs = int(n.item())
    else:
        total_rs = local_rs

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        rs, dt, ncell, desc = cpu_port(grid, args.cpu_sample, args.cpu_budget, threads)
        cpu = {"value": rs / dt, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc,
               "cpu_model": cpu_model()}
        if os.path.isdir(os.path.join(REF_DIR, "slosim")):
            ref = PythonReference(grid, threads, args.ref_sample)
            rrs, rdt = ref.step()
            ref.close()
            cpu["reference_python"] = {
                "value": rrs / rdt, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"a stratified {len(ref.pairs)}-cell sample through "
                          f"slosim.simengine.run (unmodified, baseline/_ref), one cell per task "
                          f"on {threads} processes"}

    if rank == 0:
        peak, src = peaks()
        achieved = local_rs * BYTES_PER_REQUEST_STEP / t_kernel / 1e9
        prof = sim_kernel_profile(args.n_requests, eng.n_sims)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_source": src,
                "bytes_per_unit": BYTES_PER_REQUEST_STEP,
                "kernel": "sl_sim_fast_kernel<hot> (+ WRec pre-pass and 2 handoff launches)",
                "kernel_ms": 1e3 * t_kernel}
        if prof is not None:
            dur = prof["gpu_time_ns"] * 1e-9
            roof["traffic"] = prof["dram_bytes"]
            # measured-DRAM fraction and issue-slot fraction of the same launch
            # (ncu, profiles/sim_kernel_ncu.json): the kernel is issue/latency bound
            roof["dram_frac"] = prof["dram_bytes"] / dur / 1e9 / peak
            roof["issue_frac"] = prof["inst_executed"] / (
                prof["sms"] * 4 * prof["sm_clock_hz"] * dur)
            roof["ncu"] = {k: prof[k] for k in ("inst_executed", "gpu_time_ns", "dram_bytes",
                                                "sm_clock_hz", "source")}
        line = {
            "metric": METRIC, "value": total_rs / t_step, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64+int64", "data": "synthetic (reference workload generator, seeded)",
            "config": config_label(grid, world),
            "workload_detail": {"sims_per_gpu": eng.n_sims, "request_steps": total_rs,
                                "setup_s": round(setup_s, 2)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": total_rs / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * t_e2e,
                    "timed": "pack_cells (cell columns) + BatchEngine upload from the pinned host trace table + sweep + "
                             "result-row read-back (+ gather), wall clock"},
            "gpu_launches": args.steps * N.lib().sl_run_batch_launches(),
            "clocks": clk.summary(),
        }
        if not args.no_plan and world == 1:
            line["config2_plan_step"] = plan_microbench(dev, peak)
        if not args.no_config4 and world == 1:
            line["config4_noisy_predictor_sweep"] = config4_sweep(dev)
        if not args.no_report and world == 1:
            line["run_report_on_device"] = report_bench(grid, dev)
        if not args.no_baselines and world == 1:
            line["baseline_policies"] = baselines_bench(grid, dev)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def build_cells(grid, owned, traces):
    """The Cell list build_local made for this rank (same order)."""
    from paper_2505_23022_b200.batch import Cell

    need = sorted({int(c) // len(grid.scales) for c in owned})
    tix = {ri: k for k, ri in enumerate(need)}
    return [Cell(tix[int(c) // len(grid.scales)], grid.config,
                 slo_scale=float(grid.scales[int(c) % len(grid.scales)])) for c in owned]


def relaunch_distributed(n: int) -> None:
    """`bench.py --gpus N` outside torchrun: N ranks under torch.distributed.run
    (one per GPU, rendezvous on 127.0.0.1), or a loud failure without N GPUs."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n:
        sys.exit(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rates", type=int, default=64)
    ap.add_argument("--scales", type=int, default=64, help="SLO scales per GPU")
    ap.add_argument("--n-requests", type=int, default=10_000)
    ap.add_argument("--cpu-sample", type=int, default=4096,
                    help="cells timed for cpu_baseline (>= grid size: the whole grid)")
    ap.add_argument("--cpu-budget", type=float, default=15.0,
                    help="wall seconds after which the cpu_baseline stops submitting cells")
    ap.add_argument("--ref-budget", type=float, default=12.0,
                    help="wall seconds per --impl reference step (C-port fallback only)")
    ap.add_argument("--ref-sample", type=int, default=32,
                    help="stratified cells the Python reference cycles through")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-plan", action="store_true", help="skip the config-2 plan microbench")
    ap.add_argument("--no-config4", action="store_true",
                    help="skip the config-4 sweep (16k sims, noisy predictor in the loop)")
    ap.add_argument("--no-baselines", action="store_true",
                    help="skip the baseline-policy sweeps (greedy / sjf / early_reject)")
    ap.add_argument("--no-report", action="store_true",
                    help="skip the device RunReport timing (config-3 sweep with outcomes)")
    args = ap.parse_args()
    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args.gpus)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
