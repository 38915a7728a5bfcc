"""Sharded sweep on the GPU (SURVEY 8(e), config 5 reduced): ranks own
rate-balanced cell shards (sweep.shard_cells), each runs its shard on the
device, the result rows are all-gathered -- and the gathered table must be
bit-identical to the unsharded single-process sweep of the same grid.

Two processes share cuda:0 here (the gpurun lease has one GPU) and gather over
gloo; the NCCL gather runs when two GPUs are visible.  `bench.py --gpus 2`
must refuse to run on fewer than two GPUs rather than silently sweeping one."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _grid(world):
    from paper_2505_23022_b200.core import default_slo_table
    from paper_2505_23022_b200.sweep import SweepGrid

    assert len(default_slo_table().rows) == 6  # heterogeneous 6-category SLO mix
    return SweepGrid(rates=tuple(np.linspace(2.0, 32.0, 6)),
                     scales=tuple(np.geomspace(0.5, 2.0, 4 * world)), n_requests=1500)


def _worker(rank, world, port, backend, q):
    import torch.distributed as dist

    from paper_2505_23022_b200.sweep import build_local, gather_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank if backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    grid = _grid(2)
    eng, owned, _ = build_local(grid, rank, world, device=dev)
    eng.launch()
    torch.cuda.synchronize()
    rows = eng.results_device()
    full = gather_rows(rows if backend == "nccl" else rows.cpu(), owned, grid.n_cells)
    q.put((rank, owned.tolist(), full.tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def _run(backend):
    from paper_2505_23022_b200 import _native as N
    from paper_2505_23022_b200.sweep import build_local

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + os.getpid() % 1000 + (7 if backend == "nccl" else 0)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, backend, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    grid = _grid(2)
    eng, owned, _ = build_local(grid, 0, 1)
    eng.launch()
    want = eng.results()
    assert ((want["status"] & 3) == 0).all()
    assert sorted(sum((o for _, o, _ in got), [])) == list(range(grid.n_cells))
    for _, own, full in got:
        assert len(own) == grid.n_cells // 2
        rows = np.frombuffer(full, N.RESULT_DTYPE)
        assert rows.tobytes() == want.tobytes()  # every field, every cell, bit for bit


def test_sharded_gloo_two_ranks_bit_identical_to_unsharded():
    _run("gloo")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NCCL gather needs 2 GPUs")
def test_sharded_nccl_two_gpus_bit_identical_to_unsharded():
    _run("nccl")


def _nccl_one_rank(port, q):
    import torch.distributed as dist

    from paper_2505_23022_b200.sweep import build_local, gather_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    grid = _grid(1)
    eng, owned, _ = build_local(grid, 0, 1, device=dev)
    eng.launch()
    torch.cuda.synchronize()
    full = gather_rows(eng.results_device(), owned, grid.n_cells)  # NCCL on device tensors
    q.put((full.tobytes(), eng.results().tobytes()))
    dist.destroy_process_group()


def test_gather_rows_over_nccl_on_device_tensors():
    """The NCCL all_gather path of gather_rows (what bench.py runs at N > 1), on the
    one GPU this lease has: a single-rank NCCL group gathers the device rows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_one_rank, args=(32000 + os.getpid() % 1000, q))
    p.start()
    full, want = q.get(timeout=300)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert full == want


def test_bench_refuses_more_gpus_than_visible():
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                        "--steps", "1", "--warmup", "1", "--rates", "2", "--scales", "2",
                        "--n-requests", "200", "--no-cpu", "--no-plan", "--no-config4",
                        "--no-report", "--no-baselines"],
                       capture_output=True, text=True, timeout=300,
                       env={k: v for k, v in os.environ.items() if k not in
                            ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode != 0
    assert f"needs {n} visible GPUs" in r.stderr
    assert '"n_gpus"' not in r.stdout
