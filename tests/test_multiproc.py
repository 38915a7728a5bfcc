"""Sim-sharded sweep plumbing across ranks: rate-balanced
sharding, no data-path collective, one all_gather of fixed-width result rows.
Exercised with world_size=2 on the gloo backend (CPU); the same code path runs
over NCCL on GPUs (bench.py --gpus N)."""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2505_23022_b200 import _native as N
    from paper_2505_23022_b200.sweep import gather_rows, shard_cells

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_cells, n_scales = 12 * 7, 7
    owned = shard_cells(n_cells, n_scales, rank, world)
    rows = np.zeros(len(owned), N.RESULT_DTYPE)
    rows["request_steps"] = owned * 10 + 1  # per-cell payload a rank would compute
    rows["goodput"] = owned / 3.0
    rows["digest"] = owned.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    t = torch.from_numpy(rows.view(np.uint8).copy())
    full = gather_rows(t, owned, n_cells)
    q.put((rank, owned.tolist(), full.tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def test_shards_partition_cells_with_balanced_rates():
    from paper_2505_23022_b200.sweep import shard_cells

    n_rates, n_scales, world = 64, 64 * 4, 4
    parts = [shard_cells(n_rates * n_scales, n_scales, r, world) for r in range(world)]
    allc = np.sort(np.concatenate(parts))
    assert np.array_equal(allc, np.arange(n_rates * n_scales))
    for p in parts:  # every rank sees every rate equally often
        counts = np.bincount(p // n_scales, minlength=n_rates)
        assert counts.min() == counts.max() == n_scales // world


def test_gloo_world2_gather_matches_single_process():
    from paper_2505_23022_b200 import _native as N

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n_cells = 12 * 7
    want = np.zeros(n_cells, N.RESULT_DTYPE)
    ids = np.arange(n_cells)
    want["request_steps"] = ids * 10 + 1
    want["goodput"] = ids / 3.0
    want["digest"] = ids.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    owned = sorted(sum((o for _, o, _ in got), []))
    assert owned == list(range(n_cells))
    for _, _, full in got:  # every rank holds the full, correctly placed table
        assert np.frombuffer(full, N.RESULT_DTYPE).tobytes() == want.tobytes()
