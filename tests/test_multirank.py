"""CPU (gloo, world_size 2) coverage of bench.py's N>1 path: whole-job
aggregation (time = max over ranks, work = sum) and the per-rank independent
soundings (weak scaling: every rank a valid, distinct transmitter)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    times, work = bench.reduce_job([10.0 + rank, 3.0 * (rank + 1)], [100 * (rank + 1)])
    out[rank] = (times, work)
    dist.destroy_process_group()


def test_reduce_job_gloo_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        times, work = out[r]
        assert times == [11.0, 6.0]          # max over ranks
        assert work == [300]                 # sum over ranks


def test_reduce_job_single_process_is_identity():
    import bench
    assert bench.reduce_job([1.5, 2.5], [7]) == ([1.5, 2.5], [7])


@pytest.mark.parametrize("name", ["tiny", "block", "large"])
def test_rank_soundings_valid_and_distinct(name):
    import bench
    from oracle import yee
    seen = set()
    for rank in range(8 if name != "tiny" else 2):
        wl = bench._workload_for_rank(name, rank)
        key = tuple(sorted(wl.source))
        assert key not in seen
        seen.add(key)
        if name != "large":
            asm = yee.assemble(wl)
            G = yee.gradient(wl.grid)
            assert np.abs(G.T @ asm.f_full).max() == 0.0        # closed loop
            assert np.count_nonzero(asm.f) == len(wl.source)     # all interior
        nx, ny, nz = wl.grid.shape
        for (c, i, j, k, s) in wl.source:
            assert 1 <= j <= ny - 1 and k == wl.surface_k
            assert 0 <= i < nx


# ---------------------------------------------------------------- shift partition
@pytest.mark.parametrize("S,world", [(14, 1), (14, 2), (14, 4), (12, 8), (3, 8), (32, 8)])
def test_shard_shifts_is_a_balanced_partition(S, world):
    from paper_2506_11657_b200.distributed import shard_shifts
    rng = np.random.default_rng(S + world)
    shifts = (10 ** rng.uniform(2, 6, S)) * np.exp(1j * rng.uniform(-1.5, 1.5, S))
    parts = shard_shifts(shifts, world)
    assert len(parts) == world
    allidx = np.sort(np.concatenate(parts))
    assert np.array_equal(allidx, np.arange(S))                    # every shift exactly once
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1                             # balanced counts
    if S >= 2 * world:                                              # snake: each rank gets hard and easy
        order = np.argsort(np.abs(shifts))
        hardest = set(order[:world].tolist())
        assert all(len(hardest & set(p.tolist())) == 1 for p in parts)


def _reduce_worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import forward as ofw
    from paper_2506_11657_b200 import RationalTable
    from paper_2506_11657_b200.distributed import reduce_channels, shard_shifts
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    table = RationalTable.load("tiny")
    rng = np.random.default_rng(5)
    X = rng.normal(size=(300, table.n_shift)) + 1j * rng.normal(size=(300, table.n_shift))
    idx = shard_shifts(table.shifts, world)[rank]
    # this rank's partial channel fields (the oracle's synthesis stands in for k_synth)
    up = ofw.synthesize(X[:, idx], table.residues[idx], table.is_pair[idx]).T.copy()
    u = reduce_channels(torch.from_numpy(up), dst=0)
    if rank == 0:
        full = ofw.synthesize(X, table.residues, table.is_pair).T
        out["err"] = float(np.abs(u.numpy() - full).max() / np.abs(full).max())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shift_partitioned_channels_reduce_to_the_full_sum_gloo(world):
    """--partition shifts: per-rank partial sums of eq:rmj over the rank's
    shifts, one reduce -> the full channel fields on rank 0."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_reduce_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out["err"] <= 1e-14
