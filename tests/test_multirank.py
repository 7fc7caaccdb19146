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
