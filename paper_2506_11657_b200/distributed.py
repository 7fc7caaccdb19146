"""Shift-partitioned forward over several GPUs (one process per GPU).

PAPER.md §3.2 (eq:rmj and the sentence after it): the shifted systems
(K - xi_i M) x_i = f are independent, and every time channel is the sum
u(t_j) = sum_i w_i Re(alpha_ij x_i) over them.  So the shifts of ONE sounding
can be dealt to the ranks, each rank solves and synthesises its own partial
sum of every channel with the library's kernels, and one collective sums the
partial channel fields (NCCL over NVLink; gloo in the CPU tests).  The sum is
the only exchange of the path.

    idx = shard_shifts(table.shifts, world)[rank]
    u_partial = forward_partial(fw, sigma, f, table, idx)      # rank-local GPU work
    reduce_channels(u_partial, dst=0)                           # u on rank 0

Host logic only: marshalling and torch.distributed plumbing; every numerical
step runs in libtem_b200.so (TemForward).
"""
from __future__ import annotations

import numpy as np
import torch


def shard_shifts(shifts, world: int) -> list[np.ndarray]:
    """Deal the shift indices to `world` ranks.

    COCG on the Jacobi-preconditioned shifted system converges slower the
    closer s is to the origin (the system is then dominated by the curl-curl
    operator's near-null space), so the shifts are sorted by |s| and dealt in
    snake order (0, 1, .., w-1, w-1, .., 0, 0, ..): every rank gets a mix of
    hard and easy systems and at most one more than any other.  Ranks beyond
    the number of shifts get an empty list.  Returns sorted index arrays."""
    s = np.asarray(shifts)
    if world < 1:
        raise ValueError("world must be >= 1")
    order = np.argsort(np.abs(s), kind="stable")
    parts: list[list[int]] = [[] for _ in range(world)]
    for n, i in enumerate(order):
        rnd, pos = divmod(n, world)
        parts[pos if rnd % 2 == 0 else world - 1 - pos].append(int(i))
    return [np.array(sorted(p), dtype=np.int64) for p in parts]


def forward_partial(fw, sigma: torch.Tensor, f: torch.Tensor, table, idx, tol: float = 1e-10,
                    maxit: int = 200000, stream=None, opts=None):
    """This rank's share of the forward: mass, COCG for the shifts `idx`,
    synthesis of their contribution to every channel (tem_forward; with
    `opts` refining, the channel-aware rule measures the corrections against
    this rank's partial channel fields).  Returns (u_partial (K, n_slots) on
    the device, iters, relres); with no shifts the contribution is zero and no
    kernel runs."""
    from .solver import RationalTable
    idx = np.asarray(idx, dtype=np.int64)
    K = table.residues.shape[1]
    if idx.size == 0:
        u = torch.zeros((K, fw.n_slots), dtype=torch.float64, device=fw.device)
        return u, np.zeros(0, np.int32), np.zeros(0)
    sub = RationalTable(table.shifts[idx], table.residues[idx], table.is_pair[idx], table.times)
    u, x, iters, relres = fw.forward(sigma, f, sub, tol=tol, maxit=maxit, stream=stream, opts=opts)
    del x
    return u, iters, relres


def reduce_channels(u_partial: torch.Tensor, dst: int = 0, group=None) -> torch.Tensor:
    """Sum the ranks' partial channel fields onto rank `dst` (in place; on the
    other ranks the tensor's content is unspecified afterwards).  One
    collective: NCCL reduce for CUDA tensors, gloo for CPU tensors."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return u_partial
    dist.reduce(u_partial, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return u_partial
