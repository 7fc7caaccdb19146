"""Run the oracle's per-shift COCG (oracle/cocg.py, unchanged) for several
shifts in parallel worker processes (test infrastructure).

Workers are spawned (not forked: the parent holds a CUDA context) and each
runs single-threaded BLAS, so that S workers on S cores do not oversubscribe.
"""
from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor
import multiprocessing as mp

import numpy as np


def _one(asm, s, tol, maxit):
    from threadpoolctl import threadpool_limits
    from oracle import cocg as ocg
    with threadpool_limits(1):
        x, it, rel = ocg.cocg(asm, complex(s), tol, maxit)
    return x, it, rel


def cocg_shifts(asm, shifts, tol, maxit=200000):
    """X[:, i] = oracle COCG solution for shifts[i]; (X, iterations)."""
    workers = max(1, min(len(shifts), os.cpu_count() or 1))
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
        futs = [ex.submit(_one, asm, complex(s), tol, maxit) for s in shifts]
        res = [fu.result() for fu in futs]
    return np.stack([r[0] for r in res], axis=1), [r[1] for r in res]
