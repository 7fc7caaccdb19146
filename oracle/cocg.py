"""ORACLE (test infrastructure): per-shift Jacobi-preconditioned COCG.

BASELINE.json's north star lets the oracle use "a per-shift COCG or sparse
direct solve".  The direct LU (oracle.forward.shifted_solves) is exact but its
fill-in makes it minutes per shift beyond ~10^4 unknowns, so mid-size parity
cases use this plain textbook COCG instead -- one shift at a time, CSR matvec,
no fusion, no batching:

    COCG (conjugate orthogonal CG, van der Vorst & Melissen) for complex
    symmetric A = K + s M (A^T = A, §4 "A_i(m) := K - xi_i M"),
    with the unconjugated bilinear form <a, b> = a^T b and the Jacobi
    preconditioner D = diag(A):

        x0 = 0, r0 = f, z0 = D^-1 r0, p0 = z0, rho0 = <r0, z0>
        q = A p; alpha = rho / <p, q>; x += alpha p; r -= alpha q
        stop when ||r||_2 / ||f||_2 <= tol
        z = D^-1 r; rho' = <r, z>; beta = rho'/rho; p = z + beta p

It is pinned against the direct LU on small grids
(tests/test_oracle_forward.py::test_cocg_matches_direct).
"""
from __future__ import annotations

import numpy as np


def cocg(asm, s: complex, tol: float = 1e-12, maxit: int = 200000):
    """Solve (K + s M) x = f; returns (x, iterations, recursive rel. residual)."""
    K, m = asm.K, asm.Mdiag
    f = asm.f.astype(np.complex128)
    D = K.diagonal() + s * m
    x = np.zeros_like(f)
    r = f.copy()
    z = r / D
    p = z.copy()
    rho = r @ z
    nf = np.linalg.norm(f)
    rel = 1.0
    for it in range(1, maxit + 1):
        q = K @ p + s * (m * p)
        alpha = rho / (p @ q)
        x += alpha * p
        r -= alpha * q
        rel = np.linalg.norm(r) / nf
        if rel <= tol:
            return x, it, rel
        z = r / D
        rho_new = r @ z
        p = z + (rho_new / rho) * p
        rho = rho_new
    return x, maxit, rel


def shifted_solves_cocg(asm, shifts, tol: float = 1e-12) -> tuple[np.ndarray, list]:
    """X[:, i] = COCG solution for shift s_i; also returns iteration counts."""
    X = np.zeros((asm.n, len(shifts)), dtype=np.complex128)
    its = []
    for i, s in enumerate(shifts):
        X[:, i], it, _ = cocg(asm, complex(s), tol=tol)
        its.append(it)
    return X, its
