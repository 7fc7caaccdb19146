"""ORACLE (test infrastructure): evaluation of the shared-pole family on the
pencil (K, M) -- PAPER.md §3.2 eq:rmj and the tall-skinny product S R.

    r^[j](M^-1 K) b = sum_i alpha_i^[j] (K - xi_i M)^-1 f          (line 185)
                    = 2 Re( sum_{i <= m/2} alpha_i^[j] (K - xi_i M)^-1 f )  (eq:rmj)

with b = M^-1 f (eq:expm).  BASELINE.json writes the shifted systems as
(K + s_i M) x_i = M b, i.e. s_i = -xi_i.

* ``shifted_solves``  -- one sparse direct LU (SuperLU via scipy) per
  representative pole: the "per-shift ... sparse direct solve" the north star
  allows for the oracle.  A library primitive, used as one step.
* ``synthesize``      -- u(t_j) = sum_i w_i Re(alpha_i^[j] x_i), w_i = 2 for a
  conjugate-pair representative and 1 for a real pole (footnote, line 187).
* ``expm_dense``      -- brute force exp(-t M^-1 K) b through the generalised
  symmetric eigendecomposition K V = M V Lambda, V^T M V = I (eq:expm).
* ``relative_residual`` -- ||f - (K + s M) x|| / ||f|| for any x (a property
  that holds at any size; used on the GPU's full-size solutions).
* ``m_norm``          -- ||x||_M = sqrt(x^T M x) (§3.3).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse.linalg as spla


def shifted_solves(asm, shifts) -> np.ndarray:
    """X[:, i] = (K + s_i M)^-1 f for each shift s_i (complex); (N, n_shift)."""
    X = np.zeros((asm.n, len(shifts)), dtype=np.complex128)
    rhs = asm.f.astype(np.complex128)
    for i, s in enumerate(shifts):
        lu = spla.splu(asm.shifted(complex(s)))
        X[:, i] = lu.solve(rhs)
    return X


def synthesize(X: np.ndarray, residues: np.ndarray, is_pair) -> np.ndarray:
    """U[:, j] = sum_i w_i Re(alpha_i^[j] X[:, i]) -- the columns of 2 Re(S R)
    (§3.2).  ``residues`` is (n_shift, K)."""
    w = np.where(np.asarray(is_pair, bool), 2.0, 1.0)
    U = np.zeros((X.shape[0], residues.shape[1]))
    for j in range(residues.shape[1]):
        for i in range(X.shape[1]):
            U[:, j] += w[i] * (residues[i, j] * X[:, i]).real
    return U


def forward(asm, family) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """All channels u(t_j) ~ exp(-t_j M^-1 K) b for a fitted family
    (oracle.rkfit.RationalFamily).  Returns (U, X, shifts)."""
    poles_x, res_x, is_pair = family.physical()
    shifts = -poles_x
    X = shifted_solves(asm, shifts)
    return synthesize(X, res_x, is_pair), X, shifts


def expm_dense(asm, times) -> np.ndarray:
    """exp(-t M^-1 K) b, b = M^-1 f, for each t (N small): with K V = M V L,
    V^T M V = I, exp(-t M^-1 K) b = V exp(-t L) V^T M b = V exp(-t L) V^T f."""
    K = asm.K.toarray()
    M = np.diag(asm.Mdiag)
    lam, V = sla.eigh(K, M)
    lam = np.maximum(lam, 0.0)            # K is PSD; clip -eps from rounding
    c = V.T @ asm.f
    return np.stack([V @ (np.exp(-t * lam) * c) for t in times], axis=1)


def relative_residual(asm, s: complex, x: np.ndarray) -> float:
    """||f - (K + s M) x||_2 / ||f||_2 (computed with the oracle's CSR)."""
    r = asm.f - (asm.K @ x + s * (asm.Mdiag * x))
    return float(np.linalg.norm(r) / np.linalg.norm(asm.f))


def m_norm(asm, x: np.ndarray) -> float:
    return float(np.sqrt(np.sum(asm.Mdiag * np.abs(x) ** 2)))
