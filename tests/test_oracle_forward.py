"""Pins for oracle/forward.py and oracle/cocg.py (CPU only).

* diagonal pencil (K = diag(lam), M = I): the evaluation reduces to the
  scalar family r^[j](lam) (closed form)   -> conjugate pairing, 2Re, t_max
* dense expm brute force: 1x1 closed form and t = 0  -> eigendecomposition
* M-norm bound of §3.3 (line 212): ||exp(-tM^-1K)b - r(M^-1K)b||_M <=
  ||b||_M max_x |e^{-tx} - r(x)| on the tiny config and a random ragged grid
* COCG vs direct LU on small grids
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import cocg, forward, rkfit, yee
from workloads import make_workload
from workloads.configs import make_custom


class _DiagPencil:
    def __init__(self, lam, f):
        self.K = sp.diags(lam).tocsr()
        self.Mdiag = np.ones_like(lam)
        self.f = f
        self.n = lam.size

    def shifted(self, s):
        return (self.K + s * sp.identity(self.n)).astype(np.complex128).tocsc()


def test_diagonal_pencil_reduces_to_scalar_family():
    times = np.logspace(-4, -1, 9)
    fam = rkfit.fit_family(times, 14)
    lam = np.logspace(0, 6, 40)
    f = np.linspace(0.5, 2.0, 40)
    U, X, shifts = forward.forward(_DiagPencil(lam, f), fam)
    for j in range(times.size):
        scalar = fam.eval(j, fam.t_max * lam).real
        np.testing.assert_allclose(U[:, j], scalar * f, rtol=1e-10, atol=1e-13)
    # and it approximates exp(-t lam) f within the family's channel error
    errs = rkfit.channel_errors(fam)
    for j in range(times.size):
        assert np.max(np.abs(U[:, j] - np.exp(-times[j] * lam) * f) / f) <= errs[j] * (1 + 1e-9)


def test_expm_dense_scalar_and_t0():
    class One:
        K = sp.csr_matrix(np.array([[2.0]]))
        Mdiag = np.array([1.0])
        f = np.array([3.0])
    E = forward.expm_dense(One, [0.5, 0.0])
    assert E[0, 0] == pytest.approx(3.0 * np.exp(-1.0), rel=1e-14)
    assert E[0, 1] == pytest.approx(3.0, rel=1e-14)
    asm = yee.assemble(make_custom(5, 4, 4))
    E0 = forward.expm_dense(asm, [0.0])[:, 0]
    np.testing.assert_allclose(E0 * asm.Mdiag, asm.f, atol=1e-9 * np.abs(asm.f).max())


@pytest.mark.parametrize("wl", [make_workload("tiny"), make_custom(9, 7, 6, seed=11)],
                         ids=["tiny", "ragged-random-sigma"])
def test_m_norm_bound(wl):
    asm = yee.assemble(wl)
    fam = rkfit.fit_family(wl.times, wl.n_poles)
    U, X, shifts = forward.forward(asm, fam)
    E = forward.expm_dense(asm, wl.times)
    b_M = forward.m_norm(asm, asm.f / asm.Mdiag)
    errs = rkfit.channel_errors(fam)
    for j in range(len(wl.times)):
        err = forward.m_norm(asm, U[:, j] - E[:, j])
        # (1 + 1e-6) for rounding in the dense eigensolver; the bound is not vacuous:
        assert err <= b_M * errs[j] * (1 + 1e-6) + 1e-12 * b_M
    # the early channel carries real signal (not a vacuous comparison of zeros)
    assert forward.m_norm(asm, E[:, 0]) > 10 * b_M * errs[0]


def test_direct_solves_residual():
    wl = make_workload("tiny")
    asm = yee.assemble(wl)
    fam = rkfit.fit_family(wl.times, wl.n_poles)
    p, _, _ = fam.physical()
    X = forward.shifted_solves(asm, -p)
    for i, s in enumerate(-p):
        assert forward.relative_residual(asm, s, X[:, i]) < 1e-13


@pytest.mark.parametrize("wl", [make_workload("tiny"), make_custom(11, 6, 7, seed=2)],
                         ids=["tiny", "ragged"])
def test_cocg_matches_direct(wl):
    """COCG to a tight tolerance reproduces the exact LU solution.  (At loose
    tolerances the error sits in the air's near-null gradient modes,
    sigma = 1e-8: DESIGN.md reading R6.)"""
    asm = yee.assemble(wl)
    fam = rkfit.fit_family(wl.times, wl.n_poles)
    p, _, _ = fam.physical()
    Xd = forward.shifted_solves(asm, -p)
    Xc, its = cocg.shifted_solves_cocg(asm, -p, tol=1e-14)
    for i, s in enumerate(-p):
        assert forward.relative_residual(asm, s, Xc[:, i]) < 1e-13
        rel = np.linalg.norm(Xc[:, i] - Xd[:, i]) / np.linalg.norm(Xd[:, i])
        assert rel < 1e-6
        relM = forward.m_norm(asm, Xc[:, i] - Xd[:, i]) / forward.m_norm(asm, Xd[:, i])
        assert relM < 1e-9
