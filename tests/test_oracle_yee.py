"""Pins for oracle/yee.py (CPU only).

Each test checks the assembly against something the mathematics fixes,
chosen so that a plausible slip (a wrong sign in a face circulation, a
transposed index, a wrong dual length, area or cell-volume share) fails one:

* curl grad = 0 exactly (integer incidence)           -> signs and indices of T
* energy of a linear field with constant curl w:
  u^T K u = |w|^2 V / mu0 (FIT is exact for it)         -> face weights W
* energy of a uniform field E: u^T M u = |E|^2 sum sigma_c V_c  -> edge mass
* closed-form spectrum of M^-1 K on a uniform box      -> K and M together
* divergence-free loop source, complex symmetry of K + sM (north star)
"""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import yee
from workloads import TensorGrid, make_workload, padded_axis, uniform_axis
from workloads.configs import make_custom


def _grids():
    return [
        TensorGrid(uniform_axis(4, 10.0), uniform_axis(5, 7.0), uniform_axis(3, 13.0)),
        TensorGrid(padded_axis(9, 25.0, 2, 3, 1.3), padded_axis(7, 20.0, 2, 2, 1.5),
                   padded_axis(8, 30.0, 3, 1, 1.2)),
    ]


@pytest.mark.parametrize("grid", _grids())
def test_curl_grad_is_zero(grid):
    T, _, _ = yee.curl_incidence(grid)
    G = yee.gradient(grid)
    CG = (T @ G).tocoo()
    assert np.all(CG.data == 0) or CG.nnz == 0
    # and T is not trivially zero: every face has exactly 4 entries of +-1
    assert np.all(np.diff(T.indptr) == 4)
    assert set(np.unique(T.data)) == {-1.0, 1.0}


@pytest.mark.parametrize("grid", _grids())
def test_linear_field_curl_energy(grid):
    """e(r) = w x r / 2 has curl e = w; FIT circulations are exact for linear
    fields, so u^T K u = (1/mu0) |w|^2 * volume."""
    rng = np.random.default_rng(3)
    w = rng.normal(size=3)
    T, W, num = yee.curl_incidence(grid)
    xn, yn, zn = grid.node_coords()
    c, i, j, k = num.keys()
    h = [grid.hx, grid.hy, grid.hz]
    nodes = [xn, yn, zn]
    mid = np.stack([nodes[0][i], nodes[1][j], nodes[2][k]], axis=1)
    length = np.empty(c.size)
    for ax in range(3):
        sel = c == ax
        idx = [i, j, k][ax][sel]
        mid[sel, ax] += 0.5 * h[ax][idx]
        length[sel] = h[ax][idx]
    e_mid = 0.5 * np.cross(w, mid)
    u = e_mid[np.arange(c.size), c] * length
    energy = u @ (T.T @ (W * (T @ u)))
    volume = grid.hx.sum() * grid.hy.sum() * grid.hz.sum()
    assert energy == pytest.approx(np.dot(w, w) * volume / yee.MU0, rel=1e-12)


@pytest.mark.parametrize("grid", _grids())
def test_uniform_field_mass_energy(grid):
    rng = np.random.default_rng(4)
    nx, ny, nz = grid.shape
    sigma = 10 ** rng.uniform(-3, 0, size=(nz, ny, nx))
    E = rng.normal(size=3)
    M = yee.edge_mass(grid, sigma)
    num = yee.EdgeNumbering(nx, ny, nz)
    c, i, j, k = num.keys()
    h = [grid.hx, grid.hy, grid.hz]
    length = np.choose(c, [h[0][np.minimum(i, nx - 1)], h[1][np.minimum(j, ny - 1)],
                           h[2][np.minimum(k, nz - 1)]])
    u = E[c] * length
    vol = grid.hz[:, None, None] * grid.hy[None, :, None] * grid.hx[None, None, :]
    assert u @ (M * u) == pytest.approx(np.dot(E, E) * np.sum(sigma * vol), rel=1e-12)


def test_uniform_box_spectrum_closed_form():
    """Uniform sigma on a uniform box (hx, hy, hz differ): the generalised
    eigenvalues of (K, M) on the interior edges are 0 (gradients, one per
    interior node) and (1/(mu0 sigma)) sum_a (4/h_a^2) sin^2(pi p_a / (2 n_a))
    for the discrete divergence-free modes, with multiplicity (number of
    nonzero p_a) - 1."""
    nx, ny, nz = 4, 5, 3
    hx, hy, hz = 10.0, 7.0, 13.0
    sig = 0.02
    g = TensorGrid(uniform_axis(nx, hx), uniform_axis(ny, hy), uniform_axis(nz, hz))

    class W:  # minimal workload
        grid = g
        sigma = np.full((nz, ny, nx), sig)
        source = []
    asm = yee.assemble(W)
    lam = np.sort(sla.eigh(asm.K.toarray(), np.diag(asm.Mdiag), eigvals_only=True))
    expect = [0.0] * ((nx - 1) * (ny - 1) * (nz - 1))
    for p in range(nx):
        for q in range(ny):
            for r in range(nz):
                mult = (p > 0) + (q > 0) + (r > 0) - 1
                val = (4 / hx**2 * np.sin(np.pi * p / (2 * nx)) ** 2
                       + 4 / hy**2 * np.sin(np.pi * q / (2 * ny)) ** 2
                       + 4 / hz**2 * np.sin(np.pi * r / (2 * nz)) ** 2) / (yee.MU0 * sig)
                expect += [val] * max(mult, 0)
    expect = np.sort(expect)
    assert lam.size == expect.size == asm.n
    scale = expect.max()
    np.testing.assert_allclose(lam, expect, rtol=0, atol=1e-9 * scale)


@pytest.mark.parametrize("name", ["tiny", "block"])
def test_source_divergence_free_and_interior(name):
    wl = make_workload(name)
    asm = yee.assemble(wl)
    G = yee.gradient(wl.grid)
    assert np.abs(G.T @ asm.f_full).max() == 0.0
    # every transmitter edge is a free unknown
    assert np.count_nonzero(asm.f) == len(wl.source)


@pytest.mark.parametrize("name", ["tiny", "block"])
def test_shifted_matrix_complex_symmetric(name):
    """north star: 'complex symmetry of K + sM' (A^T = A, A^H != A)."""
    asm = yee.assemble(make_workload(name))
    A = asm.shifted(350.0 - 1200.0j)
    assert abs(A - A.T).max() == 0.0
    assert abs(A - A.conj().T).max() > 0.0
    # K symmetric PSD-ish: diagonal positive on free edges, M > 0
    assert np.all(asm.K.diagonal() > 0) and np.all(asm.Mdiag > 0)


def test_interior_count_matches_grid():
    wl = make_custom(7, 6, 5)
    asm = yee.assemble(wl)
    assert asm.n == wl.grid.n_interior_edges()
    assert asm.numbering.n == wl.grid.n_edges()


def test_curl_z_observation_closed_forms():
    """-d_t b_z = e_z . curl e: a field with constant curl B e_z,
    e = (-B y / 2, B x / 2, c z) (its edge line integrals are exact for a
    linear field), observes B at every face; a gradient field observes 0."""
    from workloads.configs import make_custom
    wl = make_custom(9, 7, 5, seed=4)
    g = wl.grid
    num = yee.EdgeNumbering(*g.shape)
    xs, ys, zs = [np.concatenate([[0.0], np.cumsum(h)]) for h in (g.hx, g.hy, g.hz)]
    c, i, j, k = num.keys()
    B, cz = 2.5, 0.7
    u = np.empty(num.n)
    # x-edge (i,j,k): integral of -B y/2 dx along x at y_j = -B y_j/2 hx_i, etc.
    mx, my, mz = c == 0, c == 1, c == 2
    u[mx] = -0.5 * B * ys[j[mx]] * g.hx[i[mx]]
    u[my] = 0.5 * B * xs[i[my]] * g.hy[j[my]]
    u[mz] = cz * 0.5 * (zs[k[mz] + 1] ** 2 - zs[k[mz]] ** 2)
    recv = [(0, 0, 0), (8, 6, 5), (3, 2, 2), (5, 6, 1)]
    got = yee.curl_z_observation(g, u[:, None], recv)
    np.testing.assert_allclose(got[:, 0], B, rtol=1e-12)
    # gradient of a random node potential: curl-free, observes 0
    G = yee.gradient(g)
    rng = np.random.default_rng(0)
    phi = rng.normal(size=G.shape[1])
    got0 = yee.curl_z_observation(g, (G @ phi)[:, None], recv)
    assert np.abs(got0).max() <= 1e-12 * np.abs(G @ phi).max() / min(g.hx.min(), g.hy.min()) ** 2
    with pytest.raises(ValueError):
        yee.curl_z_observation(g, u[:, None], [(9, 0, 0)])
