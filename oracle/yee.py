"""ORACLE (test infrastructure): Yee/FIT assembly of K, M, f as CSR.

PAPER.md §2.2 (lines 117-139) defines, for a basis {Phi_1..Phi_N} of the
curl-conforming space with n x e = 0 on the boundary (eq:bc),

    [K]_ij = (mu^-1 curl Phi_j, curl Phi_i),   [M]_ij = (sigma Phi_j, Phi_i),
    [f]_i  = (q, Phi_i),

and the semi-discrete system K u + M u' = 0, M u(0) = f (eq:ode).

BASELINE.json's north star asks for these on "the staggered Yee edge grid".
Reading R1: lowest-order Nedelec elements on the tensor-product
hexahedral grid, degrees of freedom = line integrals of e along the edges,
with both mass matrices lumped (the Yee / finite-integration scheme):

* curl: circulation around each face, (T u)_f = sum of +-u_e over the
  face's 4 edges (Stokes, right-hand rule about the face normal);
* K = T^T W T with W_f = hdual_f / (mu0 * A_f): (1/mu0) |curl e|^2
  integrated over the face's dual cell (area A_f times the distance hdual_f
  between the centres of the two cells sharing the face);
* M_e = (sum over the <=4 cells c touching edge e of sigma_c V_c / 4) / l_e^2:
  sigma |e|^2 integrated over the edge's dual volume, e = u_e / l_e;
* f_e = (q, Phi_e) = +-I for a line current I along edge e (Phi_e has unit
  line integral along e), 0 elsewhere.

Boundary edges (tangential to the domain boundary) are removed (eq:bc), so
K, M, f are returned on the interior ("free") edges only; the ``full``
assembly over every edge is kept for the pins in tests/test_oracle_yee.py.

Everything here is fp64 numpy/scipy.sparse and shares no code with the CUDA
path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

MU0 = 4e-7 * np.pi  # PAPER.md §2.1, "mu = mu_0 = 4 pi x 10^-7 Vs/(Am)"


@dataclass
class EdgeNumbering:
    """Oracle's own edge numbering: all x-edges (C order over [k, j, i]),
    then all y-edges, then all z-edges."""

    nx: int
    ny: int
    nz: int

    def shape(self, c: int) -> tuple[int, int, int]:
        nx, ny, nz = self.nx, self.ny, self.nz
        return [(nz + 1, ny + 1, nx), (nz + 1, ny, nx + 1), (nz, ny + 1, nx + 1)][c]

    def offset(self, c: int) -> int:
        return sum(int(np.prod(self.shape(q))) for q in range(c))

    @property
    def n(self) -> int:
        return self.offset(3)

    def index(self, c: int, i, j, k):
        """Global number of edge (c, i, j, k) -- vectorised over i, j, k."""
        sk, sj, si = self.shape(c)
        return self.offset(c) + (np.asarray(k) * sj + np.asarray(j)) * si + np.asarray(i)

    def keys(self):
        """(c, i, j, k) arrays for all edges, in global order."""
        cs, is_, js, ks = [], [], [], []
        for c in range(3):
            sk, sj, si = self.shape(c)
            k, j, i = np.meshgrid(np.arange(sk), np.arange(sj), np.arange(si), indexing="ij")
            cs.append(np.full(k.size, c))
            is_.append(i.ravel())
            js.append(j.ravel())
            ks.append(k.ravel())
        return (np.concatenate(cs), np.concatenate(is_), np.concatenate(js),
                np.concatenate(ks))

    def interior_mask(self) -> np.ndarray:
        """True for edges not lying in the boundary surface (eq:bc)."""
        c, i, j, k = self.keys()
        n = np.array([self.nx, self.ny, self.nz])
        pos = np.stack([i, j, k])
        inside = np.ones(c.size, dtype=bool)
        for ax in range(3):
            # an edge along axis c lies in the boundary plane normal to ax != c
            # iff its node index along ax is 0 or n_ax
            on_b = (pos[ax] == 0) | (pos[ax] == n[ax])
            inside &= ~((c != ax) & on_b)
        return inside


def _dual_lengths(h: np.ndarray) -> np.ndarray:
    """Distance between neighbouring cell centres at each node plane
    0..n (half a cell at the two boundary planes)."""
    n = len(h)
    d = np.empty(n + 1)
    d[0] = h[0] / 2
    d[n] = h[n - 1] / 2
    d[1:n] = (h[:-1] + h[1:]) / 2
    return d


def curl_incidence(grid):
    """Face-edge incidence T (faces x all edges, entries +-1) and face
    weights W_f = hdual_f / (mu0 A_f).  Faces: normal-x, normal-y, normal-z
    blocks, each C-ordered over [k, j, i] of the face's corner node."""
    hx, hy, hz = grid.hx, grid.hy, grid.hz
    nx, ny, nz = grid.shape
    num = EdgeNumbering(nx, ny, nz)
    dx, dy, dz = _dual_lengths(hx), _dual_lengths(hy), _dual_lengths(hz)
    rows, cols, vals, weights = [], [], [], []
    n_faces = 0

    def add(face_ids, edge_ids, sign):
        rows.append(face_ids)
        cols.append(edge_ids)
        vals.append(np.full(face_ids.size, float(sign)))

    # faces normal to z at node (i, j, k), i < nx, j < ny, 0 <= k <= nz:
    # counter-clockwise about +z: +ex(i,j,k) +ey(i+1,j,k) -ex(i,j+1,k) -ey(i,j,k)
    k, j, i = [a.ravel() for a in np.meshgrid(np.arange(nz + 1), np.arange(ny),
                                              np.arange(nx), indexing="ij")]
    fid = n_faces + np.arange(i.size)
    add(fid, num.index(0, i, j, k), +1)
    add(fid, num.index(1, i + 1, j, k), +1)
    add(fid, num.index(0, i, j + 1, k), -1)
    add(fid, num.index(1, i, j, k), -1)
    weights.append(dz[k] / (MU0 * hx[i] * hy[j]))
    n_faces += i.size

    # faces normal to x at node (i, j, k), 0 <= i <= nx, j < ny, k < nz:
    # counter-clockwise about +x (y then z): +ey(i,j,k) +ez(i,j+1,k) -ey(i,j,k+1) -ez(i,j,k)
    k, j, i = [a.ravel() for a in np.meshgrid(np.arange(nz), np.arange(ny),
                                              np.arange(nx + 1), indexing="ij")]
    fid = n_faces + np.arange(i.size)
    add(fid, num.index(1, i, j, k), +1)
    add(fid, num.index(2, i, j + 1, k), +1)
    add(fid, num.index(1, i, j, k + 1), -1)
    add(fid, num.index(2, i, j, k), -1)
    weights.append(dx[i] / (MU0 * hy[j] * hz[k]))
    n_faces += i.size

    # faces normal to y at node (i, j, k), i < nx, 0 <= j <= ny, k < nz:
    # counter-clockwise about +y (z then x): +ez(i,j,k) +ex(i,j,k+1) -ez(i+1,j,k) -ex(i,j,k)
    k, j, i = [a.ravel() for a in np.meshgrid(np.arange(nz), np.arange(ny + 1),
                                              np.arange(nx), indexing="ij")]
    fid = n_faces + np.arange(i.size)
    add(fid, num.index(2, i, j, k), +1)
    add(fid, num.index(0, i, j, k + 1), +1)
    add(fid, num.index(2, i + 1, j, k), -1)
    add(fid, num.index(0, i, j, k), -1)
    weights.append(dy[j] / (MU0 * hz[k] * hx[i]))
    n_faces += i.size

    T = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n_faces, num.n))
    return T, np.concatenate(weights), num


def edge_mass(grid, sigma: np.ndarray) -> np.ndarray:
    """Lumped M_e over all edges: (sum_{cells c touching e} sigma_c V_c / 4) / l_e^2.
    ``sigma`` is (nz, ny, nx)."""
    hx, hy, hz = grid.hx, grid.hy, grid.hz
    nx, ny, nz = grid.shape
    num = EdgeNumbering(nx, ny, nz)
    vol = hz[:, None, None] * hy[None, :, None] * hx[None, None, :]
    q = sigma * vol / 4.0                       # quarter of each cell's sigma*V
    M = np.zeros(num.n)
    c, i, j, k = num.keys()
    lengths = np.where(c == 0, hx[np.minimum(i, nx - 1)],
                       np.where(c == 1, hy[np.minimum(j, ny - 1)], hz[np.minimum(k, nz - 1)]))
    # each cell (ci, cj, ck) touches 4 x-edges (ci, cj+a, ck+b), 4 y-edges, 4 z-edges
    ck, cj, ci = [a.ravel() for a in np.meshgrid(np.arange(nz), np.arange(ny),
                                                 np.arange(nx), indexing="ij")]
    qv = q.ravel()
    for a in (0, 1):
        for b in (0, 1):
            np.add.at(M, num.index(0, ci, cj + a, ck + b), qv)
            np.add.at(M, num.index(1, ci + a, cj, ck + b), qv)
            np.add.at(M, num.index(2, ci + a, cj + b, ck), qv)
    return M / lengths ** 2


def source_vector(grid, source_edges, current: float = 1.0) -> np.ndarray:
    """f over all edges: +-I on the transmitter's edges ((q, Phi_e), R1)."""
    nx, ny, nz = grid.shape
    num = EdgeNumbering(nx, ny, nz)
    f = np.zeros(num.n)
    for (c, i, j, k, s) in source_edges:
        f[num.index(c, i, j, k)] += s * current
    return f


@dataclass
class Assembly:
    """K, M, f on the free edges plus what is needed to map back."""

    K: sp.csr_matrix          # (N, N) real symmetric PSD
    Mdiag: np.ndarray         # (N,) > 0
    f: np.ndarray             # (N,)
    free: np.ndarray          # (N,) global edge numbers of the free edges
    numbering: EdgeNumbering
    T: sp.csr_matrix          # full face-edge incidence (all edges)
    W: np.ndarray             # face weights
    M_full: np.ndarray        # lumped mass over all edges
    f_full: np.ndarray

    @property
    def n(self) -> int:
        return self.free.size

    def keys(self):
        """(c, i, j, k) of each free edge, in oracle order."""
        c, i, j, k = self.numbering.keys()
        return c[self.free], i[self.free], j[self.free], k[self.free]

    def M(self) -> sp.csr_matrix:
        return sp.diags(self.Mdiag).tocsr()

    def shifted(self, s: complex) -> sp.csc_matrix:
        """K + s M (§3.2 A_i = K - xi_i M with s = -xi_i)."""
        return (self.K + s * sp.diags(self.Mdiag)).astype(np.complex128).tocsc()


def assemble(workload) -> Assembly:
    """K = T^T W T, M, f restricted to the interior edges (eq:bc)."""
    grid = workload.grid
    T, W, num = curl_incidence(grid)
    K_full = (T.T @ sp.diags(W) @ T).tocsr()
    M_full = edge_mass(grid, workload.sigma)
    f_full = source_vector(grid, workload.source)
    free = np.flatnonzero(num.interior_mask())
    K = K_full[free][:, free].tocsr()
    K.sort_indices()
    return Assembly(K=K, Mdiag=M_full[free], f=f_full[free], free=free, numbering=num,
                    T=T, W=W, M_full=M_full, f_full=f_full)


def gradient(grid) -> sp.csr_matrix:
    """Node-to-edge incidence G (all edges x all nodes): (G phi)_e =
    phi(head) - phi(tail).  Used only by the pins (curl grad = 0)."""
    nx, ny, nz = grid.shape
    num = EdgeNumbering(nx, ny, nz)

    def node(i, j, k):
        return (k * (ny + 1) + j) * (nx + 1) + i

    rows, cols, vals = [], [], []
    for c in range(3):
        sk, sj, si = num.shape(c)
        k, j, i = [a.ravel() for a in np.meshgrid(np.arange(sk), np.arange(sj),
                                                  np.arange(si), indexing="ij")]
        e = num.index(c, i, j, k)
        di, dj, dk = [(1, 0, 0), (0, 1, 0), (0, 0, 1)][c]
        rows += [e, e]
        cols += [node(i + di, j + dj, k + dk), node(i, j, k)]
        vals += [np.ones(e.size), -np.ones(e.size)]
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(num.n, (nx + 1) * (ny + 1) * (nz + 1)))


def curl_z_observation(grid, U_full, receivers) -> np.ndarray:
    """ORACLE: -d_t b_z at receivers (§5 P:398-404:
    -d_t b_z(r_0, t) = e_z . (curl e)(r_0, t) ~ Q^T(r_0) u(t)).

    Reading R12: on the tensor grid the z-component of curl e is
    constant on each z-normal face and equals the face circulation of the edge
    line integrals divided by the face area, so Q^T u for a receiver in the
    face with lower-corner node (i, j, k) is row (i, j, k) of the z-face block
    of the incidence T, scaled by 1 / (hx_i hy_j).

    U_full: (n_all_edges, K) channel fields in oracle edge order (every edge,
    boundary edges 0); receivers: iterable of (i, j, k).  Returns (R, K)."""
    T, _, num = curl_incidence(grid)
    nx, ny, nz = grid.shape
    rows = []
    scale = []
    for (i, j, k) in receivers:
        if not (0 <= i < nx and 0 <= j < ny and 0 <= k <= nz):
            raise ValueError(f"receiver face ({i}, {j}, {k}) outside the grid")
        rows.append((k * ny + j) * nx + i)        # z-face block comes first in T
        scale.append(1.0 / (grid.hx[i] * grid.hy[j]))
    return (T[rows] @ U_full) * np.asarray(scale)[:, None]
