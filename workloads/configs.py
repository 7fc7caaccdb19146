"""The five synthetic earth models of BASELINE.json ``configs``.

Each is the problem statement of PAPER.md §2 (eq:ivp-eq:source): a
conductivity sigma(r) on a grid, a transmitter q(r) (a loop of unit current
switched off at t=0), the time channels t_1..t_K of PAPER.md §3 ("K time
channels t_1, ..., t_K"), and the degree m-hat of the shared-pole family
(eq:ratfam).  BASELINE.json calls m-hat "poles".

Where BASELINE.json is silent (padding counts, air thickness, layer depths,
body shapes, loop placement) the choice is made here and listed in DESIGN.md
"Input recipe".  Padding: Jacobi-COCG iteration counts grow steeply with the
aspect ratio of stretched cells (measured: DESIGN.md "Input recipe"), so where
BASELINE leaves the padding open it is 6 cells stretching 1.15 per side.  All randomness is seeded numpy ``default_rng``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .grid import TensorGrid, padded_axis, uniform_axis

SIGMA_AIR = 1e-8  # S/m, all configs (BASELINE.json; §5 "10^{-8} S/m")

CONFIG_NAMES = ("tiny", "block", "layered", "hetero", "large")


@dataclass
class Workload:
    name: str
    grid: TensorGrid
    sigma: np.ndarray          # (nz, ny, nx) float64, S/m, C order -> cell (i,j,k) at [k,j,i]
    source: list               # [(c, i, j, k, sign)] unit-current edges (see package doc)
    times: np.ndarray          # (K,) seconds, strictly increasing
    n_poles: int               # degree m-hat of the shared-pole family
    n_air: int                 # number of air cell layers at the top
    notes: dict = field(default_factory=dict)

    @property
    def surface_k(self) -> int:
        return self.grid.shape[2] - self.n_air


def time_channels(tmin: float, tmax: float, k: int) -> np.ndarray:
    """``k`` log-spaced channels in [tmin, tmax] (BASELINE.json wording)."""
    return np.logspace(np.log10(tmin), np.log10(tmax), k)


def loop_source_edges(i0: int, i1: int, j0: int, j1: int, k: int) -> list:
    """Horizontal square loop on node plane ``k`` with corners at nodes
    (i0, j0) and (i1, j1), unit current counter-clockwise seen from +z
    (i.e. magnetic moment along +z).  Returns (c, i, j, k, sign) tuples."""
    if not (i1 > i0 and j1 > j0):
        raise ValueError("loop_source_edges: empty loop")
    edges = []
    edges += [(0, i, j0, k, +1) for i in range(i0, i1)]      # +x along y=j0
    edges += [(1, i1, j, k, +1) for j in range(j0, j1)]      # +y along x=i1
    edges += [(0, i, j1, k, -1) for i in range(i0, i1)]      # -x along y=j1
    edges += [(1, i0, j, k, -1) for j in range(j0, j1)]      # -y along x=i0
    return edges


def _centered_loop(grid: TensorGrid, k_s: int, half_cells: int) -> list:
    nx, ny, _ = grid.shape
    ci, cj = nx // 2, ny // 2
    return loop_source_edges(ci - half_cells, ci + half_cells,
                             cj - half_cells, cj + half_cells, k_s)


def _air(sigma: np.ndarray, n_air: int) -> np.ndarray:
    sigma[sigma.shape[0] - n_air:, :, :] = SIGMA_AIR
    return sigma


def _box3(a: np.ndarray) -> np.ndarray:
    """3x3x3 mean filter with edge replication (BASELINE configs[3])."""
    p = np.pad(a, 1, mode="edge")
    out = np.zeros_like(a)
    nz, ny, nx = a.shape
    for dz in range(3):
        for dy in range(3):
            for dx in range(3):
                out += p[dz:dz + nz, dy:dy + ny, dx:dx + nx]
    return out / 27.0


def _tiny() -> Workload:
    # configs[0]: 8^3 cells of 50 m; top 2 layers air, below 0.01 S/m;
    # VMD at the surface centre (a 2x2-cell loop = 100 m square, moment along z);
    # 16 poles; 31 channels 1e-5..1e-2 s.
    g = TensorGrid(uniform_axis(8, 50.0), uniform_axis(8, 50.0), uniform_axis(8, 50.0))
    n_air = 2
    sigma = _air(np.full((8, 8, 8), 0.01), n_air)
    src = _centered_loop(g, 8 - n_air, 1)
    return Workload("tiny", g, sigma, src, time_channels(1e-5, 1e-2, 31), 16, n_air)


def _block() -> Workload:
    # configs[1]: 32^3 cells, 25 m core, 6 padding cells per side stretching 1.3;
    # air = top 8 layers (6 padding + 2 core); background 0.01 S/m;
    # 8x8x4 block of 1 S/m whose top is 100 m below the surface, centred;
    # 100 m square loop centred on the surface; 16 poles; 41 channels 1e-6..1e-2.
    ax = padded_axis(32, 25.0, 6, 6, 1.3)
    g = TensorGrid(ax.copy(), ax.copy(), ax.copy())
    n_air = 8
    k_s = 32 - n_air
    sigma = np.full((32, 32, 32), 0.01)
    # 100 m = 4 core cells below the surface; block 4 cells thick beneath that
    sigma[k_s - 8:k_s - 4, 12:20, 12:20] = 1.0
    sigma = _air(sigma, n_air)
    src = _centered_loop(g, k_s, 2)
    return Workload("block", g, sigma, src, time_channels(1e-6, 1e-2, 41), 16, n_air)


def _layered() -> Workload:
    # configs[2]: 64^3 cells, 10 m core, 5 padding cells per side stretching 1.25;
    # air = top 12 layers; layers below the surface: 0.05 S/m to 50 m depth,
    # 0.005 S/m to 150 m, 0.2 S/m below; 200 m loop; 20 poles; 61 ch 1e-6..1e-1.
    ax = padded_axis(64, 10.0, 5, 5, 1.25)
    g = TensorGrid(ax.copy(), ax.copy(), ax.copy())
    n_air = 12
    k_s = 64 - n_air
    zn = g.node_coords()[2]
    zc = 0.5 * (zn[:-1] + zn[1:])
    depth = zn[k_s] - zc                       # > 0 below the surface
    prof = np.where(depth < 50.0, 0.05, np.where(depth < 150.0, 0.005, 0.2))
    sigma = np.broadcast_to(prof[:, None, None], (64, 64, 64)).copy()
    sigma = _air(sigma, n_air)
    src = _centered_loop(g, k_s, 10)
    return Workload("layered", g, sigma, src, time_channels(1e-6, 1e-1, 61), 20, n_air)


def _hetero() -> Workload:
    # configs[3]: 128x128x96 cells (~4.7M edges), 20 m core, 6 padding cells per
    # side stretching 1.15; log10 sigma ~ N(-2, 0.5^2) iid per cell (seed 0),
    # smoothed by a 3x3x3 box filter; air 1e-8 in the top 16 cells;
    # 200 m loop; 20 poles; 61 channels 1e-6..1e-1.
    g = TensorGrid(padded_axis(128, 20.0, 6, 6, 1.15),
                   padded_axis(128, 20.0, 6, 6, 1.15),
                   padded_axis(96, 20.0, 6, 6, 1.15))
    n_air = 16
    rng = np.random.default_rng(0)
    lg = rng.normal(-2.0, 0.5, size=(96, 128, 128))
    sigma = _air(10.0 ** _box3(lg), n_air)
    src = _centered_loop(g, 96 - n_air, 5)
    return Workload("hetero", g, sigma, src, time_channels(1e-6, 1e-1, 61), 20, n_air)


def _large() -> Workload:
    # configs[4]: 192x192x128 cells (~14M edges), 20 m core, 6 padding cells
    # per side stretching 1.15; background 0.01 S/m; air 1e-8 in the top 20
    # cells; 5 random axis-aligned ellipsoids (seed 1) of 0.1-1 S/m
    # (log-uniform), centres 60-500 m deep inside the core, semi-axes 40-200 m;
    # 200 m loop; 24 poles; 100 channels 1e-6..1e-1.
    g = TensorGrid(padded_axis(192, 20.0, 6, 6, 1.15),
                   padded_axis(192, 20.0, 6, 6, 1.15),
                   padded_axis(128, 20.0, 6, 6, 1.15))
    n_air = 20
    k_s = 128 - n_air
    sigma = np.full((128, 192, 192), 0.01)
    xc, yc, zc = g.cell_centers()
    xn, yn, zn = g.node_coords()
    z_s = zn[k_s]
    x_mid, y_mid = xn[-1] / 2, yn[-1] / 2
    rng = np.random.default_rng(1)
    bodies = []
    for _ in range(5):
        cx = x_mid + rng.uniform(-800.0, 800.0)
        cy = y_mid + rng.uniform(-800.0, 800.0)
        cz = z_s - rng.uniform(60.0, 500.0)
        ax3 = rng.uniform(40.0, 200.0, size=3)
        s = 10.0 ** rng.uniform(-1.0, 0.0)
        bodies.append((cx, cy, cz, *ax3, s))
        r2 = (((xc[None, None, :] - cx) / ax3[0]) ** 2
              + ((yc[None, :, None] - cy) / ax3[1]) ** 2
              + ((zc[:, None, None] - cz) / ax3[2]) ** 2)
        sigma[r2 <= 1.0] = s
    sigma = _air(sigma, n_air)
    src = _centered_loop(g, k_s, 5)
    return Workload("large", g, sigma, src, time_channels(1e-6, 1e-1, 100), 24, n_air,
                    notes={"bodies": bodies})


_MAKERS = {"tiny": _tiny, "block": _block, "layered": _layered,
           "hetero": _hetero, "large": _large}


def make_workload(name: str) -> Workload:
    """Build one of BASELINE.json's configs by name (see CONFIG_NAMES)."""
    try:
        return _MAKERS[name]()
    except KeyError:
        raise ValueError(f"unknown workload {name!r}; choose from {CONFIG_NAMES}")


def make_custom(nx: int, ny: int, nz: int, h: float = 50.0, n_air: int = 2,
                sigma_earth: float = 0.01, seed: int | None = None,
                times=None, n_poles: int = 16, loop_half: int = 1) -> Workload:
    """Small ragged-shape workloads for parity tests.  With ``seed`` the earth
    conductivity is log-uniform in [1e-3, 1] per cell."""
    g = TensorGrid(uniform_axis(nx, h), uniform_axis(ny, h * 0.8), uniform_axis(nz, h * 1.1))
    if seed is None:
        sigma = np.full((nz, ny, nx), float(sigma_earth))
    else:
        rng = np.random.default_rng(seed)
        sigma = 10.0 ** rng.uniform(-3.0, 0.0, size=(nz, ny, nx))
    sigma = _air(sigma, n_air)
    k_s = nz - n_air
    ci, cj = nx // 2, ny // 2
    i0, i1 = max(ci - loop_half, 1), min(ci + loop_half, nx - 1)
    j0, j1 = max(cj - loop_half, 1), min(cj + loop_half, ny - 1)
    ok = i1 > i0 and j1 > j0 and 1 <= k_s <= nz - 1
    src = loop_source_edges(i0, i1, j0, j1, k_s) if ok else []
    if times is None:
        times = time_channels(1e-5, 1e-2, 31)
    return Workload(f"custom{nx}x{ny}x{nz}", g, sigma, src, np.asarray(times), n_poles, n_air)
