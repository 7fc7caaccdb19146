"""Tensor-product grid description (cell widths only; no discretisation).

A grid is three 1-D arrays of cell widths.  Padding is geometric: the
``n_pad`` outermost cells on a side grow by ``stretch`` per cell away from the
core, i.e. widths ``h * stretch**1, ..., h * stretch**n_pad``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def uniform_axis(n: int, h: float) -> np.ndarray:
    """``n`` cells of width ``h``."""
    if n < 1 or not h > 0:
        raise ValueError("uniform_axis: need n >= 1 and h > 0")
    return np.full(n, float(h))


def padded_axis(n_total: int, h: float, n_pad_lo: int, n_pad_hi: int,
                stretch: float) -> np.ndarray:
    """``n_total`` cells: ``n_pad_lo`` stretched cells, a uniform core of
    width ``h``, ``n_pad_hi`` stretched cells.  Widths grow outward."""
    n_core = n_total - n_pad_lo - n_pad_hi
    if n_core < 1:
        raise ValueError("padded_axis: padding leaves no core cells")
    lo = h * stretch ** np.arange(n_pad_lo, 0, -1, dtype=np.float64)
    hi = h * stretch ** np.arange(1, n_pad_hi + 1, dtype=np.float64)
    return np.concatenate([lo, np.full(n_core, float(h)), hi])


@dataclass(frozen=True)
class TensorGrid:
    """Cell widths along x, y, z (metres).  ``z`` points up."""

    hx: np.ndarray
    hy: np.ndarray
    hz: np.ndarray

    @property
    def shape(self) -> tuple[int, int, int]:
        """(nx, ny, nz) cell counts."""
        return (len(self.hx), len(self.hy), len(self.hz))

    @property
    def n_nodes(self) -> int:
        nx, ny, nz = self.shape
        return (nx + 1) * (ny + 1) * (nz + 1)

    def n_edges(self) -> int:
        """All edges, including those on the boundary."""
        nx, ny, nz = self.shape
        return (nx * (ny + 1) * (nz + 1) + (nx + 1) * ny * (nz + 1)
                + (nx + 1) * (ny + 1) * nz)

    def n_interior_edges(self) -> int:
        """Edges not lying in the boundary surface (the free unknowns under
        n x e = 0, §2.1 eq:bc)."""
        nx, ny, nz = self.shape
        return (nx * (ny - 1) * (nz - 1) + (nx - 1) * ny * (nz - 1)
                + (nx - 1) * (ny - 1) * nz)

    def node_coords(self):
        """Node coordinates per axis, origin at the grid's lower corner."""
        return tuple(np.concatenate([[0.0], np.cumsum(h)])
                     for h in (self.hx, self.hy, self.hz))

    def cell_centers(self):
        return tuple(np.cumsum(h) - 0.5 * h for h in (self.hx, self.hy, self.hz))
