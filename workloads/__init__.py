"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no curl-curl, no mass
assembly, no rational approximation, no solves): only the problem statement
of PAPER.md §2 in the shapes of BASELINE.json's configs -- a tensor-product
grid (cell widths per axis), a conductivity per cell, the transmitter as a
signed list of edges carrying a unit current, the time channels, and the
approximant degree.  Both sides import it; neither side's numerics live here.

Conventions (shared so that both sides agree on what an index means):

* Cells are indexed ``(i, j, k)`` with ``i`` along x (fastest), ``j`` along y,
  ``k`` along z (slowest); z points UP, so the air is the top ``n_air`` cell
  layers and the earth surface is the node plane ``k_s = nz - n_air``.
* Nodes are ``(i, j, k)`` with ``0 <= i <= nx`` etc.  Every node owns three
  edges, one per axis, pointing in the + direction.  Edge ``(c, i, j, k)``
  exists iff its node index along axis ``c`` is ``< n_c``.
* The transmitter is given as ``(c, i, j, k, sign)`` tuples: a unit current
  flowing along edge ``(c, i, j, k)`` in direction ``sign * e_c``.

Configs follow BASELINE.json ``configs[0..4]``; the choices BASELINE leaves
open (padding counts, air thickness, layer depths, body shapes) are recorded
in DESIGN.md "Input recipe".
"""
from .grid import (  # noqa: F401
    TensorGrid,
    padded_axis,
    uniform_axis,
)
from .configs import (  # noqa: F401
    Workload,
    CONFIG_NAMES,
    make_workload,
    loop_source_edges,
    time_channels,
)
