"""Probe: both COCG schemes on one workload; iterations, true residuals (oracle
CSR for small grids), agreement, and timing.  Experiments only.

    python scripts/probe_solvers.py tiny|ragged|block|large [tol]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_11657_b200 import RationalTable, TemForward  # noqa: E402
from workloads import make_workload  # noqa: E402
from workloads.configs import make_custom  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
fit = name.endswith("-fit")          # e.g. large-fit: the library's own poles, as bench.py
name = name[:-4] if fit else name
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-10
solvers = sys.argv[3].split(",") if len(sys.argv) > 3 else ["two_sweep", "split"]
maxit = int(sys.argv[4]) if len(sys.argv) > 4 else 60000
wl = make_custom(11, 6, 7, seed=2) if name == "ragged" else make_workload(name)
table = RationalTable.load(name) if name != "ragged" else RationalTable.load("tiny")
if fit:
    table = RationalTable.fit(wl.times, wl.n_poles)
fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
mass = fw.edge_mass(sigma)
out = {}
for solver in solvers:
    fw.solver = solver
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, iters, relres = fw.cocg(mass, f, table.shifts, tol=tol, maxit=maxit, raise_on_noconv=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = fw.stats()
    # true residual through the library's own operator
    y = fw.apply(mass, table.shifts, x)
    r = (y - f.to(torch.complex128).unsqueeze(0))
    tr = (r.abs().pow(2).sum(1).sqrt() / f.abs().pow(2).sum().sqrt()).cpu().numpy()
    out[solver] = x
    print(f"{solver:12s} {dt*1e3:9.1f} ms loop {st['loop_ms']:9.1f} ms grid {st['grid']} "
          f"iters {list(map(int, iters))} relres max {relres.max():.2e} true max {tr.max():.2e} "
          f"SUI/s {st['shift_iterations'] * fw.n_unknowns / (st['loop_ms'] * 1e-3):.3e}")
if len(out) < 2:
    sys.exit(0)
a, b = list(out)[:2]
d = (out[a] - out[b]).abs().pow(2).sum(1).sqrt() / out[a].abs().pow(2).sum(1).sqrt()
print("rel diff per shift", d.cpu().numpy())
