"""DRAM traffic of the split passes on a subset of the bench family's shifts
(experiments; run under scripts/launch_list-style ncu metrics).

    python scripts/traffic_probe.py large 0,1,2 [maxit]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_11657_b200 import RationalTable, TemForward  # noqa: E402
from workloads import make_workload  # noqa: E402

name = sys.argv[1]
idx = [int(i) for i in sys.argv[2].split(",")]
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 40
wl = make_workload(name)
table = RationalTable.fit(wl.times, wl.n_poles)
fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
mass = fw.edge_mass(sigma)
shifts = np.ascontiguousarray(table.shifts[idx])
x, iters, relres = fw.cocg(mass, f, shifts, tol=1e-10, maxit=maxit, raise_on_noconv=False)
torch.cuda.synchronize()
st = fw.stats()
print("shifts", shifts, "grid", st["grid"], "N", fw.n_unknowns, "slots", fw.n_slots)
