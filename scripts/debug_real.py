"""Debug driver: one small split solve (tiny table) through the C ABI."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_11657_b200 import RationalTable, TemForward
from workloads import make_workload
wl = make_workload(sys.argv[1] if len(sys.argv) > 1 else "tiny")
table = RationalTable.load(wl.name)
fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
mass = fw.edge_mass(sigma)
x, it, rr = fw.cocg(mass, f, table.shifts, tol=1e-10, maxit=20000)
print("ok", it, rr.max(), fw.stats())
