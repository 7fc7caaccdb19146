#!/usr/bin/env python
"""Probe the large config: per-chunk progress of the COCG (host-side maxit slices)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_11657_b200 import RationalTable, TemForward
from workloads import make_workload
name = sys.argv[1] if len(sys.argv) > 1 else "large"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
wl = make_workload(name)
table = RationalTable.fit(wl.times, wl.n_poles) if os.environ.get("POLES") == "fit" else RationalTable.load(name)
fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
mass = fw.edge_mass(sigma)
t = time.time()
x, iters, relres = fw.cocg(mass, f, table.shifts, tol=1e-10, maxit=budget, raise_on_noconv=False)
torch.cuda.synchronize()
st = fw.stats()
N = fw.n_unknowns
print(f"[{name}] budget={budget} wall={time.time()-t:.1f}s loop_ms={st['loop_ms']:.0f} iters={list(map(int,iters))}")
print("relres", " ".join(f"{r:.1e}" for r in relres))
print(f"ms/iter={st['loop_ms']/max(st['iterations'],1):.2f} SUI/s={st['shift_iterations']*N/(st['loop_ms']*1e-3):.3e} GB/s@128={st['shift_iterations']*N*128/(st['loop_ms']*1e-3)/1e9:.0f}")
