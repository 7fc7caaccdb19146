#!/usr/bin/env python
"""Quick GPU probe: one forward per config, iteration counts and timings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_11657_b200 import RationalTable, TemForward  # noqa: E402
from workloads import make_workload  # noqa: E402


def main(names, tol=1e-10, maxit=200000):
    for name in names:
        t0 = time.time()
        wl = make_workload(name)
        table = RationalTable.load(name)
        fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
        sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
        f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
        t1 = time.time()
        mass = fw.edge_mass(sigma)
        x, iters, relres = fw.cocg(mass, f, table.shifts, tol=tol, maxit=maxit, raise_on_noconv=False)
        torch.cuda.synchronize()
        t2 = time.time()
        st = fw.stats()
        N = fw.n_unknowns
        sui = st["shift_iterations"] * N
        print(f"[{name}] N={N} S={table.n_shift} setup={t1 - t0:.1f}s solve={t2 - t1:.2f}s "
              f"loop_ms={st['loop_ms']:.1f} iters={list(iters)} max={st['iterations']} "
              f"relres_max={relres.max():.2e} grid={st['grid']}x{st['block']} "
              f"SUI/s={sui / (st['loop_ms'] * 1e-3):.3e} "
              f"GB/s@128B={sui * 128 / (st['loop_ms'] * 1e-3) / 1e9:.0f}", flush=True)
        u = fw.synthesize(x, table.residues, table.is_pair)
        torch.cuda.synchronize()
        del x, u, mass
        fw.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["tiny", "block", "layered", "hetero", "large"])
