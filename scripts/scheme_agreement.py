"""Full-size cross-check of the two COCG schemes (evidence beside the oracle
parity tests, which cannot run at these sizes): per-channel relative L2
difference of the synthesised fields u(t_j), split vs two-sweep, over all
edges and over the conducting (non-air) edges, plus each scheme's max true
residual through the library's own operator.  Writes a JSON summary.

    python scripts/scheme_agreement.py out.json layered hetero large
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_11657_b200 import RationalTable, TemForward  # noqa: E402
from workloads import make_workload  # noqa: E402


def conducting_mask(fw, wl):
    nx, ny, nz = wl.grid.shape
    k = np.arange(fw.Nn) // ((nx + 1) * (ny + 1))
    ks = wl.surface_k
    air = np.concatenate([k > ks, k > ks, k >= ks])   # x, y edges above the surface plane; z edges at/above
    return ~air


out = {}
for name in sys.argv[2:]:
    wl = make_workload(name)
    table = RationalTable.fit(wl.times, wl.n_poles)
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
    f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
    res = {}
    for solver in ("split", "two_sweep"):
        fw.solver = solver
        u, x, iters, relres = fw.forward(sigma, f, table, tol=1e-10, maxit=200000)
        mass = fw.edge_mass(sigma)
        y = fw.apply(mass, table.shifts, x)
        r = y - f.to(torch.complex128).unsqueeze(0)
        true = (r.abs().pow(2).sum(1).sqrt() / f.abs().pow(2).sum().sqrt()).cpu().numpy()
        res[solver] = (u.cpu().numpy(), iters, float(true.max()))
        del u, x, y, r
        torch.cuda.empty_cache()
    ua, ub = res["split"][0], res["two_sweep"][0]
    cond = conducting_mask(fw, wl)
    d_all = np.linalg.norm(ua - ub, axis=1) / np.linalg.norm(ub, axis=1)
    d_con = np.linalg.norm((ua - ub)[:, cond], axis=1) / np.linalg.norm(ub[:, cond], axis=1)
    out[name] = {"unknowns": fw.n_unknowns, "shifts": table.n_shift, "channels": int(ua.shape[0]),
                 "max_rel_l2_all_edges": float(d_all.max()),
                 "max_rel_l2_conducting_edges": float(d_con.max()),
                 "true_residual_max": {"split": res["split"][2], "two_sweep": res["two_sweep"][2]},
                 "iterations_total": {"split": int(np.sum(res["split"][1])),
                                      "two_sweep": int(np.sum(res["two_sweep"][1]))}}
    print(name, json.dumps(out[name]), flush=True)
    del ua, ub, res
json.dump(out, open(sys.argv[1], "w"), indent=1)
