"""Full-size cross-check of the two COCG schemes (evidence beside the oracle
parity tests, which cannot run at these sizes): per-channel relative L2
difference of the synthesised fields u(t_j), split vs two-sweep, over all
edges, over the conducting (non-air) edges and relative to the summand scale
T_j (R6), plus each scheme's max true
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
    T = None
    for solver in ("split", "two_sweep"):
        fw.solver = solver
        u, x, iters, relres = fw.forward(sigma, f, table, tol=1e-10, maxit=200000)
        mass = fw.edge_mass(sigma)
        y = fw.apply(mass, table.shifts, x)
        r = y - f.to(torch.complex128).unsqueeze(0)
        true = (r.abs().pow(2).sum(1).sqrt() / f.abs().pow(2).sum().sqrt()).cpu().numpy()
        del y, r
        if T is None:   # summand scale T_j = || sum_i w_i |alpha_ij| |x_i| || (reading R6)
            w = torch.tensor(np.where(table.is_pair, 2.0, 1.0), device=x.device)
            C = (w[:, None] * torch.from_numpy(np.abs(table.residues)).to(x.device)).T   # (K, S)
            ax = x.abs()
            T = np.array([torch.linalg.vector_norm(C[j] @ ax).item() for j in range(C.shape[0])])
            del ax
        res[solver] = (u.cpu().numpy(), iters, float(true.max()))
        del u, x
        torch.cuda.empty_cache()
    ua, ub = res["split"][0], res["two_sweep"][0]
    cond = conducting_mask(fw, wl)
    d_all = np.linalg.norm(ua - ub, axis=1) / np.linalg.norm(ub, axis=1)
    d_con = np.linalg.norm((ua - ub)[:, cond], axis=1) / np.linalg.norm(ub[:, cond], axis=1)
    d_term = np.linalg.norm(ua - ub, axis=1) / T
    out[name] = {"unknowns": fw.n_unknowns, "shifts": table.n_shift, "channels": int(ua.shape[0]),
                 "max_rel_l2_all_edges": float(d_all.max()),
                 "max_term_relative_all_edges": float(d_term.max()),
                 "channel_of_max_conducting": int(np.argmax(d_con)),
                 "rel_l2_conducting_by_channel": [float(v) for v in d_con],
                 "max_rel_l2_conducting_edges": float(d_con.max()),
                 "true_residual_max": {"split": res["split"][2], "two_sweep": res["two_sweep"][2]},
                 "iterations_total": {"split": int(np.sum(res["split"][1])),
                                      "two_sweep": int(np.sum(res["two_sweep"][1]))}}
    print(name, json.dumps(out[name]), flush=True)
    del ua, ub, res
json.dump(out, open(sys.argv[1], "w"), indent=1)
