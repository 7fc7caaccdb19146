"""Which shifted systems carry the late-channel error?  For the bench's first
solve (tol 1e-11) and a tight refined reference of the same forward: per
shift s and channel k, C_sk = ||w_s Re(alpha_ks (x_s - xref_s))||_cond /
||u_k||_cond (the shift's share of the channel error, before cancellation
between shifts), and the correction iterations each shift needs.
Experiments only.   python scripts/shift_contrib.py out.json large [hetero ...]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_11657_b200 import RationalTable, TemForward  # noqa: E402
from workloads import make_workload  # noqa: E402

out = {}
for name in sys.argv[2:]:
    wl = make_workload(name)
    table = RationalTable.fit(wl.times, wl.n_poles)
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
    f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
    nx, ny, nz = wl.grid.shape
    kk = np.arange(fw.Nn) // ((nx + 1) * (ny + 1))
    cond = torch.from_numpy(~np.concatenate([kk > wl.surface_k, kk > wl.surface_k, kk >= wl.surface_k])).cuda()
    u1, x1, it1, rr1 = fw.forward(sigma, f, table, opts=fw.opts(tol=1e-11))
    x1 = x1.clone()
    u1n = u1.clone()
    del u1
    ur, xr, itr, rrr = fw.forward(sigma, f, table, opts=fw.opts(tol=1e-11, refine=4, refine_tol=1e-8,
                                                                channel_tol=1e-13, safety=10.0))
    urn = torch.linalg.vector_norm(ur[:, cond], dim=1)
    err = (torch.linalg.vector_norm((u1n - ur)[:, cond], dim=1) / urn).cpu().numpy()
    w = torch.from_numpy(np.where(table.is_pair, 2.0, 1.0)).cuda()
    res = torch.from_numpy(table.residues).cuda()
    C = np.zeros((table.n_shift, res.shape[1]))
    for s in range(table.n_shift):
        e = (x1[s] - xr[s])[cond]
        v = w[s] * (res[s].real[:, None] * e.real[None, :] - res[s].imag[:, None] * e.imag[None, :])
        C[s] = (torch.linalg.vector_norm(v, dim=1) / urn).cpu().numpy()
        del e, v
    # the correction iterations each shift needs for a 1e-4 reduction
    o = fw.opts(tol=1e-11, refine=1, refine_tol=1e-4)
    u2, x2, it2, rr2 = fw.forward(sigma, f, table, opts=o)
    err2 = (torch.linalg.vector_norm((u2 - ur)[:, cond], dim=1) / urn).cpu().numpy()
    rec = {"shifts": [[float(z.real), float(z.imag)] for z in table.shifts],
           "is_pair": table.is_pair.tolist(), "first_iters": it1.tolist(),
           "refined_iters": it2.tolist(), "correction_iters": (it2 - it1).tolist(),
           "first_err_max": float(err.max()), "refined_err_max": float(err2.max()),
           "contrib_max_over_channels": C.max(1).tolist(),
           "contrib_at_worst_channel": C[:, int(err.argmax())].tolist(),
           "worst_channel": int(err.argmax())}
    out[name] = rec
    for s in range(table.n_shift):
        print(name, s, table.shifts[s], "first", int(it1[s]), "corr", int(it2[s] - it1[s]),
              f"contrib max {C[s].max():.2e} at worst ch {C[s, int(err.argmax())]:.2e}", flush=True)
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    del ur, xr, x1, u1n, u2, x2, fw
    torch.cuda.empty_cache()
