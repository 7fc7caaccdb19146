"""Cost and accuracy of tem_forward's channel-aware refinement (DESIGN.md
R13) on the BASELINE workloads: per setting the wall time, COCG
shift-iterations, rounds, the library's own bound, and the measured
per-channel error (relative L2 over the conducting edges) against a much
tighter refined reference.  Writes JSON.

    python scripts/accuracy_study.py out.json large [layered ...]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_11657_b200 import RationalTable, TemForward  # noqa: E402
from workloads import make_workload  # noqa: E402


def conducting_mask(fw, wl):
    nx, ny, nz = wl.grid.shape
    k = np.arange(fw.Nn) // ((nx + 1) * (ny + 1))
    ks = wl.surface_k
    return ~np.concatenate([k > ks, k > ks, k >= ks])


SETTINGS = [("default", dict(tol=1e-12, refine=True)),
            ("t12x1", dict(tol=1e-12, refine=1)),
            ("t11eta1e-4x1", dict(tol=1e-11, refine=1, refine_tol=1e-4)),
            ("t10eta1e-5x1", dict(tol=1e-10, refine=1, refine_tol=1e-5)),
            ("t11", dict(tol=1e-11, refine=True)),
            ("t12eta1e-2", dict(tol=1e-12, refine=True, refine_tol=1e-2)),
            ("plain", dict(refine=False)),
            ("plain1e-11", dict(tol=1e-11, refine=False)),
            ("plain1e-12", dict(tol=1e-12, refine=False)),
            ("plain1e-13", dict(tol=1e-13, refine=False)),
            ("plain1e-14", dict(tol=1e-14, refine=False)),
            ("t12eta1e-2x1", dict(tol=1e-12, refine=1, refine_tol=1e-2)),
            ("t12eta1e-3x1", dict(tol=1e-12, refine=1, refine_tol=1e-3)),
            ("t13eta1e-2x1", dict(tol=1e-13, refine=1, refine_tol=1e-2)),
            ("eta1e-2", dict(refine=True, refine_tol=1e-2)),
            ("eta1e-3", dict(refine=True, refine_tol=1e-3)),
            ("eta1e-5", dict(refine=True, refine_tol=1e-5))]
only = os.environ.get("SETTINGS")
if only:
    SETTINGS = [s for s in SETTINGS if s[0] in only.split(",")]

out = {}
for name in sys.argv[2:]:
    wl = make_workload(name)
    table = RationalTable.fit(wl.times, wl.n_poles)
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
    f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
    cond = torch.from_numpy(conducting_mask(fw, wl)).cuda()
    rec = {"unknowns": fw.n_unknowns, "shifts": table.n_shift, "real_shifts": int(np.sum(table.shifts.imag == 0))}
    t0 = time.time()
    o = fw.opts(tol=1e-10, refine=3, refine_tol=1e-8, channel_tol=1e-12, safety=10.0)
    ur, _, it_r, rr_r = fw.forward(sigma, f, table, opts=o)
    torch.cuda.synchronize()
    st = fw.forward_stats()
    rec["reference"] = {"s": time.time() - t0, "stats": st, "relres_dd": rr_r.tolist()}
    urn = torch.linalg.vector_norm(ur[:, cond], dim=1)
    print(name, "reference", json.dumps(rec["reference"]), flush=True)
    for label, kw in SETTINGS:
        torch.cuda.synchronize()
        t0 = time.time()
        kw = dict(kw)
        kw.setdefault("tol", 1e-10)
        u, x, it, rr = fw.forward(sigma, f, table, raise_on_noconv=False, **kw)
        r_dd = fw.residual(fw.edge_mass(sigma), f, table.shifts, x)[1] / float(torch.linalg.vector_norm(f))
        torch.cuda.synchronize()
        dt = time.time() - t0
        st = fw.forward_stats()
        err = (torch.linalg.vector_norm((u - ur)[:, cond], dim=1) / urn).cpu().numpy()
        row = {"s": dt, "stats": st, "iters": it.tolist(), "max_err": float(err.max()),
               "true_relres_dd": r_dd.tolist(),
               "argmax": int(err.argmax()), "n_over_1e-7": int((err > 1e-7).sum()),
               "err_by_channel": err.tolist(), "solver_stats": fw.stats()}
        rec[label] = row
        print(name, label, json.dumps({k: v for k, v in row.items() if k != "err_by_channel"}), flush=True)
        del u, x
        torch.cuda.empty_cache()
    out[name] = rec
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    del ur, fw
    torch.cuda.empty_cache()
