"""How tight must the COCG solves be for the channel fields to meet the
north-star bar (relative L2 <= 1e-7 at every channel, conducting edges,
reading R6)?  For each workload: a tight reference solve, then solves at a
ladder of tolerances; per channel the relative L2 error against the
reference, per shift its contribution to each channel's error, iteration
counts and true residuals (library operator).  Writes a JSON summary.

    python scripts/tol_study.py out.json block layered hetero large
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
    air = np.concatenate([k > ks, k > ks, k >= ks])
    return ~air


def true_res(fw, mass, shifts, x, f):
    y = fw.apply(mass, shifts, x)
    y -= f.to(torch.complex128).unsqueeze(0)
    r = (y.abs().pow(2).sum(1).sqrt() / f.abs().pow(2).sum().sqrt()).cpu().numpy()
    del y
    return r


def chan_norms(fw, x, table, cond):
    u = fw.synthesize(x, table.residues, table.is_pair)
    return u


out = {}
tols = [float(t) for t in os.environ.get("TOLS", "1e-10,1e-11,1e-12,1e-13").split(",")]
ref_tol = float(os.environ.get("REF_TOL", "1e-14"))
for name in sys.argv[2:]:
    wl = make_workload(name)
    table = RationalTable.fit(wl.times, wl.n_poles)
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
    f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
    mass = fw.edge_mass(sigma)
    cond = torch.from_numpy(conducting_mask(fw, wl)).cuda()
    w = np.where(table.is_pair, 2.0, 1.0)
    rec = {"unknowns": fw.n_unknowns, "shifts": table.n_shift, "channels": int(table.residues.shape[1]),
           "shift_values": [[float(s.real), float(s.imag)] for s in table.shifts]}
    t0 = time.time()
    xr, it_r, rr_r = fw.cocg(mass, f, table.shifts, tol=ref_tol, maxit=60000, raise_on_noconv=False)
    torch.cuda.synchronize()
    rec["ref"] = {"tol": ref_tol, "iters": it_r.tolist(), "relres": rr_r.tolist(),
                  "true_res": true_res(fw, mass, table.shifts, xr, f).tolist(), "s": time.time() - t0}
    ur = fw.synthesize(xr, table.residues, table.is_pair)
    urn = torch.linalg.vector_norm(ur[:, cond], dim=1)
    rec["ref"]["u_norm_cond"] = urn.cpu().numpy().tolist()
    print(name, "ref", json.dumps({k: v for k, v in rec["ref"].items() if k != "u_norm_cond"}), flush=True)
    rec["ladder"] = []
    for tol in tols:
        t0 = time.time()
        x, it, rr = fw.cocg(mass, f, table.shifts, tol=tol, maxit=60000, raise_on_noconv=False)
        torch.cuda.synchronize()
        dt = time.time() - t0
        tr = true_res(fw, mass, table.shifts, x, f)
        u = fw.synthesize(x, table.residues, table.is_pair)
        err = (torch.linalg.vector_norm((u - ur)[:, cond], dim=1) / urn).cpu().numpy()
        del u
        # per-shift contributions C[i, k] = || w_i Re(alpha_ik e_i) ||_cond / ||u_k||_cond
        e = (x - xr)[:, cond]
        a2 = e.real.pow(2).sum(1)
        b2 = e.imag.pow(2).sum(1)
        ab = (e.real * e.imag).sum(1)
        del e
        res = torch.from_numpy(table.residues).cuda()          # (S, K)
        ar, ai = res.real, res.imag
        contrib = (torch.from_numpy(w).cuda()[:, None]
                   * (ar.pow(2) * a2[:, None] + ai.pow(2) * b2[:, None] - 2 * ar * ai * ab[:, None]).clamp_min(0).sqrt())
        contrib = (contrib / urn[None, :]).cpu().numpy()
        xrel = (torch.linalg.vector_norm((x - xr), dim=1) / torch.linalg.vector_norm(xr, dim=1)).cpu().numpy()
        row = {"tol": tol, "iters": it.tolist(), "iters_total": int(it.sum()), "s": dt,
               "true_res_max": float(tr.max()), "true_res": tr.tolist(),
               "x_rel_err": xrel.tolist(),
               "max_err_cond": float(err.max()), "argmax_channel": int(err.argmax()),
               "err_cond_by_channel": err.tolist(),
               "contrib_max_by_shift": contrib.max(1).tolist(),
               "n_channels_over_1e-7": int((err > 1e-7).sum())}
        rec["ladder"].append(row)
        print(name, json.dumps({k: v for k, v in row.items() if k not in ("err_cond_by_channel",)}), flush=True)
        del x
        torch.cuda.empty_cache()
    out[name] = rec
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    del xr, ur, fw
    torch.cuda.empty_cache()
json.dump(out, open(sys.argv[1], "w"), indent=1)
