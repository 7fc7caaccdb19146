"""Prototype: does iterative refinement with an extended-precision residual
lift the late-channel accuracy above what fp64 COCG alone reaches?

    x0 = COCG(f) to tol0;  repeat: r = f - A x (long double, CPU, oracle CSR);
    delta = COCG(Re r) + i COCG(Im r) to eta;  x += delta

Channel errors of each refinement level against the last one, plus long
double true residuals.  Experiment only (calls the oracle's CSR for the
residual); writes JSON.

    python scripts/refine_proto.py out.json block layered large
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import yee  # noqa: E402
from paper_2506_11657_b200 import RationalTable, TemForward  # noqa: E402
from workloads import make_workload  # noqa: E402


def ld_residual(asm, s, x):
    """f - (K + s M) x in long double, chunked over rows."""
    K = asm.K.tocsr()
    n = asm.n
    out = np.empty(n, dtype=np.clongdouble)
    xl = x.astype(np.clongdouble)
    sl = np.clongdouble(s)
    step = 1 << 20
    for a in range(0, n, step):
        b = min(n, a + step)
        p0, p1 = K.indptr[a], K.indptr[b]
        idx = K.indices[p0:p1]
        dat = K.data[p0:p1].astype(np.longdouble)
        prod = dat * xl[idx]
        starts = K.indptr[a:b] - p0
        y = np.add.reduceat(prod, starts)
        y = y + sl * asm.Mdiag[a:b].astype(np.longdouble) * xl[a:b]
        out[a:b] = asm.f[a:b].astype(np.longdouble) - y
    return out


def conducting(asm, wl):
    c, i, j, k = asm.keys()
    ks = wl.surface_k
    return ~(((c == 2) & (k >= ks)) | ((c != 2) & (k > ks)))


out = {}
tol0 = float(os.environ.get("TOL0", "1e-10"))
eta = float(os.environ.get("ETA", "1e-6"))
nref = int(os.environ.get("NREF", "3"))
for name in sys.argv[2:]:
    wl = make_workload(name)
    table = RationalTable.fit(wl.times, wl.n_poles)
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    t0 = time.time()
    asm = yee.assemble(wl)
    slots = fw.slot(*asm.keys())
    cond = conducting(asm, wl)
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
    f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
    mass = fw.edge_mass(sigma)
    S = table.n_shift
    x, it0, _ = fw.cocg(mass, f, table.shifts, tol=tol0, maxit=100000, raise_on_noconv=False)
    X = [x.cpu().numpy()[:, slots]]          # (S, N) free edges, oracle order
    iters = [it0.tolist()]
    resid = []
    for lev in range(nref):
        Xc = X[-1].copy()
        its = []
        rl = []
        for i in range(S):
            r = ld_residual(asm, table.shifts[i], Xc[i])
            rl.append(float(np.sqrt(np.sum(np.abs(r) ** 2)) / np.linalg.norm(asm.f)))
            d = np.zeros(asm.n, dtype=np.complex128)
            it_i = 0
            for part in (r.real, r.imag):
                if not np.any(part):
                    continue
                rhs = np.zeros(fw.n_slots)
                rhs[slots] = part.astype(np.float64)
                dx, itp, _ = fw.cocg(mass, torch.from_numpy(rhs).cuda(), table.shifts[i:i + 1], tol=eta,
                                     maxit=100000, raise_on_noconv=False)
                dd = dx[0].cpu().numpy()[slots]
                d += dd if part is r.real else 1j * dd
                it_i += int(itp[0])
            Xc[i] += d
            its.append(it_i)
        resid.append(rl)
        X.append(Xc)
        iters.append(its)
        print(name, "level", lev, "ld residual", ["%.1e" % v for v in rl], "iters", its, flush=True)
    rl = [float(np.sqrt(np.sum(np.abs(ld_residual(asm, table.shifts[i], X[-1][i])) ** 2)) / np.linalg.norm(asm.f))
          for i in range(S)]
    resid.append(rl)
    w = np.where(table.is_pair, 2.0, 1.0)

    def chans(Xl):
        return np.stack([(w[:, None] * (table.residues[:, k][:, None] * Xl).real).sum(0) for k in range(table.residues.shape[1])])

    U = [chans(Xl) for Xl in X]
    Ur = U[-1]
    nr = np.linalg.norm(Ur[:, cond], axis=1)
    errs = []
    for lev, Ul in enumerate(U[:-1]):
        e = np.linalg.norm((Ul - Ur)[:, cond], axis=1) / nr
        errs.append(e.tolist())
        print(name, "level", lev, "max channel err %.2e at %d, n>1e-7: %d" % (e.max(), e.argmax(), (e > 1e-7).sum()), flush=True)
    out[name] = {"tol0": tol0, "eta": eta, "iters": iters, "ld_residual": resid, "channel_err_vs_last": errs,
                 "s": time.time() - t0}
    json.dump(out, open(sys.argv[1], "w"), indent=1)
