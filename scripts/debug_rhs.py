"""Debug: tem_cocg_solve_rhs against tem_cocg_solve on scaled right-hand sides."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_11657_b200 import RationalTable, TemForward
from workloads import make_workload
from oracle import yee
wl = make_workload("tiny")
fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
asm = yee.assemble(wl); slots = fw.slot(*asm.keys())
sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
mass = fw.edge_mass(sigma)
shifts = np.array([800 - 300j, 2500 + 0j, 1200 + 0j, 5e3 + 4e3j])
x0, it0, rr0 = fw.cocg(mass, f, shifts, tol=1e-12)
for scale in (1.0, 1j, 1 + 2j):
    B = (f.to(torch.complex128) * scale).unsqueeze(0).repeat(4, 1).contiguous()
    x, it, rr = fw.cocg_rhs(mass, B, shifts, [1e-12] * 4)
    d = ((x - scale * x0).abs().max(1).values / x0.abs().max(1).values).cpu().numpy()
    print("scale", scale, "iters", it, it0, "relres", rr, "rel diff", d, "real", fw.stats()["real_shifts"])
    xg = x.cpu().numpy()
    for q in range(4):
        A = asm.shifted(complex(shifts[q]))
        b = B[q].cpu().numpy()[slots]
        print("   true res", q, np.linalg.norm(b - A @ xg[q, slots]) / np.linalg.norm(b))
rng = np.random.default_rng(1)
Bn = np.zeros((4, fw.n_slots), dtype=np.complex128)
Bn[:, slots] = rng.normal(size=(4, asm.n)) + 1j * rng.normal(size=(4, asm.n))
x, it, rr = fw.cocg_rhs(mass, torch.from_numpy(Bn).cuda(), shifts, [1e-12] * 4)
xg = x.cpu().numpy()
for q in range(4):
    A = asm.shifted(complex(shifts[q]))
    print("random rhs", q, it[q], rr[q], np.linalg.norm(Bn[q, slots] - A @ xg[q, slots]) / np.linalg.norm(Bn[q, slots]))
