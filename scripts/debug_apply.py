import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import yee
from paper_2506_11657_b200 import TemForward
from workloads import make_workload
from workloads.configs import make_custom
def run(wl, S, label):
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    asm = yee.assemble(wl)
    c,i,j,k = asm.keys()
    slots = fw.slot(c,i,j,k)
    rng = np.random.default_rng(S)
    shifts = (10 ** rng.uniform(1, 6, S)) * np.exp(1j * rng.uniform(-np.pi, np.pi, S))
    X = rng.normal(size=(asm.n, S)) + 1j * rng.normal(size=(asm.n, S))
    xg = np.zeros((S, fw.n_slots), dtype=np.complex128); xg[:, slots] = X.T
    mass = fw.edge_mass(torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda())
    y = fw.apply(mass, shifts, torch.from_numpy(xg).cuda()).cpu().numpy()
    worst = 0
    for s in range(S):
        ref = asm.K @ X[:, s] + shifts[s] * asm.Mdiag * X[:, s]
        scale = np.abs(asm.K) @ np.abs(X[:, s]) + abs(shifts[s]) * asm.Mdiag * np.abs(X[:, s])
        rel = np.abs(y[s, slots] - ref) / scale
        bad = np.flatnonzero(rel > 1e-13)
        worst = max(worst, rel.max())
        if bad.size and s < 3:
            print(f"  [{label}] s={s} bad={bad.size}/{rel.size} max={rel.max():.2e}; first bad (c,i,j,k):",
                  [(int(c[b]), int(i[b]), int(j[b]), int(k[b])) for b in bad[:6]])
            cs, ks_ = c[bad], k[bad]
            print("     bad by comp", np.bincount(cs, minlength=3), "k values", np.unique(ks_)[:20], "j values", np.unique(j[bad])[:20], "i values", np.unique(i[bad])[:20])
    print(f"[{label}] S={S} worst rel {worst:.2e}", flush=True)
for nzc in ("1", "2"):
    os.environ["TEM_FORCE_NZC"] = nzc
    run(make_workload("tiny"), 2, f"tiny nzc={nzc}")
    run(make_custom(40, 20, 12, seed=3), 2, f"40x20x12 nzc={nzc}")
    run(make_workload("block"), 2, f"block nzc={nzc}")
    run(make_workload("block"), 32, f"block nzc={nzc}")
