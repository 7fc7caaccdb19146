"""Graph path vs persistent kernel (TEM_LAUNCH_*) on the small BASELINE
configs: wall time of one plain split solve (tol 1e-10, committed table),
iterations, kernel launches; CUDA events on the solve's stream.

    python scripts/launch_modes.py out.json tiny block layered
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
    mass = fw.edge_mass(sigma)
    rec = {"unknowns": fw.n_unknowns, "shifts": table.n_shift}
    xs = {}
    for mode in ("graphs", "persistent"):
        fw.launch_mode = mode
        for _ in range(2):
            fw.cocg(mass, f, table.shifts, tol=1e-10, maxit=200000)
        times = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            x, it, rr = fw.cocg(mass, f, table.shifts, tol=1e-10, maxit=200000)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        st = fw.stats()
        xs[mode] = x.clone()
        rec[mode] = {"ms_median": float(np.median(times)), "ms": times, "iters": it.tolist(),
                     "shift_iterations": int(it.sum()), "loop_ms": st["loop_ms"],
                     "launches": st["kernel_launches"], "persistent": st["persistent"],
                     "sui_per_s": float(it.sum()) * fw.n_unknowns / (np.median(times) * 1e-3)}
        print(name, mode, json.dumps(rec[mode]), flush=True)
    d = (xs["graphs"] - xs["persistent"]).abs().pow(2).sum(1).sqrt() / xs["graphs"].abs().pow(2).sum(1).sqrt()
    rec["x_rel_diff"] = d.cpu().numpy().tolist()
    rec["speedup"] = rec["graphs"]["ms_median"] / rec["persistent"]["ms_median"]
    print(name, "speedup", rec["speedup"], "x diff max", max(rec["x_rel_diff"]), flush=True)
    out[name] = rec
    json.dump(out, open(sys.argv[1], "w"), indent=1)
