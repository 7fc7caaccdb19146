"""Per-graph trace (TEM_TRACE) of one bench-config solve: time spent at each
active-shift count.  Experiments only.
    python scripts/trace_solve.py [solver] [forward]
`forward`: the bench's channel-accurate forward (first solve 1e-11 + one
refinement round to 1e-4) instead of one plain 1e-10 solve."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
solver = sys.argv[1] if len(sys.argv) > 1 else "split"
fwd = len(sys.argv) > 2 and sys.argv[2] == "forward"
code = f"""
import sys; sys.path.insert(0, {ROOT!r})
import torch
from paper_2506_11657_b200 import RationalTable, TemForward
from workloads import make_workload
wl = make_workload('large')
table = RationalTable.fit(wl.times, wl.n_poles)
fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
fw.solver = {solver!r}
sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
mass = fw.edge_mass(sigma)
if {fwd!r}:
    fw.forward(sigma, f, table, opts=fw.opts(tol=1e-11, refine=1, refine_tol=1e-4))
    print('loop_ms', fw.forward_stats()['loop_ms'])
else:
    fw.cocg(mass, f, table.shifts, tol=1e-10, maxit=200000)
    print('loop_ms', fw.stats()['loop_ms'])
"""
env = dict(os.environ, TEM_TRACE="1")
res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
print(res.stdout)
agg = {}
for ln in res.stderr.splitlines():
    if not ln.startswith("[tem trace]"):
        continue
    if "persistent" in ln:
        continue
    kv = dict(t.split("=", 1) for t in ln.split()[2:] if "=" in t)
    if "slots" not in kv or "chunk_ms" not in kv:   # other trace lines (refinement rounds)
        continue
    key = (int(kv["slots"]), int(kv["nzc"]))
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += float(kv["chunk_ms"])
tot = sum(v[1] for v in agg.values())
for (slots, nzc), (n, ms) in sorted(agg.items(), reverse=True):
    print(f"slots {slots:2d} nzc {nzc:2d}: {n:4d} graphs  {ms:9.1f} ms  ({100*ms/tot:5.1f}%)  "
          f"{ms/n/16:.3f} ms/iter  {ms/n/16/slots:.3f} ms/slot-iter")
