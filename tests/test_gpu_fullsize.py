"""GPU checks at BASELINE.json's full sizes, in the launch configuration
bench.py times (default z-chunking, all shifts in one batch, tol 1e-10).

The oracle cannot solve these grids in seconds, so parity is checked
(i) element-wise on sampled rows the oracle computes one by one (operator
apply: rows of its CSR; synthesis: its per-row sum), and (ii) through a
property that holds at any size: the true relative residual of every GPU
solution, computed with the oracle's own CSR assembly of K and M.
"""
import numpy as np
import pytest
import torch

from oracle import forward as ofw
from oracle import yee
from workloads import make_workload

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_11657_b200 import RationalTable, TemForward  # noqa: E402

_CACHE = {}


def _solved(name, solver="split"):
    if (name, solver) not in _CACHE:
        wl = make_workload(name)
        table = RationalTable.load(name)
        fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
        fw.solver = solver
        sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
        f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
        mass = fw.edge_mass(sigma)
        x, iters, relres = fw.cocg(mass, f, table.shifts, tol=1e-10, maxit=200000)
        asm = yee.assemble(wl)
        slots = fw.slot(*asm.keys())
        _CACHE.clear()
        _CACHE[(name, solver)] = (wl, table, fw, mass, x, iters, relres, asm, slots)
    return _CACHE[(name, solver)]


@pytest.mark.parametrize("name,solver", [("layered", "split"), ("hetero", "split"), ("large", "split"),
                                         ("layered", "two_sweep")])
def test_true_residual_every_shift(name, solver):
    wl, table, fw, mass, x, iters, relres, asm, slots = _solved(name, solver)
    assert np.all(relres <= 1e-10) and np.all(iters > 0)
    for i, s in enumerate(table.shifts):
        xi = x[i].cpu().numpy()[slots]
        rr = ofw.relative_residual(asm, s, xi)
        assert rr <= 5e-10, (i, rr)


@pytest.mark.parametrize("name", ["layered", "large"])
def test_apply_sampled_rows(name):
    wl, table, fw, mass, x, iters, relres, asm, slots = _solved(name)
    rng = np.random.default_rng(7)
    rows = rng.choice(asm.n, size=4000, replace=False)
    # a random complex block with zeros on the non-free slots
    S = table.n_shift
    X = torch.zeros((S, fw.n_slots), dtype=torch.complex128)
    Xf = rng.normal(size=(S, asm.n)) + 1j * rng.normal(size=(S, asm.n))
    X[:, torch.from_numpy(slots)] = torch.from_numpy(Xf)
    y = fw.apply(mass, table.shifts, X.cuda()).cpu().numpy()
    Ks = asm.K[rows]
    for s in range(S):
        ref = Ks @ Xf[s] + table.shifts[s] * asm.Mdiag[rows] * Xf[s, rows]
        scale = abs(Ks) @ np.abs(Xf[s]) + abs(table.shifts[s]) * asm.Mdiag[rows] * np.abs(Xf[s, rows])
        assert np.all(np.abs(y[s, slots[rows]] - ref) <= 1e-13 * scale)


@pytest.mark.parametrize("name", ["large"])
def test_synthesis_sampled_rows(name):
    wl, table, fw, mass, x, iters, relres, asm, slots = _solved(name)
    u = fw.synthesize(x, table.residues, table.is_pair)
    rng = np.random.default_rng(3)
    rows = slots[rng.choice(asm.n, size=5000, replace=False)]
    xr = x[:, torch.from_numpy(rows).cuda()].cpu().numpy().T          # (rows, S)
    ur = u[:, torch.from_numpy(rows).cuda()].cpu().numpy().T          # (rows, K)
    uo = ofw.synthesize(xr, table.residues, table.is_pair)
    w = np.where(table.is_pair, 2.0, 1.0)
    T = np.abs(xr) @ (w[:, None] * np.abs(table.residues))
    assert np.all(np.abs(ur - uo) <= 1e-14 * T + 1e-300)
    # the channels carry signal: the earliest channel is not a cancellation to zero
    assert np.linalg.norm(uo[:, 0]) > 1e-6 * np.linalg.norm(T[:, 0])


def test_bench_config_deterministic_and_synthesis_consistent():
    """Two solves of the bench workload in bench's configuration give
    bit-identical iterates and iteration counts (fixed-order reductions)."""
    wl = make_workload("hetero")
    table = RationalTable.load("hetero")
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
    f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
    mass = fw.edge_mass(sigma)
    x1, i1, _ = fw.cocg(mass, f, table.shifts)
    x2, i2, _ = fw.cocg(mass, f, table.shifts)
    assert np.array_equal(i1, i2)
    assert torch.equal(x1, x2)


def test_bench_default_poles_true_residual():
    """bench.py's default inputs: the library's own host fit (tem_fit_family)
    for the 14M config; every shift's true residual via the oracle CSR."""
    wl = make_workload("large")
    table = RationalTable.fit(wl.times, wl.n_poles)
    assert table.uniform_error < 1e-3
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
    f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
    mass = fw.edge_mass(sigma)
    x, iters, relres = fw.cocg(mass, f, table.shifts, tol=1e-10, maxit=200000)
    assert np.all(relres <= 1e-10)
    asm = yee.assemble(wl)
    slots = fw.slot(*asm.keys())
    for i, s in enumerate(table.shifts):
        assert ofw.relative_residual(asm, s, x[i].cpu().numpy()[slots]) <= 5e-10
