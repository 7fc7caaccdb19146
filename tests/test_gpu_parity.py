"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars:
* edge mass, operator apply, synthesis: element-wise, rel. 1e-13 .. 1e-14
  (same arithmetic, different summation order);
* solves: per-shift true residual of the GPU solution, computed with the
  oracle's own CSR, <= the requested tolerance (2e-10 at tol 1e-10, 2e-13
  at tol 1e-14); at tol 1e-10 the solutions agree with the oracle's exact
  LU in the M-norm (< 1e-6) on grids of < 20 000 unknowns;
* channel fields u(t_j) of a tight solve (tol 1e-14, single-tile grids):
  relative L2 <= 1e-7 at every channel over the conducting edges, and
  <= 1e-7 of the summand scale T_j = || sum_i w_i |alpha_ij| |x_i| ||_2
  over all edges (reading R6); the plain all-edge error is printed only;
* GPU fields vs dense expm on `tiny`: the M-norm bound of P:210-217.
The channel bar at the north-star tolerance 1e-10 (refined forward,
multi-tile `block` included) is in test_gpu_accuracy.py.
"""
import numpy as np
import pytest
import torch

from oracle import forward as ofw
from oracle import yee
from workloads import make_workload
from workloads.configs import make_custom

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_11657_b200 import RationalTable, TemForward  # noqa: E402
from paper_2506_11657_b200 import _lib  # noqa: E402


# COCG scheme x launch path (TEM_SOLVER_*, TEM_LAUNCH_* of include/tem_b200.h):
# the split scheme in the persistent cooperative kernel and in CUDA graphs of
# two kernels per iteration, and the two-sweep scheme
SOLVERS = ["split_persistent", "split_graphs", "two_sweep"]


def _configure(fw, solver):
    if solver.startswith("split"):
        fw.solver = "split"
        fw.launch_mode = {"split": "auto", "split_persistent": "persistent", "split_graphs": "graphs"}[solver]
    else:
        fw.solver = solver


def _setup(wl, table_name=None, table=None, solver="split"):
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    _configure(fw, solver)
    asm = yee.assemble(wl)
    slots = fw.slot(*asm.keys())
    if table is None:
        table = RationalTable.load(table_name or wl.name)
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
    f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
    return fw, asm, slots, table, sigma, f


def _oracle_table(wl, degree=None):
    from oracle import rkfit
    fam = rkfit.fit_family(wl.times, degree or wl.n_poles)
    p, r, pair = fam.physical()
    return RationalTable(-p, r, pair, fam.times, rkfit.uniform_error(fam))


WORKLOADS = {
    "tiny": lambda: make_workload("tiny"),
    "ragged": lambda: make_custom(11, 6, 7, seed=2),
    "ragged2": lambda: make_custom(13, 9, 5, seed=5, n_air=1),
    "min2": lambda: make_custom(2, 2, 2, n_air=0),
}


@pytest.mark.parametrize("name", ["tiny", "ragged", "ragged2", "block"])
def test_edge_mass(name):
    wl = make_workload(name) if name in ("tiny", "block") else WORKLOADS[name]()
    fw, asm, slots, _, sigma, _ = _setup(wl, table=RationalTable([1.0], [[1.0]], [False], [1.0]))
    m = fw.edge_mass(sigma).cpu().numpy()
    np.testing.assert_allclose(m[slots], asm.Mdiag, rtol=1e-14, atol=0)
    mask = np.ones(m.size, bool)
    mask[slots] = False
    assert np.all(m[mask] == 0.0)


@pytest.mark.parametrize("nzc", ["", "2", "3"])
@pytest.mark.parametrize("name,S", [("tiny", 8), ("ragged", 10), ("ragged2", 1), ("block", 32),
                                    ("min2", 3)])
def test_apply_shifted(name, S, nzc, monkeypatch):
    """Operator apply vs the oracle CSR, element-wise; also with the z-range
    of each tile split into 2 / 3 chunks (TEM_FORCE_NZC), which exercises
    the pipeline prologue at k > 0."""
    if nzc:
        monkeypatch.setenv("TEM_FORCE_NZC", nzc)
    wl = make_workload(name) if name in ("tiny", "block") else WORKLOADS[name]()
    fw, asm, slots, _, sigma, _ = _setup(wl, table=RationalTable([1.0], [[1.0]], [False], [1.0]))
    rng = np.random.default_rng(S)
    shifts = (10 ** rng.uniform(1, 6, S)) * np.exp(1j * rng.uniform(-np.pi, np.pi, S))
    X = rng.normal(size=(asm.n, S)) + 1j * rng.normal(size=(asm.n, S))
    xg = np.zeros((S, fw.n_slots), dtype=np.complex128)
    xg[:, slots] = X.T
    mass = fw.edge_mass(sigma)
    y = fw.apply(mass, shifts, torch.from_numpy(xg).cuda()).cpu().numpy()
    mask = np.ones(fw.n_slots, bool)
    mask[slots] = False
    assert np.all(y[:, mask] == 0)
    for s in range(S):
        ref = asm.K @ X[:, s] + shifts[s] * asm.Mdiag * X[:, s]
        scale = np.abs(asm.K) @ np.abs(X[:, s]) + abs(shifts[s]) * asm.Mdiag * np.abs(X[:, s])
        assert np.all(np.abs(y[s, slots] - ref) <= 1e-13 * scale + 1e-300)


def _term_scale(X, table):
    w = np.where(table.is_pair, 2.0, 1.0)
    return np.abs(X) @ (w[:, None] * np.abs(table.residues))    # (N, K)


def _air_edges(asm, wl):
    """Free edges with all touching cells in the air layer (sigma = 1e-8)."""
    c, i, j, k = asm.keys()
    ks = wl.surface_k
    return ((c == 2) & (k >= ks)) | ((c != 2) & (k > ks))


@pytest.mark.parametrize("solver", SOLVERS)
@pytest.mark.parametrize("name", ["tiny", "ragged", "ragged2"])
def test_forward_parity_vs_exact_lu(name, solver):
    """Tight solve (tol 1e-14) vs the oracle's exact LU, channel fields u(t_j):
    relative L2 <= 1e-7 at EVERY channel over the conducting (non-air)
    edges, and <= 1e-7 of the summand scale T_j over all edges.  The air's
    curl-free gradient components are fixed only to eps * cond(A) by any fp64
    solver (reading R6); their plain relative error is reported, not gated."""
    wl = WORKLOADS[name]()
    table = RationalTable.load("tiny") if name == "tiny" else _oracle_table(wl)
    fw, asm, slots, table, sigma, f = _setup(wl, table=table, solver=solver)
    mass = fw.edge_mass(sigma)
    x, iters, relres = fw.cocg(mass, f, table.shifts, tol=1e-14, maxit=50000,
                               raise_on_noconv=False)
    u = fw.synthesize(x, table.residues, table.is_pair)
    Xo = ofw.shifted_solves(asm, table.shifts)
    Uo = ofw.synthesize(Xo, table.residues, table.is_pair)
    ug = u.cpu().numpy()[:, slots].T                      # (N, K)
    xg = x.cpu().numpy()[:, slots].T
    for i, s in enumerate(table.shifts):
        assert ofw.relative_residual(asm, s, xg[:, i]) <= 2e-13
    earth = ~_air_edges(asm, wl)
    E = ug - Uo
    rel_earth = np.linalg.norm(E[earth], axis=0) / np.linalg.norm(Uo[earth], axis=0)
    assert np.all(rel_earth <= 1e-7), rel_earth.max()
    T = np.linalg.norm(_term_scale(Xo, table), axis=0)
    rel_term = np.linalg.norm(E, axis=0) / T
    assert np.all(rel_term <= 1e-7), rel_term.max()
    plain = np.linalg.norm(E, axis=0) / np.linalg.norm(Uo, axis=0)
    print(f"[{name}] per-channel rel L2: earth max {rel_earth.max():.2e}, "
          f"term max {rel_term.max():.2e}, plain (incl. air) max {plain.max():.2e}")


@pytest.mark.parametrize("solver", SOLVERS)
@pytest.mark.parametrize("name", ["tiny", "ragged", "block"])
def test_cocg_default_tolerance(name, solver):
    """North-star tolerance 1e-10: every shift converged, true residual
    (oracle CSR) within the tolerance, M-norm agreement with the oracle."""
    wl = make_workload(name) if name in ("tiny", "block") else WORKLOADS[name]()
    table = RationalTable.load(name) if name in ("tiny", "block") else _oracle_table(wl)
    fw, asm, slots, table, sigma, f = _setup(wl, table=table, solver=solver)
    mass = fw.edge_mass(sigma)
    x, iters, relres = fw.cocg(mass, f, table.shifts, tol=1e-10, maxit=50000)
    assert np.all(relres <= 1e-10) and np.all(iters > 0)
    xg = x.cpu().numpy()[:, slots].T
    for i, s in enumerate(table.shifts):
        assert ofw.relative_residual(asm, s, xg[:, i]) <= 2e-10
    if asm.n < 20000:
        Xo = ofw.shifted_solves(asm, table.shifts)
        for i in range(table.n_shift):
            relM = ofw.m_norm(asm, xg[:, i] - Xo[:, i]) / ofw.m_norm(asm, Xo[:, i])
            assert relM < 1e-6


def test_synthesis_exact():
    wl = make_workload("block")
    fw, asm, slots, table, sigma, f = _setup(wl)
    rng = np.random.default_rng(0)
    S = table.n_shift
    X = rng.normal(size=(asm.n, S)) + 1j * rng.normal(size=(asm.n, S))
    xg = np.zeros((S, fw.n_slots), dtype=np.complex128)
    xg[:, slots] = X.T
    u = fw.synthesize(torch.from_numpy(xg).cuda(), table.residues, table.is_pair).cpu().numpy()
    Uo = ofw.synthesize(X, table.residues, table.is_pair)
    T = _term_scale(X, table)
    assert np.all(np.abs(u[:, slots].T - Uo) <= 1e-14 * T + 1e-300)
    mask = np.ones(fw.n_slots, bool)
    mask[slots] = False
    assert np.all(u[:, mask] == 0)


@pytest.mark.parametrize("solver", SOLVERS)
def test_edge_cases(solver):
    wl = make_workload("tiny")
    fw, asm, slots, table, sigma, f = _setup(wl, solver=solver)
    mass = fw.edge_mass(sigma)
    # zero source: converged at iteration 0 with x = 0
    x, iters, relres = fw.cocg(mass, torch.zeros_like(f), table.shifts)
    assert np.all(iters == 0) and torch.count_nonzero(x) == 0
    # maxit too small: TEM_ENOCONV, reported
    with pytest.raises(_lib.TemError) as ei:
        fw.cocg(mass, f, table.shifts, maxit=3)
    assert ei.value.code == _lib.TEM_ENOCONV
    # S out of range
    with pytest.raises(_lib.TemError):
        fw.cocg(mass, f, np.ones(33) * (100 + 1j))
    # single shift equals the corresponding column of the batched solve
    xb, _, _ = fw.cocg(mass, f, table.shifts, tol=1e-12)
    x1, _, _ = fw.cocg(mass, f, table.shifts[2:3], tol=1e-12)
    d = (xb[2] - x1[0]).abs().max().item() / xb[2].abs().max().item()
    assert d < 1e-6


def test_index_range_rejected_before_launch():
    """The sweeps use unsigned 32-bit element indices: a grid with
    S * 6 * nodes >= 2^32 is refused (TEM_EINVAL) before any launch."""
    import ctypes
    lib = _lib.load()
    nx, ny, nz = 330, 330, 220            # 24.2 M nodes: 32 * 6 * Nn > 2^32, 8 * 6 * Nn < 2^32
    h = ctypes.c_void_p()
    w = np.ones(nx)
    dp = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    with torch.cuda.device(0):
        assert lib.tem_create(nx, ny, nz, dp, dp, dp, ctypes.byref(h)) == 0
        try:
            dummy = torch.zeros(8, dtype=torch.float64, device="cuda")
            ptr = ctypes.c_void_p(dummy.data_ptr())
            sh = np.ones(64)
            rc = lib.tem_apply_shifted(h, ptr, 32, sh.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ptr, ptr, None)
            assert rc == -1                                   # TEM_EINVAL
            assert b"2^32" in lib.tem_last_error()
        finally:
            lib.tem_destroy(h)


def test_forward_host_matches_device_path():
    wl = make_workload("tiny")
    fw, asm, slots, table, sigma, f = _setup(wl)
    u_dev, _, it_dev, _ = fw.forward(sigma, f, table)
    u_host, it_host, _ = fw.forward_host(wl.sigma, fw.source_vector(wl.source), table)
    assert np.array_equal(it_dev, it_host)
    np.testing.assert_array_equal(u_dev.cpu().numpy(), u_host)


@pytest.mark.parametrize("solver", SOLVERS)
def test_deterministic_repeat(solver):
    wl = make_workload("block")
    fw, asm, slots, table, sigma, f = _setup(wl, solver=solver)
    mass = fw.edge_mass(sigma)
    x1, i1, _ = fw.cocg(mass, f, table.shifts)
    x2, i2, _ = fw.cocg(mass, f, table.shifts)
    assert np.array_equal(i1, i2)
    assert torch.equal(x1, x2)


@pytest.mark.parametrize("solver", SOLVERS)
def test_tall_grid_forced_chunks_vs_oracle_cocg(solver):
    """nz = 136 > kMaxChunk (128) forces z-chunking in every launch; 32 shifts
    (the ABI maximum) on a ragged 19x15x136 grid with random conductivity,
    full COCG to 1e-12 vs the oracle's own COCG to 1e-13 for two shifts:
    M-norm and conducting-edge agreement, true residual of all 32."""
    from oracle import cocg as ocg
    wl = make_custom(19, 15, 136, h=30.0, n_air=8, seed=9)
    rng = np.random.default_rng(4)
    S = 32
    shifts = (10 ** rng.uniform(2.5, 5.5, S)) * np.exp(1j * rng.uniform(-1.2, 1.2, S))
    table = RationalTable(shifts, np.ones((S, 1)), np.zeros(S, bool), [1.0])
    fw, asm, slots, table, sigma, f = _setup(wl, table=table, solver=solver)
    mass = fw.edge_mass(sigma)
    x, iters, relres = fw.cocg(mass, f, table.shifts, tol=1e-12, maxit=100000)
    xg = x.cpu().numpy()[:, slots].T
    res = [ofw.relative_residual(asm, s, xg[:, i]) for i, s in enumerate(table.shifts)]
    assert max(res) <= 5e-12, res
    earth = ~_air_edges(asm, wl)
    for i in (0, 31):
        xo, _, _ = ocg.cocg(asm, complex(table.shifts[i]), tol=1e-13, maxit=20000)
        relM = ofw.m_norm(asm, xg[:, i] - xo) / ofw.m_norm(asm, xo)
        rel_e = np.linalg.norm((xg[:, i] - xo)[earth]) / np.linalg.norm(xo[earth])
        assert relM < 1e-9 and rel_e < 1e-8, (i, relM, rel_e)


@pytest.mark.parametrize("mode", ["split_persistent", "split_graphs"])
@pytest.mark.parametrize("maxit", [5, 6, 37, 38])
def test_split_iterate_bookkeeping(maxit, mode, monkeypatch):
    """The split scheme advances x every second iteration (and re-forms
    p_{i-1} from p_i, z_i); stopped after an odd or even number of
    iterations, x must be the COCG iterate whose residual the recursion
    reports: ||f - A x|| / ||f|| (oracle CSR) equals relres, and both the
    p-re-reading and the re-forming path give the same x."""
    wl = make_workload("block")
    fw, asm, slots, table, sigma, f = _setup(wl, solver=mode)
    mass = fw.edge_mass(sigma)
    x, iters, relres = fw.cocg(mass, f, table.shifts, tol=1e-14, maxit=maxit,
                               raise_on_noconv=False)
    assert fw.stats()["persistent"] == (mode == "split_persistent")
    assert np.all(iters == maxit)
    xg = x.cpu().numpy()[:, slots].T
    for i, s in enumerate(table.shifts):
        true = ofw.relative_residual(asm, s, xg[:, i])
        assert abs(true - relres[i]) <= 1e-6 * relres[i], (i, true, relres[i])
    monkeypatch.setenv("TEM_XDIRECT", "1")
    x2, iters2, relres2 = fw.cocg(mass, f, table.shifts, tol=1e-14, maxit=maxit,
                                  raise_on_noconv=False)
    d = ((x2 - x).abs().pow(2).sum(1).sqrt() / x.abs().pow(2).sum(1).sqrt()).cpu().numpy()
    assert np.all(d <= 1e-12), d


def test_split_and_two_sweep_agree():
    """Both COCG schemes, and the split scheme on both launch paths, converge
    to the same solutions (M-norm, conducting edges) on the block model."""
    wl = make_workload("block")
    out = {}
    for solver in SOLVERS:
        fw, asm, slots, table, sigma, f = _setup(wl, solver=solver)
        mass = fw.edge_mass(sigma)
        x, iters, relres = fw.cocg(mass, f, table.shifts, tol=1e-12, maxit=50000)
        out[solver] = x.cpu().numpy()[:, slots].T
    # both stop at recursive residual 1e-12; their errors (and so their
    # difference) are that times the conditioning of the shifted system, the
    # same bar test_cocg_default_tolerance applies against the exact LU
    earth = ~_air_edges(asm, wl)
    for va, vb in (("split_persistent", "two_sweep"), ("split_graphs", "two_sweep"),
                   ("split_persistent", "split_graphs")):
        relM, rele = [], []
        for i in range(table.n_shift):
            a, b = out[va][:, i], out[vb][:, i]
            relM.append(ofw.m_norm(asm, a - b) / ofw.m_norm(asm, b))
            rele.append(np.linalg.norm((a - b)[earth]) / np.linalg.norm(b[earth]))
        print(f"{va} vs {vb}: M-norm max {max(relM):.2e}, conducting edges max {max(rele):.2e}")
        assert max(relM) <= 1e-6 and max(rele) <= 1e-9, (va, vb, relM, rele)   # r01: 1.5e-8, 4.4e-11


def test_shift_partitioned_forward_sums_to_full(monkeypatch):
    """--partition shifts on one GPU: the per-rank partial forwards
    (paper_2506_11657_b200.distributed.forward_partial) over a 3-way shift
    partition add up to the full forward (the NCCL reduce is a plain sum).
    The z-chunking is pinned so every shift sees the same CTA geometry, and
    so the same iterates, in the full and in the partial batches."""
    from paper_2506_11657_b200.distributed import forward_partial, shard_shifts
    monkeypatch.setenv("TEM_FORCE_NZC", "2")
    wl = make_workload("tiny")
    fw, asm, slots, table, sigma, f = _setup(wl)
    u_full, _, it_full, _ = fw.forward(sigma, f, table, tol=1e-12)
    parts = shard_shifts(table.shifts, 3)
    u_sum = torch.zeros_like(u_full)
    its = np.zeros(table.n_shift, dtype=int)
    for idx in parts:
        u, it, _ = forward_partial(fw, sigma, f, table, idx, tol=1e-12)
        u_sum += u
        its[idx] = it
    assert np.array_equal(its, it_full)
    Xo = ofw.shifted_solves(asm, table.shifts)
    T = np.linalg.norm(_term_scale(Xo, table), axis=0)
    d = (u_sum - u_full).cpu().numpy()[:, slots].T
    assert np.all(np.linalg.norm(d, axis=0) <= 1e-13 * T)


def test_curl_z_observation_vs_oracle():
    """tem_curl_z (-d_t b_z at receivers, reading R12)
    against the oracle's observation operator on the channel fields of a
    forward; receivers at the loop centre, inside and outside the loop, on
    the surface and below it."""
    wl = make_workload("tiny")
    fw, asm, slots, table, sigma, f = _setup(wl)
    u, _, _, _ = fw.forward(sigma, f, table, tol=1e-12)
    nx, ny, nz = wl.grid.shape
    ks = wl.surface_k
    recv = [(nx // 2, ny // 2, ks), (nx // 2 - 1, ny // 2 - 1, ks), (0, 0, ks), (nx - 1, 2, ks),
            (nx // 2, ny // 2, ks - 2), (3, 5, nz)]
    got = fw.dbzdt(u, recv).cpu().numpy()                      # (K, R)
    c, i, j, k = asm.numbering.keys()
    U_full = u.cpu().numpy()[:, fw.slot(c, i, j, k)].T       # every edge, oracle order
    ref = yee.curl_z_observation(wl.grid, U_full, recv).T    # (K, R)
    scale = np.abs(U_full).max() / (wl.grid.hx.min() * wl.grid.hy.min())
    assert np.all(np.abs(got - ref) <= 1e-13 * scale)
    assert np.all(np.abs(ref[:, 0]) > 0)                       # the loop centre sees a transient
    with pytest.raises(_lib.TemError):
        fw.dbzdt(u, [(nx, 0, 0)])


def test_gpu_fields_vs_dense_expm_tiny():
    """BASELINE configs[0] "also checked against dense expm": the GPU channel
    fields (tight solve) against brute-force exp(-t_j M^-1 K) b (oracle
    eigendecomposition, eq:expm P:134-139) obey the M-norm bound of P:210-217,
        ||u_GPU(t_j) - exp(-t_j M^-1 K) b||_M <= ||b||_M * error_j,
    at all 31 channels, with error_j = max_x |exp(-t_j x) - r^[j](x)| of the
    table (eq:error, computed by the oracle fit); the early channels carry
    real signal, so the comparison is not between zeros."""
    wl = make_workload("tiny")
    fw, asm, slots, table, sigma, f = _setup(wl)
    import json, os
    meta = json.load(open(os.path.join(os.path.dirname(__file__), "..", "data", "rational", "tiny.json")))
    errs = np.asarray(meta["channel_errors"])
    u, x, iters, relres = fw.forward(sigma, f, table, tol=1e-14, maxit=50000)
    ug = u.cpu().numpy()[:, slots].T                       # (N, K)
    E = ofw.expm_dense(asm, wl.times)
    b_M = ofw.m_norm(asm, asm.f / asm.Mdiag)
    ratios = []
    for j in range(len(wl.times)):
        err = ofw.m_norm(asm, ug[:, j] - E[:, j])
        ratios.append(err / (b_M * errs[j]))
        assert err <= b_M * errs[j] * (1 + 1e-6) + 1e-12 * b_M, (j, err, b_M * errs[j])
    assert ofw.m_norm(asm, E[:, 0]) > 10 * b_M * errs[0]
    print(f"GPU vs dense expm: max ||u-E||_M / (||b||_M err_j) = {max(ratios):.3f}")


def test_launch_mode_auto_choice():
    """TEM_LAUNCH_AUTO runs the graph path (measured faster on every BASELINE
    grid); TEM_LAUNCH_PERSISTENT runs k_persist;
    an unknown mode is rejected."""
    wl = make_workload("tiny")
    fw = TemForward(wl.grid.hx, wl.grid.hy, wl.grid.hz)
    assert fw.launch_mode == "auto"
    sigma = torch.from_numpy(fw.sigma_layout(wl.sigma)).cuda()
    f = torch.from_numpy(fw.source_vector(wl.source)).cuda()
    shifts = np.logspace(3, 5, 8) * (1 + 0.5j)
    mass = fw.edge_mass(sigma)
    fw.cocg(mass, f, shifts, tol=1e-6, maxit=20000)
    assert fw.stats()["persistent"] == 0
    fw.launch_mode = "persistent"
    fw.cocg(mass, f, shifts, tol=1e-6, maxit=20000)
    assert fw.stats()["persistent"] == 1
    with pytest.raises(_lib.TemError):
        _lib.check(fw.lib.tem_set_launch_mode(fw._h, 7))
