"""Python face of the C ABI (include/tem_b200.h) -- marshalling only.

Every numerical step runs in libtem_b200.so's sm_100a kernels; this module
only moves pointers, sizes and small host arrays across the boundary.
PyTorch provides device memory and streams.

    fw = TemForward(hx, hy, hz)                 # grid (§2.2)
    mass = fw.edge_mass(sigma)                  # M, lumped          (§2.2)
    x, iters, relres = fw.cocg(mass, f, shifts) # (K + s_i M) x_i = f (§3.2, eq:rmj)
    u = fw.synthesize(x, residues, is_pair)     # u(t_j) = 2 Re(S R)  (§3.2)
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np
import torch

from . import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def _cplx(z) -> np.ndarray:
    """complex array -> contiguous interleaved (re, im) float64."""
    z = np.ascontiguousarray(np.asarray(z, dtype=np.complex128))
    return np.ascontiguousarray(z.view(np.float64).reshape(-1))


def _stream_ptr(stream, device=None) -> ctypes.c_void_p:
    s = torch.cuda.current_stream(device) if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda(t: torch.Tensor, dtype, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
    if t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous {dtype}")


class RationalTable:
    """Shared poles and residue table (§3.2 eq:ratfam) in the
    physical variable: shifts s_i = -xi_i (1/s), residues (n_shift, K),
    is_pair (w_i = 2 for a conjugate pair, eq:rmj)."""

    def __init__(self, shifts, residues, is_pair, times, uniform_error=None):
        self.shifts = np.asarray(shifts, dtype=np.complex128)
        self.residues = np.asarray(residues, dtype=np.complex128)
        self.is_pair = np.asarray(is_pair, dtype=bool)
        self.times = np.asarray(times, dtype=np.float64)
        self.uniform_error = uniform_error

    @property
    def n_shift(self) -> int:
        return self.shifts.size

    @classmethod
    def fit(cls, times, degree: int, weights=None, iters: int = 12) -> "RationalTable":
        """Shared-pole family for these time channels, computed by the
        library's host-side fit (tem_fit_family; §3.2 eq:ratfam /
        eq:rkfit).  CPU only, once per channel set."""
        lib = _lib.load()
        t = np.ascontiguousarray(times, dtype=np.float64)
        K, m = t.size, int(degree)
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        n_rep = ctypes.c_int()
        sh = np.zeros(2 * m)
        res = np.zeros(2 * m * K)
        ip = np.zeros(m, dtype=np.int32)
        ue = ctypes.c_double()
        _lib.check(lib.tem_fit_family(K, _dptr(t), None if w is None else _dptr(w), m, int(iters),
                                      ctypes.byref(n_rep), _dptr(sh), _dptr(res), _iptr(ip),
                                      ctypes.byref(ue)))
        n = n_rep.value
        shifts = sh.view(np.complex128)[:n].copy()
        residues = res.view(np.complex128).reshape(m, K)[:n].copy()
        return cls(shifts, residues, ip[:n].astype(bool), t, ue.value)

    def to_json(self) -> dict:
        """The table in the layout of data/rational/*.json (load() reads it)."""
        def c(a):
            return [[float(z.real), float(z.imag)] for z in np.asarray(a, dtype=np.complex128).ravel()]
        return {"shifts": c(self.shifts), "residues": [c(r) for r in self.residues],
                "is_pair": [bool(b) for b in self.is_pair], "times": [float(t) for t in self.times],
                "uniform_error": None if self.uniform_error is None else float(self.uniform_error)}

    @classmethod
    def load(cls, name_or_path: str) -> "RationalTable":
        """Read data/rational/<name>.json (inputs computed once on the host
        by scripts/make_rational_tables.py)."""
        path = name_or_path
        if not os.path.exists(path):
            path = os.path.join(ROOT, "data", "rational", f"{name_or_path}.json")
        with open(path) as fh:
            t = json.load(fh)

        def c(lst):
            return np.array([complex(a, b) for a, b in lst])
        return cls(c(t["shifts"]), np.stack([c(r) for r in t["residues"]]), t["is_pair"],
                   t["times"], t.get("uniform_error"))


class TemForward:
    """One tensor grid on one GPU.  All device buffers are torch tensors."""

    def __init__(self, hx, hy, hz, device=None):
        self.lib = _lib.load()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("TemForward runs on CUDA only")
        self.hx = np.ascontiguousarray(hx, dtype=np.float64)
        self.hy = np.ascontiguousarray(hy, dtype=np.float64)
        self.hz = np.ascontiguousarray(hz, dtype=np.float64)
        self.shape = (self.hx.size, self.hy.size, self.hz.size)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.tem_create(*self.shape, _dptr(self.hx), _dptr(self.hy),
                                           _dptr(self.hz), ctypes.byref(h)))
        self._h = h
        self.Nn = int(self.lib.tem_num_nodes(h))
        self.n_unknowns = int(self.lib.tem_num_unknowns(h))
        self._work = {}

    SOLVERS = {"split": 0, "two_sweep": 1}   # TEM_SOLVER_* of include/tem_b200.h

    @property
    def solver(self) -> str:
        """COCG iteration scheme of tem_cocg_solve (tem_set_solver)."""
        code = int(self.lib.tem_get_solver(self._h))
        return {v: k for k, v in self.SOLVERS.items()}[code]

    @solver.setter
    def solver(self, name: str):
        if name not in self.SOLVERS:
            raise ValueError(f"solver must be one of {sorted(self.SOLVERS)}")
        _lib.check(self.lib.tem_set_solver(self._h, self.SOLVERS[name]))

    LAUNCH_MODES = {"auto": 0, "graphs": 1, "persistent": 2}   # TEM_LAUNCH_* (include/tem_b200.h)

    @property
    def launch_mode(self) -> str:
        """How the split scheme's iterations are launched (tem_set_launch_mode)."""
        code = int(self.lib.tem_get_launch_mode(self._h))
        return {v: k for k, v in self.LAUNCH_MODES.items()}[code]

    @launch_mode.setter
    def launch_mode(self, name: str):
        if name not in self.LAUNCH_MODES:
            raise ValueError(f"launch_mode must be one of {sorted(self.LAUNCH_MODES)}")
        _lib.check(self.lib.tem_set_launch_mode(self._h, self.LAUNCH_MODES[name]))

    def close(self):
        if self._h:
            self.lib.tem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ layout
    @property
    def n_slots(self) -> int:
        return 3 * self.Nn

    def slot(self, c, i, j, k):
        """Slot index of edge (c, i, j, k) in an edge vector ([3][Nn])."""
        nx, ny, _ = self.shape
        return np.asarray(c) * self.Nn + (np.asarray(k) * (ny + 1) + np.asarray(j)) * (nx + 1) \
            + np.asarray(i)

    def source_vector(self, source_edges, current: float = 1.0) -> np.ndarray:
        """Host edge vector f: +-I on the transmitter's edges (layout only)."""
        f = np.zeros(self.n_slots)
        for (c, i, j, k, s) in source_edges:
            f[self.slot(c, i, j, k)] += s * current
        return f

    def sigma_layout(self, sigma: np.ndarray) -> np.ndarray:
        nx, ny, nz = self.shape
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        if sigma.shape != (nz, ny, nx):
            raise ValueError(f"sigma must have shape (nz, ny, nx) = {(nz, ny, nx)}")
        return sigma

    # ------------------------------------------------------------ calls
    # Every call runs with the context's device current (the C ABI rejects a
    # different current device) and on that device's current stream.
    def _call(self, fn, *args):
        with torch.cuda.device(self.device):
            return fn(*args)

    def _stream(self, stream):
        return _stream_ptr(stream, self.device)

    def edge_mass(self, sigma: torch.Tensor, stream=None) -> torch.Tensor:
        _need_cuda(sigma, torch.float64, "sigma")
        if sigma.numel() != self.shape[0] * self.shape[1] * self.shape[2]:
            raise ValueError("sigma size mismatch")
        mass = torch.empty(self.n_slots, dtype=torch.float64, device=self.device)
        _lib.check(self._call(self.lib.tem_edge_mass, self._h, ctypes.c_void_p(sigma.data_ptr()),
                              ctypes.c_void_p(mass.data_ptr()), self._stream(stream)))
        return mass

    def apply(self, mass: torch.Tensor, shifts, x: torch.Tensor, stream=None) -> torch.Tensor:
        """y[s] = (K + s M) x[s]; x is complex128 (S, n_slots), non-free slots 0."""
        sh = _cplx(shifts)
        S = sh.size // 2
        _need_cuda(x, torch.complex128, "x")
        if x.shape != (S, self.n_slots):
            raise ValueError(f"x must be (S, n_slots) = {(S, self.n_slots)}")
        y = torch.empty_like(x)
        _lib.check(self._call(self.lib.tem_apply_shifted, self._h, ctypes.c_void_p(mass.data_ptr()), S,
                              _dptr(sh), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                              self._stream(stream)))
        return y

    def workspace(self, S: int) -> torch.Tensor:
        if S not in self._work:
            nbytes = int(self.lib.tem_cocg_workspace_bytes(self._h, S))
            self._work[S] = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self._work[S]

    def cocg(self, mass: torch.Tensor, f: torch.Tensor, shifts, tol: float = 1e-10,
             maxit: int = 100000, x: torch.Tensor | None = None, stream=None,
             raise_on_noconv: bool = True):
        """Batched multi-shift Jacobi-COCG.  Returns (x, iters, relres)."""
        _need_cuda(mass, torch.float64, "mass")
        _need_cuda(f, torch.float64, "f")
        sh = _cplx(shifts)
        S = sh.size // 2
        if x is None:
            x = torch.empty((S, self.n_slots), dtype=torch.complex128, device=self.device)
        work = self.workspace(S)
        iters = np.zeros(S, dtype=np.int32)
        relres = np.zeros(S, dtype=np.float64)
        rc = self._call(self.lib.tem_cocg_solve, self._h, ctypes.c_void_p(mass.data_ptr()),
                        ctypes.c_void_p(f.data_ptr()), S, _dptr(sh), float(tol), int(maxit),
                        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(work.data_ptr()), work.numel(),
                        _iptr(iters), _dptr(relres), self._stream(stream))
        if rc != 0 and (raise_on_noconv or rc != _lib.TEM_ENOCONV):
            _lib.check(rc)
        return x, iters, relres

    def cocg_rhs(self, mass: torch.Tensor, rhs: torch.Tensor, shifts, tols, maxit: int = 100000,
                 stream=None, raise_on_noconv: bool = True):
        """Per-shift right-hand sides (complex (S, n_slots)) and tolerances
        (tem_cocg_solve_rhs).  Returns (x, iters, relres)."""
        _need_cuda(mass, torch.float64, "mass")
        _need_cuda(rhs, torch.complex128, "rhs")
        sh = _cplx(shifts)
        S = sh.size // 2
        if rhs.shape != (S, self.n_slots):
            raise ValueError(f"rhs must be (S, n_slots) = {(S, self.n_slots)}")
        t = np.ascontiguousarray(np.broadcast_to(np.asarray(tols, dtype=np.float64), (S,)))
        x = torch.empty_like(rhs)
        work = self.workspace(S)
        iters = np.zeros(S, dtype=np.int32)
        relres = np.zeros(S, dtype=np.float64)
        rc = self._call(self.lib.tem_cocg_solve_rhs, self._h, ctypes.c_void_p(mass.data_ptr()),
                        ctypes.c_void_p(rhs.data_ptr()), S, _dptr(sh), _dptr(t), int(maxit),
                        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(work.data_ptr()), work.numel(),
                        _iptr(iters), _dptr(relres), self._stream(stream))
        if rc != 0 and (raise_on_noconv or rc != _lib.TEM_ENOCONV):
            _lib.check(rc)
        return x, iters, relres

    def residual(self, mass: torch.Tensor, f: torch.Tensor, shifts, x: torch.Tensor, stream=None):
        """r_s = f - (K + s M) x_s in double-double (tem_residual).  Returns
        (r (S, n_slots) complex, ||r_s||_2 per shift)."""
        _need_cuda(mass, torch.float64, "mass")
        _need_cuda(f, torch.float64, "f")
        _need_cuda(x, torch.complex128, "x")
        sh = _cplx(shifts)
        S = sh.size // 2
        if x.shape != (S, self.n_slots):
            raise ValueError(f"x must be (S, n_slots) = {(S, self.n_slots)}")
        r = torch.empty_like(x)
        nrm = np.zeros(S)
        _lib.check(self._call(self.lib.tem_residual, self._h, ctypes.c_void_p(mass.data_ptr()),
                              ctypes.c_void_p(f.data_ptr()), S, _dptr(sh), ctypes.c_void_p(x.data_ptr()),
                              ctypes.c_void_p(r.data_ptr()), _dptr(nrm), self._stream(stream)))
        return r, nrm

    def stats(self) -> dict:
        st = _lib.SolveStats()
        _lib.check(self.lib.tem_last_solve_stats(self._h, ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in _lib.SolveStats._fields_}

    def synthesize(self, x: torch.Tensor, residues, is_pair, stream=None) -> torch.Tensor:
        """u[k] = sum_s w_s Re(residues[s, k] x[s]); residues (S, K), x (S, n_slots)."""
        res = np.asarray(residues, dtype=np.complex128)
        S, K = res.shape
        _need_cuda(x, torch.complex128, "x")
        if x.shape != (S, self.n_slots):
            raise ValueError("x shape mismatch")
        r = _cplx(res.T.copy())           # ABI wants [K][S]
        ip = np.ascontiguousarray(np.asarray(is_pair, dtype=np.int32))
        u = torch.empty((K, self.n_slots), dtype=torch.float64, device=self.device)
        _lib.check(self._call(self.lib.tem_synthesize, self._h, S, K, _dptr(r), _iptr(ip),
                              ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(u.data_ptr()),
                              self._stream(stream)))
        return u

    def dbzdt(self, u: torch.Tensor, receivers, stream=None) -> torch.Tensor:
        """-d_t b_z(r_0, t_k) = e_z . curl e at receivers
        given as z-face lower-corner nodes (i, j, k); u (K, n_slots) from
        synthesize.  Returns (K, R) on the device."""
        _need_cuda(u, torch.float64, "u")
        if u.dim() != 2 or u.shape[1] != self.n_slots:
            raise ValueError("u must be (K, n_slots)")
        rec = np.ascontiguousarray(np.asarray(receivers, dtype=np.int32).reshape(-1, 3))
        K, R = u.shape[0], rec.shape[0]
        out = torch.empty((K, R), dtype=torch.float64, device=self.device)
        _lib.check(self._call(self.lib.tem_curl_z, self._h, K, ctypes.c_void_p(u.data_ptr()), R, _iptr(rec),
                              ctypes.c_void_p(out.data_ptr()), self._stream(stream)))
        return out

    @staticmethod
    def opts(tol: float = 1e-10, maxit: int = 200000, refine: bool | int = False, refine_tol: float = 1e-4,
             channel_tol: float = 1e-7, safety: float = 1.5) -> "_lib.ForwardOpts":
        """tem_forward_opts.  refine=True: up to 8 rounds of iterative
        refinement with the channel-aware stopping rule (R13); an
        int sets the round limit."""
        o = _lib.ForwardOpts()
        o.tol, o.maxit = float(tol), int(maxit)
        o.max_refine = (8 if refine is True else int(refine)) if refine else 0
        o.refine_tol, o.channel_tol, o.safety = float(refine_tol), float(channel_tol), float(safety)
        return o

    def forward_workspace(self, S: int, K: int) -> torch.Tensor:
        key = ("fwd", S, K)
        if key not in self._work:
            nbytes = int(self.lib.tem_forward_workspace_bytes(self._h, S, K))
            self._work[key] = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self._work[key]

    def forward_host(self, sigma: np.ndarray, f: np.ndarray, table: RationalTable,
                     tol: float = 1e-10, maxit: int = 100000, out: np.ndarray | None = None,
                     opts=None, **kw):
        """End-to-end with host buffers (tem_forward_host).  Returns
        (u (K, n_slots) host array, iters, relres)."""
        sig = self.sigma_layout(sigma)
        f = np.ascontiguousarray(f, dtype=np.float64)
        S, K = table.residues.shape
        sh = _cplx(table.shifts)
        r = _cplx(table.residues.T.copy())
        ip = np.ascontiguousarray(table.is_pair.astype(np.int32))
        o = opts if opts is not None else self.opts(tol, maxit, **kw)
        u = np.empty((K, self.n_slots)) if out is None else out
        iters = np.zeros(S, dtype=np.int32)
        relres = np.zeros(S)
        rc = self._call(self.lib.tem_forward_host, self._h, _dptr(sig), _dptr(f), S, _dptr(sh), K,
                        _dptr(r), _iptr(ip), ctypes.byref(o), _dptr(u), _iptr(iters), _dptr(relres))
        _lib.check(rc)
        return u, iters, relres

    def forward_stats(self) -> dict:
        st = _lib.ForwardStats()
        _lib.check(self.lib.tem_last_forward_stats(self._h, ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in _lib.ForwardStats._fields_}

    def forward(self, sigma: torch.Tensor, f: torch.Tensor, table: RationalTable,
                tol: float = 1e-10, maxit: int = 200000, stream=None, opts=None,
                raise_on_noconv: bool = True, **kw):
        """Device-resident forward (tem_forward): mass, COCG, synthesis and,
        with refine=..., the channel-aware refinement.  Returns
        (u, x, iters, relres)."""
        _need_cuda(f, torch.float64, "f")
        mass = self.edge_mass(sigma, stream)
        S, K = table.residues.shape
        sh = _cplx(table.shifts)
        r = _cplx(table.residues.T.copy())
        ip = np.ascontiguousarray(table.is_pair.astype(np.int32))
        o = opts if opts is not None else self.opts(tol, maxit, **kw)
        x = torch.empty((S, self.n_slots), dtype=torch.complex128, device=self.device)
        u = torch.empty((K, self.n_slots), dtype=torch.float64, device=self.device)
        work = self.forward_workspace(S, K)
        iters = np.zeros(S, dtype=np.int32)
        relres = np.zeros(S)
        st = _lib.ForwardStats()
        rc = self._call(self.lib.tem_forward, self._h, ctypes.c_void_p(mass.data_ptr()),
                        ctypes.c_void_p(f.data_ptr()), S, _dptr(sh), K, _dptr(r), _iptr(ip), ctypes.byref(o),
                        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(u.data_ptr()),
                        ctypes.c_void_p(work.data_ptr()), work.numel(), _iptr(iters), _dptr(relres),
                        ctypes.byref(st), self._stream(stream))
        if rc != 0 and (raise_on_noconv or rc != _lib.TEM_ENOCONV):
            _lib.check(rc)
        return u, x, iters, relres
