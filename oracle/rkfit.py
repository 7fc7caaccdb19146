"""ORACLE (test infrastructure): the shared-pole rational family of §3.2.

PAPER.md §3.2 eq:ratfam (lines 171-175): a family

    r^[j](x) = sum_{i=1}^{m} alpha_i^[j] / (x - xi_i)  ~  exp(-t_j x),  x >= 0,

with poles xi_i SHARED by all time channels t_j (type [(m-1)/m], "dropped the
absolute terms", line 183).  The poles are found by RKFIT (Berljafa & Guettel,
cited at line 171) minimising eq:rkfit (line 177),

    sum_j w_j || r^[j](S) v - exp(-t_j S) v ||_2^2,

"where ... S is a diagonal surrogate matrix with 'dense' eigenvalues on
[0, +inf), v is the vector of all ones" (line 181).

The RKFIT iteration, as cited, for a diagonal S = diag(lambda):

  1. V = orthonormal basis of the rational Krylov space
     Q_{m+1}(S, v, q_m) = span{v, (S - xi_1)^-1 v, ..., (S - xi_m)^-1 v}
     (q_m(z) = prod (z - xi_i); for distinct poles this partial-fraction
     spanning set spans the same space);
  2. c = right singular vector, smallest singular value, of the stacked
     matrices sqrt(w_j) (I - W W^*) F_j V, F_j = exp(-t_j S), where W spans
     the type [(m-1)/m] part span{(S - xi_i)^-1 v} (the family has no
     absolute term, Table 1 caption "type [(m-1)/m]");
  3. the new poles are the roots of the rational function rhat with
     rhat(S) v = V c (pole relocation);
  4. repeat; finally the residues alpha^[j] of each channel are the linear
     least-squares fit of F_j v from span{(S - xi_i)^-1 v} (type [(m-1)/m]).

Time is normalised by t_max (reading R3): the fit is done for
exp(-tau_j y), tau_j = t_j / t_max in [t_min/t_max, 1], which is the
variable of PAPER.md Fig. 1 (interval [10^-3, 1], nearest pole pair
-7.574 +- 12.45i).  In the physical variable x = y / t_max the poles are
xi / t_max and the residues alpha / t_max.

Conjugate symmetry: the problem is real, so the spaces are built from real
spanning vectors (Re and Im of (S - xi)^-1 v for each pair) and the relocated
rational function has real coefficients; its complex roots are then exact
conjugate pairs (we symmetrise the last bits).  A real root on [0, inf)
would make a shifted system singular (§3.3 "stay away from the spectral
region"); such a root is reflected to the negative axis (reading R4).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class RationalFamily:
    """Shared poles + residue table in the NORMALISED variable y = t_max x."""

    poles: np.ndarray        # (m,) complex, conjugate-closed
    residues: np.ndarray     # (m, K) complex; column j = alpha^[j]
    taus: np.ndarray         # (K,) t_j / t_max
    t_max: float
    weights: np.ndarray      # (K,) w_j
    history: list = field(default_factory=list)

    @property
    def degree(self) -> int:
        return self.poles.size

    @property
    def times(self) -> np.ndarray:
        return self.taus * self.t_max

    def eval(self, j: int, y) -> np.ndarray:
        """r^[j](y) = sum_i alpha_i^[j] / (y - xi_i), complex y allowed."""
        y = np.asarray(y, dtype=np.complex128)
        return np.sum(self.residues[:, j][:, None] / (y.ravel()[None, :] - self.poles[:, None]),
                      axis=0).reshape(y.shape)

    def representatives(self):
        """One pole per conjugate pair (Im > 0) followed by the real poles;
        returns (poles, residues (n_rep, K), is_pair) for eq:rmj."""
        pos = np.flatnonzero(self.poles.imag > 0)
        real = np.flatnonzero(self.poles.imag == 0)
        idx = np.concatenate([pos[np.argsort(np.abs(self.poles[pos]))], real])
        is_pair = np.concatenate([np.ones(pos.size, bool), np.zeros(real.size, bool)])
        return self.poles[idx], self.residues[idx], is_pair

    def physical(self):
        """Representative poles/residues in the physical variable x (1/s):
        xi_x = xi / t_max, alpha_x = alpha / t_max, so that
        r^[j](M^-1 K) b = sum over reps of w * Re(alpha_x (K - xi_x M)^-1 f),
        w = 2 for a conjugate pair, 1 for a real pole (eq:rmj)."""
        p, r, is_pair = self.representatives()
        return p / self.t_max, r / self.t_max, is_pair


def default_surrogate(ratio: float, n: int = 1200) -> np.ndarray:
    """Diagonal surrogate eigenvalues in y: 0 plus ``n-1`` log-spaced points
    from 1e-3 to 1e3 * ratio (reading R3: "dense" on [0, inf) over the decades
    where exp(-tau y) decays for tau in [1/ratio, 1])."""
    return np.concatenate([[0.0], np.logspace(-3.0, np.log10(ratio) + 3.0, n - 1)])


def _spanning_set(lam: np.ndarray, poles: np.ndarray, with_const: bool) -> np.ndarray:
    """Real spanning vectors of span{[v], (S - xi)^-1 v} for a conjugate-closed
    pole set (Re/Im parts for each pair, one vector per real pole)."""
    cols = [np.ones_like(lam)] if with_const else []
    for xi in poles:
        if xi.imag > 0:
            w = 1.0 / (lam - xi)
            cols += [w.real, w.imag]
        elif xi.imag == 0:
            cols.append(1.0 / (lam - xi.real))
    return np.stack(cols, axis=1)


def _pf_coefficients(poles: np.ndarray, d: np.ndarray, with_const: bool):
    """Map real coefficients ``d`` of _spanning_set to (const, e) with
    rational function const + sum_i e_i / (z - xi_i) over ALL poles
    (pole set as produced by _symmetrise: each upper pole followed by its
    conjugate)."""
    const = d[0] if with_const else 0.0
    pos = 1 if with_const else 0
    e = np.zeros(poles.size, dtype=np.complex128)
    n = 0
    while n < poles.size:
        xi = poles[n]
        if xi.imag > 0:
            if not (n + 1 < poles.size and poles[n + 1] == np.conj(xi)):
                raise ValueError("pole set is not in (p, conj p) order")
            a, b = d[pos], d[pos + 1]
            # a Re w + b Im w = ((a - ib)/2) w + ((a + ib)/2) conj(w), w = 1/(z - xi)
            e[n] = 0.5 * (a - 1j * b)
            e[n + 1] = 0.5 * (a + 1j * b)
            pos += 2
            n += 2
        elif xi.imag == 0:
            e[n] = d[pos]
            pos += 1
            n += 1
        else:
            raise ValueError("pole set is not in (p, conj p) order")
    return const, e


def _symmetrise(z: np.ndarray, tol: float = 1e-10) -> np.ndarray:
    """Make a root set exactly conjugate-closed (pairs ordered (p, conj p)),
    and keep it off [0, inf): a real root >= 0 would make K - xi M singular
    on the spectrum, so it is reflected to -|xi| (reading R4).  Complex roots
    are kept where RKFIT puts them, in either half-plane."""
    z = np.asarray(z, dtype=np.complex128)
    real = np.abs(z.imag) <= tol * np.maximum(np.abs(z), 1e-300)
    upper = list(z[(~real) & (z.imag > 0)])
    lower = list(z[(~real) & (z.imag < 0)])
    pairs = []
    for u in upper:
        if lower:
            q = int(np.argmin([abs(u - np.conj(l)) for l in lower]))
            pairs.append(0.5 * (u + np.conj(lower.pop(q))))
        else:
            pairs.append(u)
    pairs += [np.conj(l) for l in lower]
    reals = list(z[real].real)
    # odd leftovers (a near-real pair split by rounding): the pair with the
    # smallest imaginary part becomes two real roots, keeping the degree
    while 2 * len(pairs) + len(reals) > z.size and pairs:
        q = int(np.argmin([abs(p.imag) for p in pairs]))
        p = pairs.pop(q)
        reals += [p.real, p.real * (1 + 1e-8)]
    out = []
    for p in pairs:
        out += [p, np.conj(p)]
    out += [complex(-abs(r), 0.0) for r in reals]
    return np.array(out[: z.size], dtype=np.complex128)


def initial_poles(m: int, ratio: float) -> np.ndarray:
    """Deterministic start: m/2 conjugate pairs with log-spaced moduli in
    [1, 10 ratio] on the rays arg = +-(pi - pi/3), plus one real pole if m
    is odd."""
    npair = m // 2
    mod = np.logspace(0.0, np.log10(10.0 * ratio), max(npair, 1))[:npair]
    ang = np.pi - np.pi / 3
    p = []
    for r in mod:
        z = r * np.exp(1j * ang)
        p += [z, np.conj(z)]
    if m % 2:
        p.append(complex(-np.sqrt(10.0 * ratio), 0.0))
    return np.array(p, dtype=np.complex128)


def fit_residues(lam: np.ndarray, F: np.ndarray, poles: np.ndarray) -> np.ndarray:
    """Step 4: per channel j, least squares min || F_j v - sum alpha_i (S-xi_i)^-1 v ||
    in a real spanning set; returns complex alpha (m, K) over all poles."""
    B = _spanning_set(lam, poles, with_const=False)
    D, *_ = np.linalg.lstsq(B, F.T, rcond=None)        # (nb, K)
    res = np.zeros((poles.size, F.shape[0]), dtype=np.complex128)
    for j in range(F.shape[0]):
        _, e = _pf_coefficients(poles, D[:, j], with_const=False)
        res[:, j] = e
    return res


def rational_arnoldi(lam: np.ndarray, v: np.ndarray, poles: np.ndarray):
    """Step 1 in RKFIT's stable form: a rational Arnoldi decomposition (RAD)
    S V K = V H of Q_{m+1}(S, v, q_m) for S = diag(lam), with orthonormal V
    (N x (m+1)) and upper-Hessenberg (m+1) x m pencil (H, K) whose
    subdiagonal ratios h_{k+1,k}/k_{k+1,k} are the poles.  Step k solves
    (S - xi_k I) w = v_k (continuation vector = last basis vector) and
    orthogonalises w with two Gram-Schmidt passes."""
    n, m = lam.size, poles.size
    V = np.zeros((n, m + 1), dtype=np.complex128)
    H = np.zeros((m + 1, m), dtype=np.complex128)
    Kp = np.zeros((m + 1, m), dtype=np.complex128)
    V[:, 0] = v / np.linalg.norm(v)
    for k in range(m):
        xi = poles[k]
        w = V[:, k] / (lam - xi)
        c = np.zeros(m + 1, dtype=np.complex128)
        for _ in range(2):
            h = V[:, : k + 1].conj().T @ w
            w = w - V[:, : k + 1] @ h
            c[: k + 1] += h
        c[k + 1] = np.linalg.norm(w)
        V[:, k + 1] = w / c[k + 1]
        # (S - xi I) V c = v_k  =>  S V c = V (xi c + e_k)
        Kp[:, k] = c
        H[:, k] = xi * c
        H[k, k] += 1.0
    return V, H, Kp


def relocate(H: np.ndarray, Kp: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Step 3: the roots of rhat with rhat(S) v = V c are the eigenvalues of
    the lower m x m part of the rotated pencil (Q^* H, Q^* K), Q unitary with
    first column c (Berljafa & Guettel's RKFIT relocation)."""
    import scipy.linalg as sla
    m1 = c.size
    # Householder reflector P with P e_1 = c (up to a unimodular factor)
    e1 = np.zeros(m1, dtype=np.complex128)
    e1[0] = 1.0
    alpha = -np.exp(1j * np.angle(c[0])) if c[0] != 0 else -1.0
    u = c - alpha * e1
    nu = np.linalg.norm(u)
    Q = np.eye(m1, dtype=np.complex128) if nu == 0 else \
        np.eye(m1) - 2.0 * np.outer(u, u.conj()) / nu ** 2
    # Q e1 = alpha e1 reflected -> proportional to c; Q is Hermitian unitary
    Hq = Q.conj().T @ H
    Kq = Q.conj().T @ Kp
    return sla.eig(Hq[1:], Kq[1:], right=False)


def rkfit(taus, m: int, weights=None, lam=None, iters: int = 12,
          poles0=None) -> RationalFamily:
    """Shared-pole RKFIT family of degree ``m`` for exp(-tau_j y), y >= 0.

    ``taus`` are t_j / t_max (so max(taus) == 1 for the normalisation R3).
    Returns the iterate with the smallest objective eq:rkfit."""
    taus = np.asarray(taus, dtype=np.float64)
    K = taus.size
    w = np.ones(K) if weights is None else np.asarray(weights, dtype=np.float64)
    ratio = taus.max() / taus.min()
    lam = default_surrogate(ratio) if lam is None else np.asarray(lam, dtype=np.float64)
    F = np.exp(-np.outer(taus, lam))                    # F_j v, v = ones
    v = np.ones_like(lam)
    xi = initial_poles(m, ratio) if poles0 is None else np.asarray(poles0, np.complex128)

    def objective(p):
        res = fit_residues(lam, F, p)
        R = (res.T[:, :, None] / (lam[None, None, :] - p[None, :, None])).sum(axis=1)
        return float(np.sum(w[:, None] * np.abs(R - F) ** 2)), res

    best = None
    history = []
    for _ in range(iters):
        obj, res = objective(xi)
        history.append(obj)
        if best is None or obj < best[0]:
            best = (obj, xi.copy(), res)
        # step 1: RAD of Q_{m+1}(S, v, q_m)
        V, H, Kp = rational_arnoldi(lam, v, xi)
        # step 2 for type [(m-1)/m]: stacked sqrt(w_j) (I - W W^*) F_j V with W an
        # orthonormal basis of the functions vanishing at infinity,
        # span{(S - xi_i)^-1 v}; smallest right singular vector
        Wb, _ = np.linalg.qr(_spanning_set(lam, xi, with_const=False))
        blocks = []
        for j in range(K):
            FV = F[j][:, None] * V
            blocks.append(np.sqrt(w[j]) * (FV - Wb @ (Wb.conj().T @ FV)))
        _, _, Vh = np.linalg.svd(np.vstack(blocks), full_matrices=False)
        c = Vh[-1].conj()
        # step 3: new poles = roots of rhat
        xi = _symmetrise(relocate(H, Kp, c))
        if xi.size != m or not np.all(np.isfinite(xi)):
            break
    if xi.size == m and np.all(np.isfinite(xi)):
        obj, res = objective(xi)
        history.append(obj)
        if obj < best[0]:
            best = (obj, xi.copy(), res)
    return RationalFamily(poles=best[1], residues=best[2], taus=taus, t_max=1.0,
                          weights=w, history=history)


def fit_family(times, m: int, weights=None, iters: int = 12) -> RationalFamily:
    """Fit for physical channels ``times`` (s); stores t_max for x = y/t_max."""
    times = np.asarray(times, dtype=np.float64)
    t_max = float(times.max())
    fam = rkfit(times / t_max, m, weights=weights, iters=iters)
    fam.t_max = t_max
    return fam


def error_grid(ratio: float, n: int = 4000) -> np.ndarray:
    """Evaluation grid for eq:error: 0 plus log-spaced points covering the
    decay of every channel and the far tail (reading R3)."""
    return np.concatenate([[0.0], np.logspace(-4.0, np.log10(ratio) + 5.0, n - 1)])


def channel_errors(fam: RationalFamily, grid=None) -> np.ndarray:
    """eq:error per channel: max_{y in grid} |exp(-tau_j y) - r^[j](y)|."""
    ratio = fam.taus.max() / fam.taus.min()
    y = error_grid(ratio) if grid is None else np.asarray(grid, dtype=np.float64)
    R = (fam.residues.T[:, :, None] / (y[None, None, :] - fam.poles[None, :, None])).sum(axis=1)
    return np.max(np.abs(np.exp(-np.outer(fam.taus, y)) - R.real), axis=1)


def uniform_error(fam: RationalFamily, grid=None) -> float:
    """eq:uniform_error: max_j w_j * error_j."""
    return float(np.max(fam.weights * channel_errors(fam, grid)))
