// tem_rkfit.cpp -- host-side construction of the shared-pole rational family
// (§3.2 eq:ratfam, objective eq:rkfit), computed once on the host and
// handed to the GPU path as shifts and residues (BASELINE north star (1)).
//
//   r^[j](y) = sum_i alpha_i^[j] / (y - xi_i) ~ exp(-tau_j y),  y >= 0,
//   tau_j = t_j / t_max (reading R3), poles xi_i shared by all channels.
//
// Pole relocation for a diagonal surrogate S = diag(lambda) with v = 1,
// all in REAL arithmetic (the data are real and the pole set conjugate-closed):
//   1. V = orthonormal basis of span{1, Re/Im (S - xi)^-1 v per pair, (S - xi)^-1 v
//      per real pole} (= the rational Krylov space Q_{m+1}(S, v, q_m)); W the same
//      without the constant (type [(m-1)/m] functions, Table 1 caption);
//   2. c = right singular vector of the smallest singular value of the stacked
//      sqrt(w_j) (I - W W^T) F_j V, F_j = diag(exp(-tau_j lambda));
//   3. new poles = zeros of the rational function with coefficients c, i.e. the
//      eigenvalues of diag(xi) - 1 g^T with g its partial-fraction coefficients
//      divided by its constant term (complex Hessenberg QR here);
//   4. residues of each channel by linear least squares with the poles fixed.
// The best iterate of eq:rkfit's objective is returned.  Independent of the
// CPU oracle (a different formulation of step 3 and its own linear algebra).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tem_b200.h"

namespace {

using cd = std::complex<double>;
using Vec = std::vector<double>;

// ---------------------------------------------------------------- real LA
// Column-major dense matrix.
struct Mat {
  int r = 0, c = 0;
  Vec a;
  Mat() = default;
  Mat(int r_, int c_) : r(r_), c(c_), a((size_t)r_ * c_, 0.0) {}
  double& operator()(int i, int j) { return a[(size_t)j * r + i]; }
  double operator()(int i, int j) const { return a[(size_t)j * r + i]; }
  double* col(int j) { return a.data() + (size_t)j * r; }
  const double* col(int j) const { return a.data() + (size_t)j * r; }
};

double dot(const double* x, const double* y, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}

// Householder QR in place: A (m x n, m >= n) -> R in the upper triangle, the
// reflectors below; tau[n].  Returns false on a zero column.
void householder_qr(Mat& A, Vec& tau) {
  const int m = A.r, n = A.c;
  tau.assign(n, 0.0);
  for (int k = 0; k < n; ++k) {
    double* a = A.col(k);
    double nrm = 0.0;
    for (int i = k; i < m; ++i) nrm += a[i] * a[i];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    const double alpha = a[k] > 0 ? -nrm : nrm;
    const double v0 = a[k] - alpha;
    for (int i = k + 1; i < m; ++i) a[i] /= v0;
    tau[k] = -v0 / alpha;   // H = I - tau v v^T with v = (1, a[k+1:])
    a[k] = alpha;
    for (int j = k + 1; j < n; ++j) {
      double* b = A.col(j);
      double s = b[k];
      for (int i = k + 1; i < m; ++i) s += a[i] * b[i];
      s *= tau[k];
      b[k] -= s;
      for (int i = k + 1; i < m; ++i) b[i] -= s * a[i];
    }
  }
}

// Orthonormal basis Q (m x n) of the columns of B by Householder QR; also R.
void orth(const Mat& B, Mat& Q, Mat& R) {
  Mat A = B;
  Vec tau;
  householder_qr(A, tau);
  const int m = A.r, n = A.c;
  R = Mat(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j; ++i) R(i, j) = A(i, j);
  Q = Mat(m, n);
  for (int j = 0; j < n; ++j) Q(j, j) = 1.0;
  for (int k = n - 1; k >= 0; --k) {
    const double* v = A.col(k);
    for (int j = k; j < n; ++j) {
      double* q = Q.col(j);
      double s = q[k];
      for (int i = k + 1; i < m; ++i) s += v[i] * q[i];
      s *= tau[k];
      q[k] -= s;
      for (int i = k + 1; i < m; ++i) q[i] -= s * v[i];
    }
  }
}

// One-sided Jacobi SVD of a small square R (n x n): returns V (right singular
// vectors as columns) and singular values.
void jacobi_svd(Mat U, Mat& V, Vec& sv) {
  const int n = U.c, m = U.r;
  V = Mat(n, n);
  for (int i = 0; i < n; ++i) V(i, i) = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double alpha = dot(U.col(p), U.col(p), m), beta = dot(U.col(q), U.col(q), m);
        double gamma = dot(U.col(p), U.col(q), m);
        if (gamma == 0.0) continue;
        off = std::max(off, std::fabs(gamma) / std::sqrt(alpha * beta));
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        for (int i = 0; i < m; ++i) {
          const double up = U(i, p), uq = U(i, q);
          U(i, p) = cs * up - sn * uq;
          U(i, q) = sn * up + cs * uq;
        }
        for (int i = 0; i < n; ++i) {
          const double vp = V(i, p), vq = V(i, q);
          V(i, p) = cs * vp - sn * vq;
          V(i, q) = sn * vp + cs * vq;
        }
      }
    if (off < 1e-15) break;
  }
  sv.assign(n, 0.0);
  for (int j = 0; j < n; ++j) sv[j] = std::sqrt(dot(U.col(j), U.col(j), m));
}

// Least squares min ||B x - y|| for several right-hand sides (columns of Y)
// through Householder QR of B; returns X (n x k).
Mat lstsq(const Mat& B, const Mat& Y) {
  Mat A = B;
  Vec tau;
  householder_qr(A, tau);
  const int m = A.r, n = A.c, k = Y.c;
  Mat X(n, k);
  Vec y(m);
  for (int col = 0; col < k; ++col) {
    for (int i = 0; i < m; ++i) y[i] = Y(i, col);
    for (int j = 0; j < n; ++j) {  // apply Q^T
      const double* v = A.col(j);
      double s = y[j];
      for (int i = j + 1; i < m; ++i) s += v[i] * y[i];
      s *= tau[j];
      y[j] -= s;
      for (int i = j + 1; i < m; ++i) y[i] -= s * v[i];
    }
    for (int j = n - 1; j >= 0; --j) {  // back substitution with R
      double s = y[j];
      for (int l = j + 1; l < n; ++l) s -= A(j, l) * X(l, col);
      X(j, col) = (A(j, j) != 0.0) ? s / A(j, j) : 0.0;
    }
  }
  return X;
}

// ---------------------------------------------------------------- complex eig
// Eigenvalues of a general complex n x n matrix (row-major H[i*n+j]):
// Householder reduction to upper Hessenberg, then shifted QR with Givens
// rotations and Wilkinson shifts, deflating from the bottom.
bool complex_eig(std::vector<cd> H, int n, std::vector<cd>& ev) {
  auto at = [&](int i, int j) -> cd& { return H[(size_t)i * n + j]; };
  for (int k = 0; k < n - 2; ++k) {  // Hessenberg reduction
    double nrm = 0.0;
    for (int i = k + 1; i < n; ++i) nrm += std::norm(at(i, k));
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    std::vector<cd> v(n, 0.0);
    const cd x0 = at(k + 1, k);
    const cd ph = std::abs(x0) > 0 ? x0 / std::abs(x0) : cd(1.0);
    v[k + 1] = x0 + ph * nrm;
    for (int i = k + 2; i < n; ++i) v[i] = at(i, k);
    double vn = 0.0;
    for (int i = k + 1; i < n; ++i) vn += std::norm(v[i]);
    if (vn == 0.0) continue;
    for (int j = 0; j < n; ++j) {  // H = (I - 2vv*/v*v) H
      cd s = 0.0;
      for (int i = k + 1; i < n; ++i) s += std::conj(v[i]) * at(i, j);
      s *= 2.0 / vn;
      for (int i = k + 1; i < n; ++i) at(i, j) -= s * v[i];
    }
    for (int i = 0; i < n; ++i) {  // H = H (I - 2vv*/v*v)
      cd s = 0.0;
      for (int j = k + 1; j < n; ++j) s += at(i, j) * v[j];
      s *= 2.0 / vn;
      for (int j = k + 1; j < n; ++j) at(i, j) -= s * std::conj(v[j]);
    }
  }
  ev.assign(n, 0.0);
  int hi = n - 1;
  int iter = 0;
  while (hi >= 0) {
    if (hi == 0) {
      ev[0] = at(0, 0);
      break;
    }
    int lo = hi;  // find the active block [lo, hi]
    while (lo > 0) {
      const double s = std::abs(at(lo, lo)) + std::abs(at(lo - 1, lo - 1));
      if (std::abs(at(lo, lo - 1)) <= 1e-15 * (s > 0 ? s : 1.0)) {
        at(lo, lo - 1) = 0.0;
        break;
      }
      --lo;
    }
    if (lo == hi) {
      ev[hi] = at(hi, hi);
      --hi;
      iter = 0;
      continue;
    }
    if (++iter > 300 * n) return false;
    // Wilkinson shift from the trailing 2x2
    const cd a = at(hi - 1, hi - 1), b = at(hi - 1, hi), c = at(hi, hi - 1), d = at(hi, hi);
    const cd tr = a + d, det = a * d - b * c;
    const cd disc = std::sqrt(tr * tr - 4.0 * det);
    const cd l1 = 0.5 * (tr + disc), l2 = 0.5 * (tr - disc);
    cd mu = std::abs(l1 - d) < std::abs(l2 - d) ? l1 : l2;
    if (iter % 11 == 10) mu += std::abs(at(hi, hi - 1)) * cd(0.75, 0.5);  // exceptional shift
    // QR step on the block via Givens rotations: H - mu I = Q R, H <- R Q + mu I
    std::vector<cd> gc(hi - lo), gs(hi - lo);
    for (int i = lo; i <= hi; ++i) at(i, i) -= mu;
    for (int k = lo; k < hi; ++k) {
      const cd x = at(k, k), y = at(k + 1, k);
      const double r = std::sqrt(std::norm(x) + std::norm(y));
      cd cc = 1.0, ss = 0.0;
      if (r > 0) {
        cc = x / r;
        ss = y / r;
      }
      gc[k - lo] = cc;
      gs[k - lo] = ss;
      for (int j = k; j < n; ++j) {  // rows k, k+1: G^* applied from the left
        const cd u = at(k, j), w = at(k + 1, j);
        at(k, j) = std::conj(cc) * u + std::conj(ss) * w;
        at(k + 1, j) = -ss * u + cc * w;
      }
    }
    for (int k = lo; k < hi; ++k) {  // columns k, k+1: G from the right
      const cd cc = gc[k - lo], ss = gs[k - lo];
      for (int i = 0; i <= std::min(k + 2, hi); ++i) {
        const cd u = at(i, k), w = at(i, k + 1);
        at(i, k) = u * cc + w * ss;
        at(i, k + 1) = -u * std::conj(ss) + w * std::conj(cc);
      }
    }
    for (int i = lo; i <= hi; ++i) at(i, i) += mu;
  }
  return true;
}

// ---------------------------------------------------------------- the fit
struct Fit {
  std::vector<cd> poles;       // conjugate-closed, pairs as (p, conj p), then reals
  double obj = INFINITY;
};

// real spanning set of span{[1], (lambda - xi)^-1} for the pole set
Mat spanning(const Vec& lam, const std::vector<cd>& xi, bool with_const) {
  int ncol = with_const ? 1 : 0;
  for (const cd& p : xi) ncol += (p.imag() > 0) ? 2 : (p.imag() == 0 ? 1 : 0);
  Mat B((int)lam.size(), ncol);
  int c = 0;
  if (with_const) {
    for (size_t i = 0; i < lam.size(); ++i) B(i, c) = 1.0;
    ++c;
  }
  for (const cd& p : xi) {
    if (p.imag() > 0) {
      for (size_t i = 0; i < lam.size(); ++i) {
        const cd w = 1.0 / (lam[i] - p);
        B(i, c) = w.real();
        B(i, c + 1) = w.imag();
      }
      c += 2;
    } else if (p.imag() == 0) {
      for (size_t i = 0; i < lam.size(); ++i) B(i, c) = 1.0 / (lam[i] - p.real());
      ++c;
    }
  }
  return B;
}

// real coefficients d over the spanning set -> (const, e_i) over all poles
void pf_coeffs(const std::vector<cd>& xi, const double* d, bool with_const, double& cst,
               std::vector<cd>& e) {
  size_t pos = 0;
  cst = with_const ? d[pos++] : 0.0;
  e.assign(xi.size(), 0.0);
  for (size_t n = 0; n < xi.size(); ++n) {
    if (xi[n].imag() > 0) {
      const double a = d[pos], b = d[pos + 1];
      e[n] = cd(0.5 * a, -0.5 * b);      // a Re w + b Im w = ((a - ib)/2) w + c.c.
      e[n + 1] = cd(0.5 * a, 0.5 * b);
      pos += 2;
      ++n;
    } else if (xi[n].imag() == 0) {
      e[n] = d[pos++];
    }
  }
}

// conjugate-closed, ordered (p, conj p) pairs then reals; reals >= 0 reflected
std::vector<cd> tidy(const std::vector<cd>& z, size_t m) {
  std::vector<cd> up, lowc;
  std::vector<double> re;
  for (const cd& r : z) {
    const double tol = 1e-10 * std::max(std::abs(r), 1e-300);
    if (std::fabs(r.imag()) <= tol) re.push_back(r.real());
    else if (r.imag() > 0) up.push_back(r);
    else lowc.push_back(std::conj(r));
  }
  std::vector<cd> pairs;
  std::vector<bool> used(lowc.size(), false);
  for (const cd& u : up) {
    int best = -1;
    double bd = INFINITY;
    for (size_t q = 0; q < lowc.size(); ++q)
      if (!used[q] && std::abs(u - lowc[q]) < bd) {
        bd = std::abs(u - lowc[q]);
        best = (int)q;
      }
    if (best >= 0) {
      used[best] = true;
      pairs.push_back(0.5 * (u + lowc[best]));
    } else {
      pairs.push_back(u);
    }
  }
  for (size_t q = 0; q < lowc.size(); ++q)
    if (!used[q]) pairs.push_back(lowc[q]);
  while (2 * pairs.size() + re.size() > m && !pairs.empty()) {  // split a near-real pair
    size_t q = 0;
    for (size_t i = 1; i < pairs.size(); ++i)
      if (std::fabs(pairs[i].imag()) < std::fabs(pairs[q].imag())) q = i;
    re.push_back(pairs[q].real());
    re.push_back(pairs[q].real() * (1 + 1e-8));
    pairs.erase(pairs.begin() + q);
  }
  std::vector<cd> out;
  for (const cd& p : pairs) {
    out.push_back(p);
    out.push_back(std::conj(p));
  }
  for (double r : re) out.push_back(cd(-std::fabs(r), 0.0));
  if (out.size() > m) out.resize(m);
  return out;
}

// residues for fixed poles: per channel LS, returns complex (npoles x K) and the objective
double residues_for(const Vec& lam, const Mat& F, const Vec& w, const std::vector<cd>& xi,
                    std::vector<cd>& res) {
  const Mat B = spanning(lam, xi, false);
  const Mat D = lstsq(B, F);   // (ncol x K)
  const int K = F.c, N = F.r;
  res.assign(xi.size() * (size_t)K, 0.0);
  double obj = 0.0;
  std::vector<cd> e;
  for (int j = 0; j < K; ++j) {
    double cst;
    pf_coeffs(xi, D.col(j), false, cst, e);
    for (size_t i = 0; i < xi.size(); ++i) res[i * K + j] = e[i];
    for (int l = 0; l < N; ++l) {
      double fit = 0.0;
      for (int c = 0; c < B.c; ++c) fit += B(l, c) * D(c, j);
      const double r = fit - F(l, j);
      obj += w[j] * r * r;
    }
  }
  return obj;
}

int fit_family(int K, const double* t, const double* wts, int m, int iters, std::vector<cd>& poles_x,
               std::vector<cd>& res_x, std::vector<int>& is_pair, double& uerr, std::string& err) {
  if (K < 1 || !t) {
    err = "need K >= 1 time channels";
    return TEM_EINVAL;
  }
  if (m < 2 || m > 2 * TEM_MAX_SHIFTS) {
    err = "degree must be in [2, 64]";
    return TEM_EINVAL;
  }
  double tmin = INFINITY, tmax = 0.0;
  for (int j = 0; j < K; ++j) {
    if (!(t[j] > 0.0)) {
      err = "time channels must be > 0";
      return TEM_EINVAL;
    }
    tmin = std::min(tmin, t[j]);
    tmax = std::max(tmax, t[j]);
  }
  const double ratio = tmax / tmin;
  Vec tau(K), w(K, 1.0);
  for (int j = 0; j < K; ++j) {
    tau[j] = t[j] / tmax;
    if (wts) w[j] = wts[j];
  }
  // surrogate (reading R3)
  const int Ns = 1200;
  Vec lam(Ns);
  lam[0] = 0.0;
  const double l0 = -3.0, l1 = std::log10(ratio) + 3.0;
  for (int i = 1; i < Ns; ++i) lam[i] = std::pow(10.0, l0 + (l1 - l0) * (i - 1) / (Ns - 2));
  Mat F(Ns, K);
  for (int j = 0; j < K; ++j)
    for (int i = 0; i < Ns; ++i) F(i, j) = std::exp(-tau[j] * lam[i]);
  // deterministic start: pairs with log-spaced moduli in [1, 10 ratio] at arg 2 pi / 3
  std::vector<cd> xi;
  const int npair = m / 2;
  for (int q = 0; q < npair; ++q) {
    const double mod = std::pow(10.0, npair > 1 ? std::log10(10.0 * ratio) * q / (npair - 1) : 0.0);
    const cd z = std::polar(mod, 2.0 * M_PI / 3.0);
    xi.push_back(z);
    xi.push_back(std::conj(z));
  }
  if (m % 2) xi.push_back(cd(-std::sqrt(10.0 * ratio), 0.0));

  Fit best;
  std::vector<cd> res;
  for (int it = 0; it <= iters; ++it) {
    const double obj = residues_for(lam, F, w, xi, res);
    if (obj < best.obj) {
      best.obj = obj;
      best.poles = xi;
    }
    if (it == iters) break;
    // 1. bases
    const Mat B = spanning(lam, xi, true);
    Mat V, RB;
    orth(B, V, RB);
    Mat Wb, RW;
    orth(spanning(lam, xi, false), Wb, RW);
    // 2. stacked sqrt(w_j) (I - W W^T) F_j V, smallest right singular vector
    const int n1 = V.c;
    Mat Cst((int)Ns * K, n1);
    Vec tmp(Ns), proj(Wb.c);
    for (int j = 0; j < K; ++j) {
      const double sw = std::sqrt(w[j]);
      for (int c = 0; c < n1; ++c) {
        for (int i = 0; i < Ns; ++i) tmp[i] = F(i, j) * V(i, c);
        for (int q = 0; q < Wb.c; ++q) proj[q] = dot(Wb.col(q), tmp.data(), Ns);
        for (int q = 0; q < Wb.c; ++q) {
          const double* wq = Wb.col(q);
          for (int i = 0; i < Ns; ++i) tmp[i] -= proj[q] * wq[i];
        }
        double* dst = Cst.col(c) + (size_t)j * Ns;
        for (int i = 0; i < Ns; ++i) dst[i] = sw * tmp[i];
      }
    }
    Vec tau_c;
    householder_qr(Cst, tau_c);
    Mat R(n1, n1);
    for (int c = 0; c < n1; ++c)
      for (int r = 0; r <= c; ++r) R(r, c) = Cst(r, c);
    Mat Vs;
    Vec sv;
    jacobi_svd(R, Vs, sv);
    int jmin = 0;
    for (int q = 1; q < n1; ++q)
      if (sv[q] < sv[jmin]) jmin = q;
    // 3. coefficients over the spanning set: d = RB^-1 c
    Vec d(n1);
    for (int r = n1 - 1; r >= 0; --r) {
      double s = Vs(r, jmin);
      for (int l = r + 1; l < n1; ++l) s -= RB(r, l) * d[l];
      d[r] = RB(r, r) != 0.0 ? s / RB(r, r) : 0.0;
    }
    double cst;
    std::vector<cd> e;
    pf_coeffs(xi, d.data(), true, cst, e);
    if (cst == 0.0) break;
    const int mm = (int)xi.size();
    std::vector<cd> Hm((size_t)mm * mm);
    for (int r = 0; r < mm; ++r)
      for (int c = 0; c < mm; ++c) Hm[(size_t)r * mm + c] = (r == c ? xi[r] : 0.0) - e[c] / cst;
    std::vector<cd> roots;
    if (!complex_eig(Hm, mm, roots)) break;
    std::vector<cd> nxt = tidy(roots, (size_t)m);
    bool ok = nxt.size() == (size_t)m;
    for (const cd& p : nxt) ok = ok && std::isfinite(p.real()) && std::isfinite(p.imag());
    if (!ok) break;
    xi = nxt;
  }
  xi = best.poles;
  residues_for(lam, F, w, xi, res);
  // uniform error on {0} U logspace(-4, log10 ratio + 5) (eq:uniform_error)
  uerr = 0.0;
  const int Ng = 4000;
  for (int j = 0; j < K; ++j) {
    double ej = 0.0;
    for (int g = 0; g < Ng; ++g) {
      const double y = g == 0 ? 0.0 : std::pow(10.0, -4.0 + (std::log10(ratio) + 9.0) * (g - 1) / (Ng - 2));
      cd r = 0.0;
      for (size_t i = 0; i < xi.size(); ++i) r += res[i * K + j] / (y - xi[i]);
      ej = std::max(ej, std::fabs(std::exp(-tau[j] * y) - r.real()));
    }
    uerr = std::max(uerr, w[j] * ej);
  }
  // representatives (one per pair, Im > 0, by modulus; then reals) in the physical variable
  std::vector<int> idx;
  for (size_t i = 0; i < xi.size(); ++i)
    if (xi[i].imag() > 0) idx.push_back((int)i);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return std::abs(xi[a]) < std::abs(xi[b]); });
  const size_t npairs = idx.size();
  for (size_t i = 0; i < xi.size(); ++i)
    if (xi[i].imag() == 0) idx.push_back((int)i);
  poles_x.clear();
  res_x.clear();
  is_pair.clear();
  for (size_t q = 0; q < idx.size(); ++q) {
    poles_x.push_back(xi[idx[q]] / tmax);
    for (int j = 0; j < K; ++j) res_x.push_back(res[(size_t)idx[q] * K + j] / tmax);
    is_pair.push_back(q < npairs ? 1 : 0);
  }
  return TEM_OK;
}

}  // namespace

void tem_set_error(const std::string& msg);   // tem_b200.cu

extern "C" int tem_fit_family(int K, const double* t, const double* w, int m, int iters, int* n_rep,
                              double* shifts, double* residues, int* is_pair, double* uniform_error) {
  if (!n_rep || !shifts || !residues || !is_pair) {
    tem_set_error("tem_fit_family: null pointer");
    return TEM_EINVAL;
  }
  std::vector<cd> px, rx;
  std::vector<int> ip;
  double uerr = 0.0;
  std::string err;
  const int rc = fit_family(K, t, w, m, iters > 0 ? iters : 12, px, rx, ip, uerr, err);
  if (rc != TEM_OK) {
    tem_set_error("tem_fit_family: " + err);
    return rc;
  }
  *n_rep = (int)px.size();
  if (*n_rep > TEM_MAX_SHIFTS) {   // the solver's batch limit (real poles need one system each)
    tem_set_error("tem_fit_family: the family needs " + std::to_string(*n_rep) + " shifted systems (" +
                  std::to_string(m) + " poles with real ones), more than TEM_MAX_SHIFTS = " +
                  std::to_string(TEM_MAX_SHIFTS) + "; lower the degree");
    return TEM_EINVAL;
  }
  for (size_t q = 0; q < px.size(); ++q) {
    shifts[2 * q] = -px[q].real();       // s = -xi
    shifts[2 * q + 1] = -px[q].imag();
    is_pair[q] = ip[q];
  }
  for (size_t i = 0; i < rx.size(); ++i) {
    residues[2 * i] = rx[i].real();
    residues[2 * i + 1] = rx[i].imag();
  }
  if (uniform_error) *uniform_error = uerr;
  return TEM_OK;
}
