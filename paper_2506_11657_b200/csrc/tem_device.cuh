// tem_device.cuh -- device-side building blocks of the B200 TEM hot path.
//
// Yee / finite-integration curl-curl on the node-owned edge layout of
// include/tem_b200.h (reading R1):
//   (K u)_a(m) = W_d(m) C_d(m) - W_d(m-e_b) C_d(m-e_b) - W_b(m) C_b(m) + W_b(m-e_d) C_b(m-e_d)
// for the edge along axis a at node m, (a, b, d) a cyclic permutation of
// (x, y, z), where C_d(m') is the circulation around the face normal to d
// with lower corner m' (right-hand rule about +d):
//   C_d(m') = u_a(m') + u_b(m'+e_a) - u_a(m'+e_b) - u_b(m')
//   C_b(m') = u_d(m') + u_a(m'+e_d) - u_d(m'+e_a) - u_a(m')
// and W_d(m') = hdual_d[m'_d] / (mu0 h_a[m'_a] h_b[m'_b]).  This is
// K = T^T W T (§2.2 [K]_ij = (mu^-1 curl Phi_j, curl Phi_i)) written
// as a 13-point gather; nothing is assembled.  The gather itself lives in
// tem_sweep.cuh (shared-memory plane ring); this header holds the grid,
// complex helpers and the per-edge face weights.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tem {

constexpr double kMu0 = 4e-7 * 3.14159265358979323846;  // PAPER.md §2.1

struct Grid {
  int n[3];               // cells per axis
  long long st[3];        // node strides: 1, nx+1, (nx+1)(ny+1)
  long long Nn;           // nodes
  // Real-arithmetic shifts keep their COCG vectors as fp64 edge vectors whose
  // node rows carry one leading zero column and are padded to an even length
  // px: slot c * NnP + (k (ny+1) + j) px + i + 1, stored at the start of the
  // shift's complex slot region (8 * 3 NnP <= 16 * 3 Nn bytes).  Even px
  // makes every TMA global stride a multiple of 16 B; the leading column
  // puts the halo tile origin (node tx0 - 1, column tx0) on an even element,
  // because a TMA box must start on a 16-byte boundary of the innermost
  // dimension (measured: odd fp64 coordinates fault on sm_100a).
  int px;                 // nx + 2 rounded up to even
  long long NnP;          // px (ny+1) (nz+1)
  const double* ih[3];    // 1 / h_a[i], i < n_a                     (device)
  const double* hdm[3];   // hdual_a[i] / mu0, i = 0..n_a             (device)
};

// ---------------------------------------------------------------- complex
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a + b*c
__device__ __forceinline__ double2 cfma(double2 b, double2 c, double2 a) {
  return make_double2(fma(b.x, c.x, fma(-b.y, c.y, a.x)), fma(b.x, c.y, fma(b.y, c.x, a.y)));
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double inv = 1.0 / fma(b.x, b.x, b.y * b.y);
  return make_double2(fma(a.x, b.x, a.y * b.y) * inv, fma(a.y, b.x, -a.x * b.y) * inv);
}
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }
// 1/b: hardware reciprocal seed + two Newton steps on |b|^2 (no slow-path
// branch of the IEEE division; relative error ~1 ulp for normal |b|^2)
__device__ __forceinline__ double2 crcp(double2 b, double& n) {
  n = fma(b.x, b.x, b.y * b.y);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(n));
  r = fma(r, fma(-n, r, 1.0), r);
  r = fma(r, fma(-n, r, 1.0), r);
  return make_double2(b.x * r, -b.y * r);
}
__device__ __forceinline__ double2 crcp(double2 b) {
  double n;
  return crcp(b, n);
}
__device__ __forceinline__ double2 csq(double2 a) { return make_double2(fma(a.x, a.x, -a.y * a.y), 2.0 * a.x * a.y); }
__device__ __forceinline__ double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

// The same operations on real values: a shift with a real pole (footnote to
// eq:rmj) has a real SPD system K + s M and a real right-hand side,
// so its COCG runs in real arithmetic (8 B per value, a quarter of the FP64
// work).  Kernels are written once over the value type V = double2 | double.
__device__ __forceinline__ double cadd(double a, double b) { return a + b; }
__device__ __forceinline__ double csub(double a, double b) { return a - b; }
__device__ __forceinline__ double cscale(double s, double a) { return s * a; }
__device__ __forceinline__ double cmul(double a, double b) { return a * b; }
__device__ __forceinline__ double cfma(double b, double c, double a) { return fma(b, c, a); }
__device__ __forceinline__ double cdiv(double a, double b) { return a / b; }
__device__ __forceinline__ double csq(double a) { return a * a; }
__device__ __forceinline__ double cabs2(double a) { return a * a; }
__device__ __forceinline__ double crcp(double b, double& n) {
  n = b * b;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  r = fma(r, fma(-b, r, 1.0), r);
  return fma(r, fma(-b, r, 1.0), r);
}

// Two real shifts in one complex-sized slot (R16): the systems
// K + s_A M and K + s_B M of two real poles are real and independent, and K, M
// are real, so their COCG vectors travel as the two components of one
// 16-byte value through the complex layout, tensor maps and tiles, with
// every operation component-wise (no cross terms: fewer FP64 operations than
// a complex shift at the same bytes).
struct dpair {
  double x, y;
};
__device__ __forceinline__ dpair make_dpair(double x, double y) {
  dpair r;
  r.x = x;
  r.y = y;
  return r;
}
__device__ __forceinline__ dpair cadd(dpair a, dpair b) { return make_dpair(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ dpair csub(dpair a, dpair b) { return make_dpair(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ dpair cscale(double s, dpair a) { return make_dpair(s * a.x, s * a.y); }
__device__ __forceinline__ dpair cmul(dpair a, dpair b) { return make_dpair(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ dpair cfma(dpair b, dpair c, dpair a) {
  return make_dpair(fma(b.x, c.x, a.x), fma(b.y, c.y, a.y));
}
__device__ __forceinline__ dpair cdiv(dpair a, dpair b) { return make_dpair(a.x / b.x, a.y / b.y); }
__device__ __forceinline__ dpair csq(dpair a) { return make_dpair(a.x * a.x, a.y * a.y); }
__device__ __forceinline__ dpair crcp(dpair b, dpair& n) {
  double nx, ny;
  const double rx = crcp(b.x, nx), ry = crcp(b.y, ny);
  n = make_dpair(nx, ny);
  return make_dpair(rx, ry);
}

// acc + s * a for a real scalar s (component-wise fma)
__device__ __forceinline__ double2 sfma(double s, double2 a, double2 acc) {
  return make_double2(fma(s, a.x, acc.x), fma(s, a.y, acc.y));
}
__device__ __forceinline__ double sfma(double s, double a, double acc) { return fma(s, a, acc); }
__device__ __forceinline__ dpair sfma(double s, dpair a, dpair acc) {
  return make_dpair(fma(s, a.x, acc.x), fma(s, a.y, acc.y));
}

template <typename V>
struct VT;
template <>
struct VT<double2> {
  static constexpr bool kReal = false;
  static constexpr bool kPair = false;
  typedef double R;
  __device__ __forceinline__ static double2 diag(double kd, double m, double2 sh) {
    return make_double2(kd + m * sh.x, m * sh.y);
  }
  __device__ __forceinline__ static R rzero() { return 0.0; }
  __device__ __forceinline__ static R rone() { return 1.0; }
  __device__ __forceinline__ static R abs2(double2 v) { return fma(v.x, v.x, v.y * v.y); }
  __device__ __forceinline__ static R rfma(R a, R b, R c) { return fma(a, b, c); }
  __device__ __forceinline__ static bool small_beta(double2 beta, double2, double2, double thr) {
    return fma(beta.x, beta.x, beta.y * beta.y) < thr;
  }
  __device__ __forceinline__ static double2 div0(double2 a, double2 b) { return cdiv(a, b); }
  __device__ __forceinline__ static double r0(R r) { return r; }
  __device__ __forceinline__ static double r1(R) { return 0.0; }
  __device__ __forceinline__ static double2 zero() { return make_double2(0.0, 0.0); }
  __device__ __forceinline__ static double2 from(double2 v) { return v; }     // scalar state -> V
  __device__ __forceinline__ static double2 cplx(double2 v) { return v; }     // V -> complex
  __device__ __forceinline__ static double2 make(double re, double im) { return make_double2(re, im); }
  __device__ __forceinline__ static double re(double2 v) { return v.x; }
  __device__ __forceinline__ static double im(double2 v) { return v.y; }
};
template <>
struct VT<dpair> {
  static constexpr bool kReal = false;   // complex layout (16-byte slots)
  static constexpr bool kPair = true;
  typedef dpair R;                       // squared magnitudes, one per component
  __device__ __forceinline__ static dpair zero() { return make_dpair(0.0, 0.0); }
  __device__ __forceinline__ static dpair from(double2 v) { return make_dpair(v.x, v.y); }   // packed (A, B)
  __device__ __forceinline__ static double2 cplx(dpair v) { return make_double2(v.x, v.y); }  // packed (A, B)
  __device__ __forceinline__ static dpair diag(double kd, double m, dpair sh) {
    return make_dpair(fma(m, sh.x, kd), fma(m, sh.y, kd));
  }
  __device__ __forceinline__ static R rzero() { return make_dpair(0.0, 0.0); }
  __device__ __forceinline__ static R rone() { return make_dpair(1.0, 1.0); }
  __device__ __forceinline__ static R abs2(dpair v) { return make_dpair(v.x * v.x, v.y * v.y); }
  __device__ __forceinline__ static R rfma(R a, R b, R c) { return make_dpair(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y)); }
  // R11: p_{i-1} must be re-read when a component that still moves x has a small beta;
  // a frozen member (alpha = alpha_prev = 0, beta = 0) adds nothing to x and does not count
  __device__ __forceinline__ static bool small_beta(dpair beta, dpair alpha, dpair alpha_prev, double thr) {
    const bool mx = alpha.x != 0.0 || alpha_prev.x != 0.0, my = alpha.y != 0.0 || alpha_prev.y != 0.0;
    return (mx && beta.x * beta.x < thr) || (my && beta.y * beta.y < thr);
  }
  __device__ __forceinline__ static dpair div0(dpair a, dpair b) {   // a / b, 0 where b = 0
    return make_dpair(b.x != 0.0 ? a.x / b.x : 0.0, b.y != 0.0 ? a.y / b.y : 0.0);
  }
  __device__ __forceinline__ static double r0(R r) { return r.x; }
  __device__ __forceinline__ static double r1(R r) { return r.y; }
};
template <>
struct VT<double> {
  static constexpr bool kReal = true;
  static constexpr bool kPair = false;
  typedef double R;
  __device__ __forceinline__ static double diag(double kd, double m, double sh) { return fma(m, sh, kd); }
  __device__ __forceinline__ static R rzero() { return 0.0; }
  __device__ __forceinline__ static R rone() { return 1.0; }
  __device__ __forceinline__ static R abs2(double v) { return v * v; }
  __device__ __forceinline__ static R rfma(R a, R b, R c) { return fma(a, b, c); }
  __device__ __forceinline__ static bool small_beta(double beta, double, double, double thr) {
    return beta * beta < thr;
  }
  __device__ __forceinline__ static double div0(double a, double b) { return a / b; }
  __device__ __forceinline__ static double r0(R r) { return r; }
  __device__ __forceinline__ static double r1(R) { return 0.0; }
  __device__ __forceinline__ static double zero() { return 0.0; }
  __device__ __forceinline__ static double from(double2 v) { return v.x; }
  __device__ __forceinline__ static double2 cplx(double v) { return make_double2(v, 0.0); }
  __device__ __forceinline__ static double make(double re, double) { return re; }
  __device__ __forceinline__ static double re(double v) { return v; }
  __device__ __forceinline__ static double im(double) { return 0.0; }
};

// Face weights of the four faces around edge (A, pos): W_d(m), W_d(m-e_b), W_b(m), W_b(m-e_d).
struct EdgeWeights {
  double wd0, wd1, wb0, wb1;
  __device__ __forceinline__ double diag() const { return wd0 + wd1 + wb0 + wb1; }
};

template <int A>
__device__ __forceinline__ EdgeWeights edge_weights(const Grid& g, const int pos[3]) {
  constexpr int B = (A + 1) % 3, D = (A + 2) % 3;
  const double iha = __ldg(g.ih[A] + pos[A]);
  const double hdD = __ldg(g.hdm[D] + pos[D]);
  const double hdB = __ldg(g.hdm[B] + pos[B]);
  EdgeWeights w;
  w.wd0 = hdD * iha * __ldg(g.ih[B] + pos[B]);
  w.wd1 = hdD * iha * __ldg(g.ih[B] + pos[B] - 1);
  w.wb0 = hdB * iha * __ldg(g.ih[D] + pos[D]);
  w.wb1 = hdB * iha * __ldg(g.ih[D] + pos[D] - 1);
  return w;
}

__device__ __forceinline__ void node_pos(const Grid& g, long long n, int pos[3]) {
  const long long nx1 = g.n[0] + 1, ny1 = g.n[1] + 1;
  const long long q = n / nx1;
  pos[0] = (int)(n - q * nx1);
  pos[1] = (int)(q % ny1);
  pos[2] = (int)(q / ny1);
}

}  // namespace tem
