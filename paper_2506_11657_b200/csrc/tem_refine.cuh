// tem_refine.cuh -- accuracy kernels of the forward: the residual of the
// shifted systems in double-double arithmetic, and the reductions the
// channel-aware refinement reads (reading R13).
//
// Why: u(t_j) = sum_i w_i Re(alpha_ij x_i) (§3.2 eq:rmj) is, at late
// channels, a sum of terms far larger than the result, so the channel error
// is the solve error amplified (measured on the 14M config: 4.6e7 x the
// relative residual).  An fp64 COCG stalls at a true residual ~1e-14, which
// leaves late channels at ~1e-6.  Iterative refinement -- r = f - (K + s M) x
// evaluated in double-double (so r is exact to ~1e-32 relative to the terms
// that cancel in it), A delta = r solved by the same batched COCG, x += delta
// -- drives the error of x below what the fp64 recursion can reach.
#pragma once
#include "tem_device.cuh"

namespace tem {

// ------------------------------------------------------- double-double
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo = fma(a.lo, b, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_from(double a) { return {a, 0.0}; }

struct cdd {
  dd re, im;
};
__device__ __forceinline__ cdd cdd_from(double2 a) { return {dd_from(a.x), dd_from(a.y)}; }
__device__ __forceinline__ cdd cdd_add(cdd a, cdd b) { return {dd_add(a.re, b.re), dd_add(a.im, b.im)}; }
__device__ __forceinline__ cdd cdd_sub(cdd a, cdd b) { return {dd_add(a.re, dd_neg(b.re)), dd_add(a.im, dd_neg(b.im))}; }
__device__ __forceinline__ cdd cdd_scale(cdd a, double w) { return {dd_mul_d(a.re, w), dd_mul_d(a.im, w)}; }
// circulation a + b - c - d of four fp64 values, exact to dd
__device__ __forceinline__ cdd circ4(double2 a, double2 b, double2 c, double2 d) {
  cdd r = {two_sum(a.x, b.x), two_sum(a.y, b.y)};
  r = cdd_sub(r, cdd_from(c));
  return cdd_sub(r, cdd_from(d));
}

// value of complex shift-block vector v at edge (c, i, j, k), 0 outside the grid
__device__ __forceinline__ double2 vat(const Grid& g, const double2* v, int c, int i, int j, int k) {
  if (i < 0 || j < 0 || k < 0 || i > g.n[0] || j > g.n[1] || k > g.n[2]) return czero();
  return __ldg(v + c * g.Nn + ((long long)k * (g.n[1] + 1) + j) * (g.n[0] + 1) + i);
}

// r_s = f - (K + s M) x_s on every free edge (0 elsewhere), in double-double,
// rounded to fp64; the face weights are formed with the same fp64 products as
// the sweeps (stencil3p), so K is the operator the solver iterates with.
// Grid (blocks, S): blockIdx.y = shift slot, list[y] = shift.  Partial sums
// of |r|^2 per (slot, block) into part[y * gridDim.x + x].
struct ResidArgs {
  Grid g;
  const double* mass;
  const double* f;        // real [3][Nn]
  const double2* x;       // shift block
  double2* r;             // shift block (output; only the listed shifts are written)
  double* part;           // [nlist][gridDim.x]
  double* part_abs;       // [nlist][gridDim.x]: || |A| |x| ||^2 partials (rounding floor), or NULL
  int list[32];
  double2 shifts[32];     // shift of list[y]
};

__global__ void __launch_bounds__(256) k_resid_dd(const __grid_constant__ ResidArgs A) {
  const Grid& g = A.g;
  const int y = blockIdx.y, s = A.list[y];
  const double2 sh = A.shifts[y];
  const double2* x = A.x + (long long)s * 3 * g.Nn;
  double2* r = A.r + (long long)s * 3 * g.Nn;
  const int nx1 = g.n[0] + 1, ny1 = g.n[1] + 1;
  double acc = 0.0, acc_abs = 0.0;
  auto ab = [](double2 v) { return fabs(v.x) + fabs(v.y); };
  for (long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x; n < g.Nn;
       n += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(n % nx1);
    const int j = (int)((n / nx1) % ny1);
    const int k = (int)(n / ((long long)nx1 * ny1));
    // column / plane factors exactly as in make_column_ij / stencil3p
    const bool in_ij = i < g.n[0] && j < g.n[1];
    const double ihx = in_ij ? __ldg(g.ih[0] + i) : 0.0;
    const double ihxm = (in_ij && i >= 1) ? __ldg(g.ih[0] + i - 1) : 0.0;
    const double ihy = in_ij ? __ldg(g.ih[1] + j) : 0.0;
    const double ihym = (in_ij && j >= 1) ? __ldg(g.ih[1] + j - 1) : 0.0;
    const double hdx = in_ij ? __ldg(g.hdm[0] + i) : 0.0;
    const double hdy = in_ij ? __ldg(g.hdm[1] + j) : 0.0;
    const double ihz = k < g.n[2] ? __ldg(g.ih[2] + k) : 0.0;
    const double ihzm = k >= 1 ? __ldg(g.ih[2] + k - 1) : 0.0;
    const double hdz = k < g.n[2] ? __ldg(g.hdm[2] + k) : 0.0;
    const double pxy = ihx * ihy, pxym = ihx * ihym, pxmy = ihxm * ihy;
    const double cyx = hdy * ihx, cyxm = hdy * ihxm, cxy = hdx * ihy, cxym = hdx * ihym;
    const double wz = hdz * pxy, wz_y = hdz * pxym, wz_x = hdz * pxmy;
    const double wy = cyx * ihz, wy_z = cyx * ihzm, wy_x = cyxm * ihz;
    const double wx = cxy * ihz, wx_z = cxy * ihzm, wx_y = cxym * ihz;
    auto X = [&](int di, int dj, int dk) { return vat(g, x, 0, i + di, j + dj, k + dk); };
    auto Y = [&](int di, int dj, int dk) { return vat(g, x, 1, i + di, j + dj, k + dk); };
    auto Z = [&](int di, int dj, int dk) { return vat(g, x, 2, i + di, j + dj, k + dk); };
    const bool fr[3] = {in_ij && i < g.n[0] && j >= 1 && j <= g.n[1] - 1 && k >= 1 && k <= g.n[2] - 1,
                        in_ij && i >= 1 && i <= g.n[0] - 1 && j < g.n[1] && k >= 1 && k <= g.n[2] - 1,
                        in_ij && i >= 1 && i <= g.n[0] - 1 && j >= 1 && j <= g.n[1] - 1 && k < g.n[2]};
    cdd q[3] = {};
    // (K v)_x = Gz - Gz(m-ey) - Gy + Gy(m-ez); (K v)_y = Gx - Gx(m-ez) - Gz + Gz(m-ex);
    // (K v)_z = Gy - Gy(m-ex) - Gx + Gx(m-ey), G = W * circulation (tem_device.cuh)
    if (fr[0] || fr[1]) {
      const cdd Gz = cdd_scale(circ4(X(0, 0, 0), Y(1, 0, 0), X(0, 1, 0), Y(0, 0, 0)), wz);
      q[0] = Gz;
      q[1] = {dd_neg(Gz.re), dd_neg(Gz.im)};
    }
    if (fr[0] || fr[2]) {
      const cdd Gy = cdd_scale(circ4(Z(0, 0, 0), X(0, 0, 1), Z(1, 0, 0), X(0, 0, 0)), wy);
      q[0] = cdd_sub(q[0], Gy);
      q[2] = Gy;
    }
    if (fr[1] || fr[2]) {
      const cdd Gx = cdd_scale(circ4(Y(0, 0, 0), Z(0, 1, 0), Y(0, 0, 1), Z(0, 0, 0)), wx);
      q[1] = cdd_add(q[1], Gx);
      q[2] = cdd_sub(q[2], Gx);
    }
    if (fr[0]) {
      q[0] = cdd_sub(q[0], cdd_scale(circ4(X(0, -1, 0), Y(1, -1, 0), X(0, 0, 0), Y(0, -1, 0)), wz_y));
      q[0] = cdd_add(q[0], cdd_scale(circ4(Z(0, 0, -1), X(0, 0, 0), Z(1, 0, -1), X(0, 0, -1)), wy_z));
    }
    if (fr[1]) {
      q[1] = cdd_add(q[1], cdd_scale(circ4(X(-1, 0, 0), Y(0, 0, 0), X(-1, 1, 0), Y(-1, 0, 0)), wz_x));
      q[1] = cdd_sub(q[1], cdd_scale(circ4(Y(0, 0, -1), Z(0, 1, -1), Y(0, 0, 0), Z(0, 0, -1)), wx_z));
    }
    if (fr[2]) {
      q[2] = cdd_sub(q[2], cdd_scale(circ4(Z(-1, 0, 0), X(-1, 0, 1), Z(0, 0, 0), X(-1, 0, 0)), wy_x));
      q[2] = cdd_add(q[2], cdd_scale(circ4(Y(0, -1, 0), Z(0, 0, 0), Y(0, -1, 1), Z(0, -1, 0)), wx_y));
    }
    // (|K| |x|)_e with |x| taken as |Re| + |Im|: the scale of the rounding
    // floor of the residual, eps || |A| |x| || (the residual of x rounded)
    double qa[3] = {0.0, 0.0, 0.0};
    if (A.part_abs) {
      auto a4 = [&](double2 a, double2 b, double2 c, double2 d) { return ab(a) + ab(b) + ab(c) + ab(d); };
      const double tz = wz * a4(X(0, 0, 0), Y(1, 0, 0), X(0, 1, 0), Y(0, 0, 0));
      const double ty = wy * a4(Z(0, 0, 0), X(0, 0, 1), Z(1, 0, 0), X(0, 0, 0));
      const double tx = wx * a4(Y(0, 0, 0), Z(0, 1, 0), Y(0, 0, 1), Z(0, 0, 0));
      qa[0] = tz + ty + wz_y * a4(X(0, -1, 0), Y(1, -1, 0), X(0, 0, 0), Y(0, -1, 0)) +
              wy_z * a4(Z(0, 0, -1), X(0, 0, 0), Z(1, 0, -1), X(0, 0, -1));
      qa[1] = tz + tx + wz_x * a4(X(-1, 0, 0), Y(0, 0, 0), X(-1, 1, 0), Y(-1, 0, 0)) +
              wx_z * a4(Y(0, 0, -1), Z(0, 1, -1), Y(0, 0, 0), Z(0, 0, -1));
      qa[2] = ty + tx + wy_x * a4(Z(-1, 0, 0), X(-1, 0, 1), Z(0, 0, 0), X(-1, 0, 0)) +
              wx_y * a4(Y(0, -1, 0), Z(0, 0, 0), Y(0, -1, 1), Z(0, -1, 0));
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const long long slot = c * g.Nn + n;
      double2 out = czero();
      if (fr[c]) {
        const double m = __ldg(A.mass + slot);
        const double2 xv = __ldg(x + slot);
        // s (m x): m x exact (two products), then the complex product with s
        const dd mr = two_prod(m, xv.x), mi = two_prod(m, xv.y);
        const dd smr = dd_add(dd_mul_d(mr, sh.x), dd_neg(dd_mul_d(mi, sh.y)));
        const dd smi = dd_add(dd_mul_d(mi, sh.x), dd_mul_d(mr, sh.y));
        const dd rr = dd_add(dd_from(__ldg(A.f + slot)), dd_neg(dd_add(q[c].re, smr)));
        const dd ri = dd_neg(dd_add(q[c].im, smi));
        out = make_double2(rr.hi + rr.lo, ri.hi + ri.lo);
        acc = fma(out.x, out.x, fma(out.y, out.y, acc));
        const double ta = qa[c] + (fabs(sh.x) + fabs(sh.y)) * m * ab(xv);
        acc_abs = fma(ta, ta, acc_abs);
      }
      r[slot] = out;
    }
  }
  // block sum, fixed order
  __shared__ double red[2][8];
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_down_sync(0xffffffffu, acc, o);
    acc_abs += __shfl_down_sync(0xffffffffu, acc_abs, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = acc;
    red[1][threadIdx.x >> 5] = acc_abs;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[threadIdx.x][w];
    if (threadIdx.x == 0) A.part[(long long)y * gridDim.x + blockIdx.x] = t;
    else if (A.part_abs) A.part_abs[(long long)y * gridDim.x + blockIdx.x] = t;
  }
}

// Per listed shift: x_s += d_s (complex shift blocks), and the M-weighted
// statistics of the correction d_s that the channel-aware stopping rule
// needs: sum m (Re d)^2, sum m (Im d)^2, sum m Re d Im d, sum m |x_s|^2
// (after the update) -> part[((y * 4) + t) * gridDim.x + x].
struct UpdateArgs {
  long long Nn;
  const double* mass;
  double2* x;
  const double2* d;
  double* part;
  int list[32];
};

__global__ void __launch_bounds__(256) k_refine_update(const __grid_constant__ UpdateArgs A) {
  const int y = blockIdx.y, s = A.list[y];
  double2* x = A.x + (long long)s * 3 * A.Nn;
  const double2* d = A.d + (long long)s * 3 * A.Nn;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < 3 * A.Nn;
       e += (long long)gridDim.x * blockDim.x) {
    const double m = __ldg(A.mass + e);
    const double2 dv = __ldg(d + e);
    const double2 xv = cadd(x[e], dv);
    x[e] = xv;
    a0 = fma(m * dv.x, dv.x, a0);
    a1 = fma(m * dv.y, dv.y, a1);
    a2 = fma(m * dv.x, dv.y, a2);
    a3 = fma(m, cabs2(xv), a3);
  }
  __shared__ double red[4][8];
  double v[4] = {a0, a1, a2, a3};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    for (int o = 16; o > 0; o >>= 1) v[t] += __shfl_down_sync(0xffffffffu, v[t], o);
    if ((threadIdx.x & 31) == 0) red[t][threadIdx.x >> 5] = v[t];
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[threadIdx.x][w];
    A.part[((long long)y * 4 + threadIdx.x) * gridDim.x + blockIdx.x] = t;
  }
}

// ||u_k||_M^2 = sum_e m_e u_k[e]^2 per channel k (blockIdx.y) of the channel
// fields u[K][3][Nn] -> part[k * gridDim.x + x].
__global__ void __launch_bounds__(256) k_channel_mnorm(long long nslots, const double* __restrict__ mass,
                                                       const double* __restrict__ u, double* part) {
  const double* uk = u + (long long)blockIdx.y * nslots;
  double acc = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nslots;
       e += (long long)gridDim.x * blockDim.x) {
    const double v = __ldg(uk + e);
    acc = fma(__ldg(mass + e) * v, v, acc);
  }
  __shared__ double red[8];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[(long long)blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// Net change of every channel in a refinement round (reading R13): per
// channel k, ||sum_s w_s Re(res[k][s] d_s)||_M^2 over the correction block d
// (shift block; d_s = 0 for shifts not refined this round) -> part[k][x].
// The per-shift contributions cancel in late channels exactly as the
// channel fields do (eq:rmj), so the NET change, not the sum of |terms|, is
// the measure of how far the channel moved.  kCB channels per block row
// (blockIdx.y); d is re-read once per row of channels.
constexpr int kCB = 8;
__global__ void __launch_bounds__(256) k_dsynth_mnorm(long long nslots, const double* __restrict__ mass, int S,
                                                      int K, const double2* __restrict__ res,
                                                      const double* __restrict__ w, const double2* __restrict__ d,
                                                      double* part) {
  __shared__ double2 sres[kCB * 32];
  const int k0 = blockIdx.y * kCB;
  for (int i = threadIdx.x; i < kCB * S; i += blockDim.x) {
    const int c = i / S, s = i - c * S;
    const double2 a = k0 + c < K ? res[(k0 + c) * S + s] : czero();
    sres[i] = make_double2(w[s] * a.x, w[s] * a.y);
  }
  __syncthreads();
  double acc[kCB];
#pragma unroll
  for (int c = 0; c < kCB; ++c) acc[c] = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nslots;
       e += (long long)gridDim.x * blockDim.x) {
    const double m = __ldg(mass + e);
    if (m == 0.0) continue;
    double v[kCB];
#pragma unroll
    for (int c = 0; c < kCB; ++c) v[c] = 0.0;
    for (int s = 0; s < S; ++s) {
      const double2 dv = __ldg(d + (long long)s * nslots + e);
#pragma unroll
      for (int c = 0; c < kCB; ++c) {
        const double2 a = sres[c * S + s];
        v[c] = fma(a.x, dv.x, fma(-a.y, dv.y, v[c]));
      }
    }
#pragma unroll
    for (int c = 0; c < kCB; ++c) acc[c] = fma(m * v[c], v[c], acc[c]);
  }
  __shared__ double red[kCB][8];
#pragma unroll
  for (int c = 0; c < kCB; ++c) {
    double t = acc[c];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) red[c][threadIdx.x >> 5] = t;
  }
  __syncthreads();
  if (threadIdx.x < kCB && k0 + (int)threadIdx.x < K) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[threadIdx.x][q];
    part[(long long)(k0 + threadIdx.x) * gridDim.x + blockIdx.x] = t;
  }
}

// Per-shift refinement targets (reading R13): the change of x_s between a
// snapshot taken when shift s first reached 10x its tolerance and the end of
// the first solve, d_s = x_s - snap_s (complex layout), and its M-weighted
// moments sum m (Re d)^2, sum m (Im d)^2, sum m Re d Im d -> part[(s*3+t)*gridDim.x + x].
// mode[s]: 0 no snapshot (d_s = 0), 1 complex snapshot, 2 real-layout snapshot,
// 3 / 4 snapshot of a pair's packed block: this shift is component x / y (R16).
struct SnapArgs {
  Grid g;
  const double* mass;
  const double2* x;       // shift block, complex layout (after the solve's epilogue)
  const double2* snap;    // shift block, per-shift layout of the solve (mode)
  double2* d;             // shift block out
  double* part;
  int mode[32];
};

__global__ void __launch_bounds__(256) k_snap_delta(const __grid_constant__ SnapArgs A) {
  const Grid& g = A.g;
  const int s = blockIdx.y, mode = A.mode[s];
  const long long n3 = 3 * g.Nn;
  const double2* x = A.x + (long long)s * n3;
  double2* d = A.d + (long long)s * n3;
  const double2* sc = A.snap + (long long)s * n3;
  const double* sr = reinterpret_cast<const double*>(sc);
  const int nx1 = g.n[0] + 1;
  double a0 = 0, a1 = 0, a2 = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n3; e += (long long)gridDim.x * blockDim.x) {
    double2 v = czero();
    if (mode) {
      const double2 xv = x[e];
      double2 sv;
      if (mode == 1) {
        sv = sc[e];
      } else if (mode >= 3) {
        sv = make_double2(mode == 3 ? sc[e].x : sc[e].y, 0.0);
      } else {
        const long long c = e / g.Nn, node = e - c * g.Nn;
        sv = make_double2(sr[c * g.NnP + (node / nx1) * g.px + node % nx1 + 1], 0.0);
      }
      v = csub(xv, sv);
      const double m = __ldg(A.mass + e);
      a0 = fma(m * v.x, v.x, a0);
      a1 = fma(m * v.y, v.y, a1);
      a2 = fma(m * v.x, v.y, a2);
    }
    d[e] = v;
  }
  __shared__ double red[3][8];
  double v3[3] = {a0, a1, a2};
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    for (int o = 16; o > 0; o >>= 1) v3[t] += __shfl_down_sync(0xffffffffu, v3[t], o);
    if ((threadIdx.x & 31) == 0) red[t][threadIdx.x >> 5] = v3[t];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[threadIdx.x][w];
    A.part[((long long)s * 3 + threadIdx.x) * gridDim.x + blockIdx.x] = t;
  }
}

// out[row] = sum_b part[row * ncol + b], one warp per row, fixed order.
__global__ void k_rows_sum(const double* __restrict__ part, int nrow, int ncol, double* out) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= nrow) return;
  double acc = 0.0;
  for (int b = lane; b < ncol; b += 32) acc += part[(long long)row * ncol + b];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0) out[row] = acc;
}

}  // namespace tem
