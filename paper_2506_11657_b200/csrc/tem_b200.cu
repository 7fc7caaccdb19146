// tem_b200.cu -- B200 (sm_100a) kernels and C ABI of the TEM forward hot path.
//
//   tem_edge_mass       lumped conductivity mass per edge          (§2.2, R1)
//   tem_apply_shifted   y_s = (K + s M) x_s for all shifts, one pass (north star (2))
//   tem_cocg_solve      batched multi-shift Jacobi-COCG               (north star (3))
//   tem_synthesize      u(t_k) = sum_s w_s Re(alpha_ks x_s)          (§3.2 eq:rmj, north star (4))
//   tem_forward_host    all of the above from host buffers
//
// Data layout: see include/tem_b200.h.  Shift blocks are shift-major
// ([S][3][Nn] complex): the CTA sweeping one shift streams one contiguous
// vector, and the S CTAs of one tile run together so every per-edge
// coefficient (mass) fetched from HBM serves every pole through L2.
//
// COCG iteration (both schemes in tem_sweep.cuh):
//   split (default): k_sweep<3|4>  p = z + beta p_old, q = A p on the fly,
//                                  z' = z - alpha D^-1 q, (odd) x; gamma, eps,
//                                  mu, ||r||^2 partials
//                    k_delta       delta = z'^T A z' by faces -> alpha, beta
//   two-sweep:       k_sweep<1>    p = z + beta p_old, mu = p^T A p -> alpha
//                    k_sweep<2>    q = A p again, x, z update -> rho, beta
// q is recomputed rather than stored (re-reading p through the TMA ring is
// cheaper than a 16 B/unknown/shift write + read).  Each reduction ends in
// the last CTA to finish (atomic ticket), which updates the per-shift scalars
// in device memory; no host round trip per iteration.  The iteration loop is
// a CUDA graph of `kChunk` iterations; the host checks the active-shift count
// once per chunk.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <string>
#include <vector>

#include "../../include/tem_b200.h"
#include "tem_device.cuh"
#include "tem_sweep.cuh"
#include "tem_persist.cuh"
#include "tem_refine.cuh"

using tem::Grid;
using tem::k_channel_mnorm;
using tem::k_rows_sum;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define TEM_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(TEM_ECUDA, std::string(#call " failed: ") + cudaGetErrorString(e_));     \
  } while (0)

constexpr int kChunk = 16;          // iterations per captured graph

// ------------------------------------------------------------------ kernels

__global__ void k_edge_mass(Grid g, const double* __restrict__ sigma, double* __restrict__ mass) {
  // M_e = (sum_{cells c touching e} sigma_c V_c / 4) / l_e^2 on free edges, 0 elsewhere.
  const long long total = 3 * g.Nn;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(idx / g.Nn);
    const long long n = idx - a * g.Nn;
    int pos[3];
    tem::node_pos(g, n, pos);
    const int b = (a + 1) % 3, d = (a + 2) % 3;
    double m = 0.0;
    const bool free_edge = pos[a] < g.n[a] && pos[b] >= 1 && pos[b] <= g.n[b] - 1 &&
                           pos[d] >= 1 && pos[d] <= g.n[d] - 1;
    if (free_edge) {
      const double ia = __ldg(g.ih[a] + pos[a]);
      for (int ob = -1; ob <= 0; ++ob)
        for (int od = -1; od <= 0; ++od) {
          int c[3];
          c[a] = pos[a];
          c[b] = pos[b] + ob;
          c[d] = pos[d] + od;
          const double vol = 1.0 / (__ldg(g.ih[0] + c[0]) * __ldg(g.ih[1] + c[1]) * __ldg(g.ih[2] + c[2]));
          m += __ldg(sigma + ((long long)c[2] * g.n[1] + c[1]) * g.n[0] + c[0]) * vol * 0.25;
        }
      m *= ia * ia;
    }
    mass[idx] = m;
  }
}

__device__ __forceinline__ double kdiag(const Grid& g, int a, const int pos[3]) {
  if (a == 0) return tem::edge_weights<0>(g, pos).diag();
  if (a == 1) return tem::edge_weights<1>(g, pos).diag();
  return tem::edge_weights<2>(g, pos).diag();
}

// COCG init (z-form): x = 0, p0 = p1 = 0, z = D^-1 b; rho = b^T z, ||b||^2,
// and (split scheme) the mass part s z^T M z of delta_0, with b = f (one real
// right-hand side for every shift) or b = rhs[s] (a shift block).  Block q
// serves shift q % S; a real shift (ShiftState::real) is laid out as a real
// vector (tem::vbase).  Its third partial sum uses A.part[9] / A.part[10] as
// scratch.
template <typename V>
__device__ __forceinline__ void init_body(const tem::SweepArgs& A, int s, int b, int nb, double2* p0,
                                          double2* p1, double2* z1, const double* __restrict__ f, double2& rho2,
                                          double& rr, double2& zmz2) {
  const Grid& g = A.g;
  const double2 sh2 = A.st[s].s;
  const long long cst = tem::vcomp<V>(g);
  const int rowp = tem::vrow<V>(g), nx1 = g.n[0] + 1;
  V* xv = tem::vbase<V>(A.x, s, g);
  V* zv = tem::vbase<V>(A.z, s, g);
  V* p0v = tem::vbase<V>(p0, s, g);
  V* p1v = tem::vbase<V>(p1, s, g);
  V* z1v = z1 ? tem::vbase<V>(z1, s, g) : nullptr;
  const double2* rhs = A.rhs ? A.rhs + (long long)s * 3 * g.Nn : nullptr;
  V rho = tem::VT<V>::zero(), zmz = tem::VT<V>::zero();
  for (long long slot = b * 256LL + threadIdx.x; slot < 3 * cst; slot += (long long)nb * 256) {
    const int a = (int)(slot / cst);
    const long long nv = slot - a * cst;                 // node in this layout
    const long long row = nv / rowp;
    const int i = (int)(nv - row * rowp) - tem::vofs<V>();
    V zv_ = tem::VT<V>::zero();
    if (i >= 0 && i < nx1) {
      const long long abi = a * g.Nn + row * nx1 + i;    // slot in the ABI layout
      const double m = __ldg(A.mass + abi);
      if (m > 0.0) {
        int pos[3];
        tem::node_pos(g, abi - a * g.Nn, pos);
        const V D = tem::VT<V>::make(kdiag(g, a, pos) + m * sh2.x, m * sh2.y);
        const V fv = rhs ? tem::VT<V>::from(__ldg(rhs + abi)) : tem::VT<V>::make(__ldg(f + abi), 0.0);
        zv_ = tem::cdiv(fv, D);
        rho = tem::cfma(fv, zv_, rho);
        rr += tem::cabs2(fv);
        zmz = tem::sfma(m, tem::csq(zv_), zmz);
      }
    }
    xv[slot] = tem::VT<V>::zero();
    zv[slot] = zv_;
    p0v[slot] = tem::VT<V>::zero();
    p1v[slot] = tem::VT<V>::zero();
    if (z1v) z1v[slot] = tem::VT<V>::zero();
  }
  rho2 = tem::VT<V>::cplx(rho);
  zmz2 = tem::VT<V>::cplx(zmz);
}

// The same for a pair of real shifts (leader s, partner sp): the packed
// vectors (component x: s, component y: sp) go to the leader's block in the
// complex layout; rr2 is ||b||^2 of the partner.
__device__ __forceinline__ void init_pair(const tem::SweepArgs& A, int s, int sp, int b, int nb, double2* p0,
                                          double2* p1, double2* z1, const double* __restrict__ f, double2& rho2,
                                          double& rr, double& rr2, double2& zmz2) {
  const Grid& g = A.g;
  const double sa = A.st[s].s.x, sb = A.st[sp].s.x;
  const long long off = (long long)s * 3 * g.Nn;
  const double2* ra = A.rhs ? A.rhs + off : nullptr;
  const double2* rb = A.rhs ? A.rhs + (long long)sp * 3 * g.Nn : nullptr;
  double2 rho = tem::czero(), zmz = tem::czero();
  for (long long slot = b * 256LL + threadIdx.x; slot < 3 * g.Nn; slot += (long long)nb * 256) {
    double2 z = tem::czero();
    const double m = __ldg(A.mass + slot);
    if (m > 0.0) {
      const int a = (int)(slot / g.Nn);
      int pos[3];
      tem::node_pos(g, slot - a * g.Nn, pos);
      const double kd = kdiag(g, a, pos);
      const double fa = ra ? __ldg(&ra[slot].x) : __ldg(f + slot);
      const double fb = rb ? __ldg(&rb[slot].x) : __ldg(f + slot);
      z = make_double2(fa / fma(m, sa, kd), fb / fma(m, sb, kd));
      rho.x = fma(fa, z.x, rho.x);
      rho.y = fma(fb, z.y, rho.y);
      rr = fma(fa, fa, rr);
      rr2 = fma(fb, fb, rr2);
      zmz.x = fma(m, z.x * z.x, zmz.x);
      zmz.y = fma(m, z.y * z.y, zmz.y);
    }
    A.x[off + slot] = tem::czero();
    A.z[off + slot] = z;
    p0[off + slot] = tem::czero();
    p1[off + slot] = tem::czero();
    if (z1) z1[off + slot] = tem::czero();
  }
  rho2 = rho;
  zmz2 = zmz;
}

__global__ void __launch_bounds__(256) k_init(tem::SweepArgs A, double2* p0, double2* p1, double2* z1,
                                              const double* __restrict__ f) {
  __shared__ double red[3 * 8];
  const int S = A.S;
  const int s = blockIdx.x % S;
  const int nb = gridDim.x / S;
  const int b = blockIdx.x / S;
  double2 rho = tem::czero(), zmz = tem::czero();
  double rr = 0.0, rr2 = 0.0;
  const int partner = A.st[s].pair - 1;
  if (partner >= 0) {   // the leader's blocks initialise the pair; the partner's blocks have nothing to do
    if (A.st[s].lead) init_pair(A, s, partner, b, nb, p0, p1, z1, f, rho, rr, rr2, zmz);
  } else if (A.st[s].real) {
    init_body<double>(A, s, b, nb, p0, p1, z1, f, rho, rr, zmz);
  } else {
    init_body<double2>(A, s, b, nb, p0, p1, z1, f, rho, rr, zmz);
  }
  tem::block_sum_n<256>(rho, rr, red);
  tem::block_sum_n<256>(zmz, rr2, red);
  if (threadIdx.x == 0) {
    A.part_c[blockIdx.x] = rho;
    A.part_r[blockIdx.x] = rr;
    A.part[9 * A.pstride + blockIdx.x] = zmz.x;
    A.part[10 * A.pstride + blockIdx.x] = zmz.y;
    A.part[11 * A.pstride + blockIdx.x] = rr2;
  }
  if (!tem::last_block(&A.ctl->ticket[0])) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = warp; q < S; q += 8) {
    // the sums of a pair live in its leader's blocks: (x, rr) the leader's, (y, rr2) the partner's
    const int qp = A.st[q].pair - 1;
    const bool second = qp >= 0 && !A.st[q].lead;
    const int src = second ? qp : q;
    double cx = 0, cy = 0, cr = 0, mx = 0, my = 0, cr2 = 0;
    for (int bb = src + lane * S; bb < (int)gridDim.x; bb += 32 * S) {
      const double2 v = __ldcg(A.part_c + bb);
      cx += v.x;
      cy += v.y;
      cr += __ldcg(A.part_r + bb);
      mx += __ldcg(A.part + 9 * A.pstride + bb);
      my += __ldcg(A.part + 10 * A.pstride + bb);
      cr2 += __ldcg(A.part + 11 * A.pstride + bb);
    }
    cx = tem::warp_sum(cx);
    cy = tem::warp_sum(cy);
    cr = tem::warp_sum(cr);
    mx = tem::warp_sum(mx);
    my = tem::warp_sum(my);
    cr2 = tem::warp_sum(cr2);
    if (qp >= 0) {   // real sums of this member
      cx = second ? cy : cx;
      mx = second ? my : mx;
      cr = second ? cr2 : cr;
      cy = 0.0;
      my = 0.0;
    }
    if (lane == 0) {
      tem::ShiftState& st = A.st[q];
      st.rho = make_double2(cx, cy);
      st.dm0 = tem::cmul(st.s, make_double2(mx, my));   // s z_0^T M z_0
      st.fnorm = sqrt(cr);
      st.relres = cr > 0 ? 1.0 : 0.0;
      st.alpha = tem::czero();
      st.beta = tem::czero();
      st.iters = 0;
      st.active = cr > 0 ? 1 : 0;
      st.status = cr > 0 ? 0 : 1;
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    __threadfence();
    tem::rebuild_list(A);
    if (threadIdx.x == 0) A.ctl->ticket[0] = 0;
  }
}

// Pairing (R16): real shifts with real right-hand sides (ShiftState::real,
// final after k_real_mask) are sorted by shift -- iteration counts grow as s
// falls, so neighbours stop at about the same time -- and paired two by two;
// an odd one out stays a single real shift.  One thread; S <= 32.
__global__ void k_pair(tem::ShiftState* st, int S, int enable) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int idx[TEM_MAX_SHIFTS], n = 0;
  for (int s = 0; s < S; ++s) {
    st[s].pair = 0;
    st[s].lead = 0;
    if (enable && st[s].real) idx[n++] = s;
  }
  for (int i = 1; i < n; ++i)   // insertion sort, descending shift
    for (int j = i; j > 0 && st[idx[j]].s.x > st[idx[j - 1]].s.x; --j) {
      const int t = idx[j];
      idx[j] = idx[j - 1];
      idx[j - 1] = t;
    }
  for (int i = 0; i + 1 < n; i += 2) {
    st[idx[i]].pair = idx[i + 1] + 1;
    st[idx[i]].lead = 1;
    st[idx[i + 1]].pair = idx[i] + 1;
    st[idx[i + 1]].lead = 0;
  }
}

// A real shift may run in real arithmetic only if its right-hand side is
// real: flag[s] = 1 if rhs[s] has a nonzero imaginary part (rhs-block solves).
__global__ void k_rhs_imag(const double2* __restrict__ rhs, long long nslots, int* flag) {
  const int s = blockIdx.y;
  const double2* r = rhs + (long long)s * nslots;
  bool any = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nslots; i += (long long)gridDim.x * blockDim.x)
    any |= __ldg(&r[i].y) != 0.0;
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr(flag + s, 1);
}

// Split solver epilogue: a shift whose last iteration i was even (iters odd)
// has x_i in x (x advances every second iteration); x_{i+1} = x_i + alpha_i p_i
// with p_i in p1.  alpha_i is `alpha` if the shift stopped, `alpha_prev` if it
// is still running (maxit reached).  Block q serves shift q % S.
template <typename V>
__device__ __forceinline__ void xfix_body(const tem::SweepArgs& A, const double2* p1, int s, int b, int nb,
                                          double2 a2) {
  const long long n = 3 * tem::vcomp<V>(A.g);
  V* x = tem::vbase<V>(A.x, s, A.g);
  const V* p = tem::vbase<V>(p1, s, A.g);
  const V a = tem::VT<V>::from(a2);
  for (long long slot = b * 256LL + threadIdx.x; slot < n; slot += (long long)nb * 256)
    x[slot] = tem::cfma(a, p[slot], x[slot]);
}

__global__ void __launch_bounds__(256) k_xfix(tem::SweepArgs A, const double2* __restrict__ p1) {
  const int S = A.S;
  const int s = blockIdx.x % S;
  const tem::ShiftState& st = A.st[s];
  if (st.pair) {
    // a pair ran max(iters) iterations; if the last one was even, each member's
    // pending step length is its alpha_prev (0 if it was frozen earlier, R16)
    if (!st.lead) return;
    const tem::ShiftState& sp = A.st[st.pair - 1];
    if ((max(st.iters, sp.iters) & 1) == 0) return;
    const double ax = st.alpha_prev.x, ay = sp.alpha_prev.x;
    double2* x = A.x + (long long)s * 3 * A.g.Nn;
    const double2* p = p1 + (long long)s * 3 * A.g.Nn;
    const int b = blockIdx.x / S, nb = gridDim.x / S;
    for (long long slot = b * 256LL + threadIdx.x; slot < 3 * A.g.Nn; slot += (long long)nb * 256) {
      const double2 pv = p[slot], xv = x[slot];
      x[slot] = make_double2(fma(ax, pv.x, xv.x), fma(ay, pv.y, xv.y));
    }
    return;
  }
  if ((st.iters & 1) == 0) return;
  const double2 a = st.active ? st.alpha_prev : st.alpha;
  if (st.real)
    xfix_body<double>(A, p1, s, blockIdx.x / S, gridDim.x / S, a);
  else
    xfix_body<double2>(A, p1, s, blockIdx.x / S, gridDim.x / S, a);
}

// Real shifts: x (real layout, in x's own region) -> complex ABI layout.
// Pass 0 copies the real vector to tmp (the same shift's region of a free
// work vector); pass 1 expands tmp into x (imaginary parts 0, non-free and
// non-existent slots 0).
// A pair's packed x (leader's block) -> the two members' blocks in the ABI
// layout (real parts, imaginary parts 0); element-wise, in place.
__global__ void __launch_bounds__(256) k_pair_out(tem::SweepArgs A) {
  const int S = A.S;
  const int s = blockIdx.x % S;
  if (!A.st[s].pair || !A.st[s].lead) return;
  const int b = blockIdx.x / S, nb = gridDim.x / S;
  double2* xa = A.x + (long long)s * 3 * A.g.Nn;
  double2* xb = A.x + (long long)(A.st[s].pair - 1) * 3 * A.g.Nn;
  for (long long slot = b * 256LL + threadIdx.x; slot < 3 * A.g.Nn; slot += (long long)nb * 256) {
    const double2 v = xa[slot];
    xa[slot] = make_double2(v.x, 0.0);
    xb[slot] = make_double2(v.y, 0.0);
  }
}

__global__ void __launch_bounds__(256) k_real_out(tem::SweepArgs A, double2* tmp, int pass) {
  const int S = A.S;
  const int s = blockIdx.x % S;
  if (!A.st[s].real || A.st[s].pair) return;
  const int b = blockIdx.x / S, nb = gridDim.x / S;
  const Grid& g = A.g;
  const double* xr = tem::vbase<double>(A.x, s, g);
  double* tr = tem::vbase<double>(tmp, s, g);
  if (pass == 0) {
    for (long long i = b * 256LL + threadIdx.x; i < 3 * g.NnP; i += (long long)nb * 256) tr[i] = xr[i];
    return;
  }
  double2* xc = A.x + (long long)s * 3 * g.Nn;
  const int nx1 = g.n[0] + 1;
  for (long long slot = b * 256LL + threadIdx.x; slot < 3 * g.Nn; slot += (long long)nb * 256) {
    const int a = (int)(slot / g.Nn);
    const long long node = slot - a * g.Nn;
    const long long row = node / nx1;
    xc[slot] = make_double2(tr[a * g.NnP + row * g.px + (node - row * nx1) + 1], 0.0);
  }
}

// u[k][slot] = sum_s w_s Re(res[k][s] x[s][slot]); 0 on non-free slots.
__device__ __forceinline__ bool free_slot(const Grid& g, long long slot) {
  const int a = (int)(slot / g.Nn);
  int pos[3];
  tem::node_pos(g, slot - a * g.Nn, pos);
  const int b = (a + 1) % 3, d = (a + 2) % 3;
  return pos[a] < g.n[a] && pos[b] >= 1 && pos[b] <= g.n[b] - 1 && pos[d] >= 1 &&
         pos[d] <= g.n[d] - 1;
}

template <int SMAX>
__global__ void k_synth(Grid g, int S, int K, const double2* __restrict__ res,
                        const double* __restrict__ wts, const double2* __restrict__ x,
                        double* __restrict__ u) {
  extern __shared__ unsigned char smem_raw[];
  double2* sres = reinterpret_cast<double2*>(smem_raw);  // [K][S], pre-multiplied by w_s
  for (int i = threadIdx.x; i < K * S; i += blockDim.x) {
    const double w = wts[i % S];
    const double2 a = res[i];
    sres[i] = make_double2(w * a.x, w * a.y);
  }
  __syncthreads();
  const long long nslots = 3 * g.Nn;
  for (long long slot = blockIdx.x * (long long)blockDim.x + threadIdx.x; slot < nslots;
       slot += (long long)gridDim.x * blockDim.x) {
    const bool live = free_slot(g, slot);
    double2 xv[SMAX];
#pragma unroll
    for (int s = 0; s < SMAX; ++s)
      xv[s] = (live && s < S) ? __ldg(x + (long long)s * nslots + slot) : tem::czero();
    for (int k = 0; k < K; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int s = 0; s < SMAX; ++s) {
        if (s < S) {
          const double2 a = sres[k * S + s];
          acc = fma(a.x, xv[s].x, fma(-a.y, xv[s].y, acc));
        }
      }
      u[(long long)k * nslots + slot] = acc;
    }
  }
}

// -d_t b_z at receivers (reading R12): the circulation of
// the channel field u(t_k) around the z-normal face with lower-corner node
// (i, j, k), divided by the face area.  One thread per (channel, receiver).
__global__ void k_curl_z(Grid g, int K, int R, const int* __restrict__ rec, const double* __restrict__ u,
                         double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * R) return;
  const int kc = t / R, r = t - kc * R;
  const int i = rec[3 * r], j = rec[3 * r + 1], k = rec[3 * r + 2];
  const long long nx1 = g.n[0] + 1, ny1 = g.n[1] + 1;
  const long long node = ((long long)k * ny1 + j) * nx1 + i;
  const double* uk = u + (long long)kc * 3 * g.Nn;
  // +x(i,j,k) + y(i+1,j,k) - x(i,j+1,k) - y(i,j,k)
  const double circ = uk[node] + uk[g.Nn + node + 1] - uk[node + nx1] - uk[g.Nn + node];
  out[t] = circ * __ldg(g.ih[0] + i) * __ldg(g.ih[1] + j);
}

}  // namespace

void tem_set_error(const std::string& msg) { g_last_error = msg; }

// ====================================================================== C ABI

struct tem_ctx {
  Grid g{};
  int device = 0;
  int num_sms = 0;
  double* dev_h = nullptr;          // ih[3] and hdm[3] packed
  cudaStream_t cap_stream = nullptr;
  int* pinned_active = nullptr;
  // cached graphs of kChunk COCG iterations: per set of buffers (+ scheme, S),
  // per (slots, z-chunks); a few buffer sets (a forward alternates the
  // initial solve and the correction solves of the refinement)
  std::map<std::vector<const void*>, std::map<long long, cudaGraphExec_t>> graphs;
  // scratch
  void* scratch = nullptr;          // residues etc.
  size_t scratch_bytes = 0;
  // e2e workspace
  void* e2e = nullptr;
  size_t e2e_bytes = 0;
  // stats of the last solve
  tem_solve_stats stats{};
  int per_sm_two = 2;               // resident CTAs per SM of k_sweep<1> (two-sweep geometry)
  int per_sm_split = 1;             // resident CTAs per SM of k_sweep<3> (split geometry)
  int per_sm_persist = 0;           // resident CTAs per SM of k_persist (0: cannot co-reside)
  int launch_mode = TEM_LAUNCH_AUTO;
  int solver = TEM_SOLVER_SPLIT;
  int band = 4;                     // tile rows per band of the block order (block_coords), 32x8 tiles
  int band_split = 96 / tem::kTYSplit;   // the same for the split scheme's 32x12 tiles: 8 (measured best)
  int real_arith = 1;               // real shifts in real arithmetic (split scheme; TEM_NO_REAL=1 disables)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;   // loop timing of the last solve
  int last_persistent = 0;          // the last solve ran k_persist
  double last_fnorm = 0.0;          // ||rhs||_2 of shift 0 of the last solve
  tem_forward_stats fstats{};       // of the last tem_forward / tem_forward_host
  void* pin = nullptr;              // pinned staging of small host arrays
  size_t pin_bytes = 0;
  cudaEvent_t stage_ev = nullptr;   // last copy out of `pin`
  void* red = nullptr;              // reduction scratch of tem_residual
  size_t red_bytes = 0;
};

static int check_S(int S) {
  if (S < 1 || S > TEM_MAX_SHIFTS)
    return fail(TEM_EINVAL, "S must be in [1, " + std::to_string(TEM_MAX_SHIFTS) + "]");
  return TEM_OK;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Every launching call runs on the device the context was created on; a
// different current device is an argument error (the caller's streams and
// buffers would belong to another device).
static int check_device(const tem_ctx* c) {
  int dev = -1;
  TEM_CUDA(cudaGetDevice(&dev));
  if (dev != c->device)
    return fail(TEM_EINVAL, "current device " + std::to_string(dev) + " is not the context's device " +
                                std::to_string(c->device));
  return TEM_OK;
}

// The sweeps index a shift block with unsigned 32-bit element indices (the
// shift's offset included; real shifts count 8-byte elements): S * 6 Nn must
// stay below 2^32.  HBM is the tighter limit (S = 14: 51 M nodes here, 53 M
// nodes of COCG state in 180 GB).
static int check_index(const tem_ctx* c, int S) {
  if ((unsigned long long)S * 6ULL * (unsigned long long)c->g.Nn >= (1ULL << 32))
    return fail(TEM_EINVAL, "S * 6 * nodes must be below 2^32 (32-bit element indices of the sweeps)");
  return TEM_OK;
}

// sweep geometry of one scheme: xy tiles x z-chunks x shift slots, for tile
// height ty (tem::kTYTwoSweep or tem::kTYSplit).  The z-range is split until
// the grid covers ~4 waves of resident CTAs, so that a few remaining
// (slow-converging) shifts still fill the machine.
static void sweep_geometry(const tem_ctx* c, int S, int nslot, tem::SweepArgs& A, int* grid,
                           int ty = tem::kTYTwoSweep, int per_sm_override = 0) {
  A.g = c->g;
  A.S = S;
  A.nslot = nslot;
  A.band = ty == tem::kTYSplit ? c->band_split : c->band;
  A.ntx = (c->g.n[0] + 32 - 1) / 32;
  A.nty = (c->g.n[1] + ty - 1) / ty;
  const int per_sm = per_sm_override > 0 ? per_sm_override
                   : ty == tem::kTYSplit ? c->per_sm_split : c->per_sm_two;
  const int base = A.ntx * A.nty * nslot;
  // z-chunk count.  W = CTAs / resident CTAs.
  // Bandwidth regime (some candidate reaches >= 4 waves with >= 8 planes per
  // chunk): keep ~2 waves or more and among those maximise (wave quantisation
  // W / ceil(W): a partial last wave idles SMs) x (march efficiency
  // kch / (kch + 3): a CTA fills its plane pipeline, ~3 steps, before it
  // computes).  Large config, 12 slots: 1152 columns = 7.8 waves of 148 -> 2
  // chunks of 64 planes, 15.6 waves; one slot left: 3 chunks of 43 planes,
  // 1.95 waves (measured 0.294 ms per iteration against 0.362 ms with the 9
  // chunks a 4-wave floor asked for; CTA durations are uniform now that real
  // shifts run in pairs, R16; `scripts/nzc_tail.sh`).
  // Latency regime (small grids, few active shifts: the whole sweep is less
  // than 4 waves): minimise the critical path, ceil(W) waves of (kch + 3)
  // plane steps each, down to one plane per chunk -- e.g. `block` with one
  // shift left: 32 chunks of 1 plane (4 steps) instead of 4 of 8 (11 steps).
  const int nz = c->g.n[2];
  const int nzc_min = (nz + tem::kMaxChunk - 1) / tem::kMaxChunk;
  int nzc = nzc_min;
  const double slots_sm = (double)c->num_sms * per_sm;
  bool bandwidth = false;
  for (int cand = nzc_min; cand <= 32 && (cand == nzc_min || nz / cand >= 8); ++cand) {
    const int kch = (nz + cand - 1) / cand;
    const int nz_eff = (nz + kch - 1) / kch;
    bandwidth |= (double)base * nz_eff / slots_sm >= 4.0;
  }
  double min_waves = 1.9;
  if (const char* env = getenv("TEM_MIN_WAVES")) min_waves = atof(env);   // experiments
  double best = bandwidth ? -1.0 : 1e300;
  for (int cand = nzc_min; cand <= (bandwidth ? 32 : std::min(nz, 64)); ++cand) {
    const int kch = (nz + cand - 1) / cand;
    const int nz_eff = (nz + kch - 1) / kch;
    if (nz_eff != cand) continue;   // the same chunking as a smaller count
    const double W = (double)base * nz_eff / slots_sm;
    if (bandwidth) {
      if (cand != nzc_min && nz / cand < 8) break;
      if (W < min_waves) continue;
      const double score = W / std::ceil(W) * (double)kch / (kch + 3.0);
      if (score > best + 1e-9) {
        best = score;
        nzc = cand;
      }
    } else {
      const double cost = std::ceil(W - 1e-9) * (kch + 3.0);
      if (cost < best - 1e-9) {
        best = cost;
        nzc = cand;
      }
    }
  }
  if (const char* env = getenv("TEM_FORCE_NZC")) nzc = std::max(nzc_min, atoi(env));  // tests
  A.kchunk = (c->g.n[2] + nzc - 1) / nzc;
  A.nzc = (c->g.n[2] + A.kchunk - 1) / A.kchunk;
  *grid = A.ntx * A.nty * A.nzc * nslot;
}

static int max_sweep_grid(const tem_ctx* c, int S) {
  int gmax = 0;
  for (int ty : {tem::kTYTwoSweep, tem::kTYSplit})
    for (int ns = 1; ns <= S; ++ns) {
      tem::SweepArgs A{};
      int gr = 0;
      sweep_geometry(c, S, ns, A, &gr, ty);
      gmax = std::max(gmax, gr);
    }
  return gmax;
}

// Dynamic shared-memory limits of the sweep kernels.  Function attributes
// belong to the CUDA context of the current device, so they are set on every
// tem_create (cheap) rather than once per process.
static int sweep_attrs() {
  using T2 = tem::Tile<tem::kTYTwoSweep>;
  using TS = tem::Tile<tem::kTYSplit>;
  const int attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
  TEM_CUDA(cudaFuncSetAttribute(tem::k_sweep<0>, (cudaFuncAttribute)attr, (int)T2::kSmemDirect));
  TEM_CUDA(cudaFuncSetAttribute(tem::k_sweep<2>, (cudaFuncAttribute)attr, (int)T2::kSmemDirect));
  TEM_CUDA(cudaFuncSetAttribute(tem::k_sweep<1>, (cudaFuncAttribute)attr, (int)T2::kSmemDirap));
  TEM_CUDA(cudaFuncSetAttribute(tem::k_sweep<3>, (cudaFuncAttribute)attr, (int)TS::kSmemUpd));
  TEM_CUDA(cudaFuncSetAttribute(tem::k_sweep<4>, (cudaFuncAttribute)attr, (int)TS::kSmemDirap));
  TEM_CUDA(cudaFuncSetAttribute(tem::k_delta<false>, (cudaFuncAttribute)attr, (int)TS::kSmemDelta));
  TEM_CUDA(cudaFuncSetAttribute(tem::k_delta<true>, (cudaFuncAttribute)attr, (int)TS::kSmemDelta));
  TEM_CUDA(cudaFuncSetAttribute(tem::k_persist<>, (cudaFuncAttribute)attr, (int)TS::kSmemUpd));
  return TEM_OK;
}

// 5-D tiled tensor map over a shift block [S][3][nz+1][ny+1][nx+1] complex
// fp64 (as 2(nx+1) doubles innermost); box = one halo-extended plane tile.
// real = true: the same buffer in the real layout of real shifts (fp64
// [3][nz+1][ny+1][px] at the start of each shift's complex region;
// tem::Grid::px), box 34 x (ty+2) doubles.
static int make_tmap(const tem_ctx* c, int S, const void* base, CUtensorMap* tm, int ty = tem::kTYTwoSweep,
                     bool real = false) {
  const int box_x = 32 + 2, box_y = ty + 2;   // halo-extended plane tile (Tile<ty>::HX, HY)
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    TEM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      return fail(TEM_ECUDA, "cuTensorMapEncodeTiled not available");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t nx1 = c->g.n[0] + 1, ny1 = c->g.n[1] + 1, nz1 = c->g.n[2] + 1;
  const cuuint64_t px = c->g.px, shift_stride = 48 * nx1 * ny1 * nz1;
  const cuuint64_t dims_c[5] = {2 * nx1, ny1, nz1, 3, (cuuint64_t)S};
  const cuuint64_t str_c[4] = {16 * nx1, 16 * nx1 * ny1, 16 * nx1 * ny1 * nz1, shift_stride};
  const cuuint64_t dims_r[5] = {nx1 + 1, ny1, nz1, 3, (cuuint64_t)S};   // leading zero column + nodes
  const cuuint64_t str_r[4] = {8 * px, 8 * px * ny1, 8 * px * ny1 * nz1, shift_stride};
  const cuuint32_t box[5] = {(real ? 1u : 2u) * (cuuint32_t)box_x, (cuuint32_t)box_y, 1, 1, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  if (const char* env = getenv("TEM_L2PROMO")) {  // experiments
    const int v = atoi(env);
    promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
          : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
          : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
  CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void*>(base), real ? dims_r : dims_c,
                      real ? str_r : str_c, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TEM_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return TEM_OK;
}

extern "C" {

const char* tem_version(void) { return "tem_b200 0.2 sm_100a"; }
const char* tem_last_error(void) { return g_last_error.c_str(); }

int tem_create(int nx, int ny, int nz, const double* hx, const double* hy, const double* hz,
               tem_ctx** out) {
  if (!out || !hx || !hy || !hz) return fail(TEM_EINVAL, "tem_create: null pointer");
  *out = nullptr;
  if (nx < 2 || ny < 2 || nz < 2) return fail(TEM_EINVAL, "tem_create: need nx, ny, nz >= 2");
  const long long Nn = (long long)(nx + 1) * (ny + 1) * (nz + 1);
  if (Nn * 3 * TEM_MAX_SHIFTS >= (1LL << 40))
    return fail(TEM_EINVAL, "tem_create: grid too large");
  const int n[3] = {nx, ny, nz};
  const double* h[3] = {hx, hy, hz};
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < n[a]; ++i)
      if (!(h[a][i] > 0.0)) return fail(TEM_EINVAL, "tem_create: cell widths must be > 0");
  tem_ctx* c = new tem_ctx();
  {
    cudaError_t e0 = cudaGetDevice(&c->device);
    if (e0 == cudaSuccess) e0 = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
    if (e0 != cudaSuccess) {
      delete c;
      return fail(TEM_ECUDA, std::string("tem_create: ") + cudaGetErrorString(e0));
    }
  }
  for (int a = 0; a < 3; ++a) c->g.n[a] = n[a];
  c->g.st[0] = 1;
  c->g.st[1] = nx + 1;
  c->g.st[2] = (long long)(nx + 1) * (ny + 1);
  c->g.Nn = Nn;
  c->g.px = (nx + 2 + 1) / 2 * 2;
  c->g.NnP = (long long)c->g.px * (ny + 1) * (nz + 1);
  // host tables: 1/h and hdual/mu0
  std::vector<double> tab;
  size_t off_ih[3], off_hd[3];
  for (int a = 0; a < 3; ++a) {
    off_ih[a] = tab.size();
    for (int i = 0; i < n[a]; ++i) tab.push_back(1.0 / h[a][i]);
  }
  for (int a = 0; a < 3; ++a) {
    off_hd[a] = tab.size();
    for (int i = 0; i <= n[a]; ++i) {
      double hd = (i == 0) ? 0.5 * h[a][0] : (i == n[a]) ? 0.5 * h[a][n[a] - 1]
                                                         : 0.5 * (h[a][i - 1] + h[a][i]);
      tab.push_back(hd / tem::kMu0);
    }
  }
  cudaError_t e = cudaMalloc(&c->dev_h, tab.size() * sizeof(double));
  if (e != cudaSuccess) {
    delete c;
    return fail(TEM_ENOMEM, std::string("tem_create: cudaMalloc: ") + cudaGetErrorString(e));
  }
  e = cudaMemcpy(c->dev_h, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMallocHost(&c->pinned_active, sizeof(int));
  if (e != cudaSuccess) {
    tem_destroy(c);
    return fail(TEM_ECUDA, std::string("tem_create: ") + cudaGetErrorString(e));
  }
  for (int a = 0; a < 3; ++a) {
    c->g.ih[a] = c->dev_h + off_ih[a];
    c->g.hdm[a] = c->dev_h + off_hd[a];
  }
  if (int rc = sweep_attrs()) {
    tem_destroy(c);
    return rc;
  }
  if (const char* env = getenv("TEM_BAND")) c->band = c->band_split = atoi(env);   // experiments
  if (const char* env = getenv("TEM_NO_REAL")) c->real_arith = atoi(env) ? 0 : 1;  // experiments, tests
  if (const char* env = getenv("TEM_LAUNCH")) c->launch_mode = atoi(env);            // experiments
  {
    int per_sm = 0;
    using T2 = tem::Tile<tem::kTYTwoSweep>;
    using TS = tem::Tile<tem::kTYSplit>;
    cudaError_t e1 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tem::k_sweep<1>, T2::NT, T2::kSmemDirap);
    c->per_sm_two = std::max(1, per_sm);
    if (e1 == cudaSuccess)
      e1 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tem::k_sweep<3>, TS::NT, TS::kSmemUpd);
    c->per_sm_split = std::max(1, per_sm);
    if (e1 == cudaSuccess)
      e1 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->per_sm_persist, tem::k_persist<>, TS::NT, TS::kSmemUpd);
    if (e1 == cudaSuccess) e1 = cudaEventCreate(&c->ev0);
    if (e1 == cudaSuccess) e1 = cudaEventCreate(&c->ev1);
    if (e1 == cudaSuccess) e1 = cudaEventCreateWithFlags(&c->stage_ev, cudaEventDisableTiming);
    if (e1 != cudaSuccess) {
      tem_destroy(c);
      return fail(TEM_ECUDA, std::string("tem_create: ") + cudaGetErrorString(e1));
    }
  }
  *out = c;
  return TEM_OK;
}

void tem_destroy(tem_ctx* c) {
  if (!c) return;
  for (auto& set : c->graphs)
    for (auto& kv : set.second) cudaGraphExecDestroy(kv.second);
  if (c->dev_h) cudaFree(c->dev_h);
  if (c->scratch) cudaFree(c->scratch);
  if (c->e2e) cudaFree(c->e2e);
  if (c->pinned_active) cudaFreeHost(c->pinned_active);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->stage_ev) cudaEventDestroy(c->stage_ev);
  if (c->red) cudaFree(c->red);
  if (c->pin) cudaFreeHost(c->pin);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  delete c;
}

size_t tem_num_nodes(const tem_ctx* c) { return c ? (size_t)c->g.Nn : 0; }

size_t tem_num_unknowns(const tem_ctx* c) {
  if (!c) return 0;
  const long long nx = c->g.n[0], ny = c->g.n[1], nz = c->g.n[2];
  return (size_t)(nx * (ny - 1) * (nz - 1) + (nx - 1) * ny * (nz - 1) + (nx - 1) * (ny - 1) * nz);
}

int tem_edge_mass(tem_ctx* c, const double* sigma, double* mass, void* stream) {
  if (!c || !sigma || !mass) return fail(TEM_EINVAL, "tem_edge_mass: null pointer");
  if (int rc = check_device(c)) return rc;
  const long long total = 3 * c->g.Nn;
  const int block = 256;
  const int grid = (int)std::min<long long>((total + block - 1) / block, (long long)c->num_sms * 32);
  k_edge_mass<<<grid, block, 0, (cudaStream_t)stream>>>(c->g, sigma, mass);
  TEM_CUDA(cudaGetLastError());
  return TEM_OK;
}

int tem_apply_shifted(tem_ctx* c, const double* mass, int S, const double* shifts,
                      const double* x, double* y, void* stream) {
  if (!c || !mass || !shifts || !x || !y) return fail(TEM_EINVAL, "tem_apply_shifted: null pointer");
  if (int rc = check_S(S)) return rc;
  if (int rc = check_device(c)) return rc;
  if (int rc = check_index(c, S)) return rc;
  tem::SweepArgs A{};
  int grid = 0;
  sweep_geometry(c, S, S, A, &grid);
  for (int s = 0; s < S; ++s) A.shifts[s] = make_double2(shifts[2 * s], shifts[2 * s + 1]);
  A.mass = mass;
  A.out = reinterpret_cast<double2*>(y);
  CUtensorMap tm;
  if (int rc = make_tmap(c, S, x, &tm)) return rc;
  TEM_CUDA(cudaMemsetAsync(y, 0, (size_t)3 * c->g.Nn * S * sizeof(double2), (cudaStream_t)stream));
  using T2 = tem::Tile<tem::kTYTwoSweep>;
  tem::k_sweep<0><<<grid, T2::NT, T2::kSmemDirect, (cudaStream_t)stream>>>(A, tm, tm, tm, tm);
  TEM_CUDA(cudaGetLastError());
  return TEM_OK;
}

struct WorkLayout {
  size_t z, z1, p0, p1, st, ctl, flags, gbar, part_c, part_r, part9, total;
  size_t nparts;
};

static WorkLayout work_layout(const tem_ctx* c, int S) {
  WorkLayout L{};
  const size_t vec = (size_t)3 * c->g.Nn * S * sizeof(double2);
  const size_t nparts = (size_t)std::max(max_sweep_grid(c, S), 1024 * S);

  size_t o = 0;
  L.z = o;      o = align_up(o + vec, 256);
  L.z1 = o;     o = align_up(o + vec, 256);
  L.p0 = o;     o = align_up(o + vec, 256);
  L.p1 = o;     o = align_up(o + vec, 256);
  L.st = o;     o = align_up(o + sizeof(tem::ShiftState) * TEM_MAX_SHIFTS, 256);
  L.ctl = o;    o = align_up(o + sizeof(tem::Control), 256);
  L.flags = o;  o = align_up(o + sizeof(int) * TEM_MAX_SHIFTS, 256);
  L.gbar = o;   o = align_up(o + 2 * sizeof(unsigned), 256);
  L.part_c = o; o = align_up(o + nparts * sizeof(double2), 256);
  L.part_r = o; o = align_up(o + nparts * sizeof(double), 256);
  L.part9 = o;  o = align_up(o + tem::kSplitPart * nparts * sizeof(double), 256);
  L.nparts = nparts;
  L.total = o;
  return L;
}

size_t tem_cocg_workspace_bytes(const tem_ctx* c, int S) {
  if (!c || S < 1 || S > TEM_MAX_SHIFTS) return 0;
  return work_layout(c, S).total;
}

// Host side of one batched COCG solve, both schemes (include/tem_b200.h
// TEM_SOLVER_*).  Per iteration i with parity q = i & 1:
//   two-sweep: k_sweep<1> (p_new = z + beta p_old in P[1-q], mu = p^T A p ->
//              alpha) then k_sweep<2> (x, z update; rho, ||r|| -> beta, stop);
//   split:     pass 1 k_sweep<3> (even i) / k_sweep<4> (odd i): p_i = z_i +
//              beta p_{i-1}, z_{i+1} = z_i - alpha_i D^-1 A p_i (Z[q] -> Z[1-q],
//              P[q] -> P[1-q]), odd i also x (R11); partials gamma, eps, mu,
//              ||r||^2; pass 2 k_delta: delta = z_{i+1}^T A z_{i+1}, the last CTA
//              forms alpha_{i+1}, beta_{i+1}, the stop test (finalize_split).
//              Start: k_delta<true> on z_0 (alpha_0 = gamma_0 / delta_0); end:
//              k_xfix for shifts whose x lags one iteration.
// Launch configurations depend on the active-slot count (and with it the
// z-chunking); each is captured once as a CUDA graph of kChunk iterations.
// The host reads the active count once per graph.
static int finish_solve(tem_ctx* c, int S, std::vector<tem::ShiftState>& st, const tem::ShiftState* dev_st,
                        cudaStream_t stream, long long launches, int grid, int block, int* iters, double* relres) {
  TEM_CUDA(cudaMemcpyAsync(st.data(), dev_st, sizeof(tem::ShiftState) * S, cudaMemcpyDeviceToHost, stream));
  TEM_CUDA(cudaStreamSynchronize(stream));
  float ms = 0.f;
  TEM_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));

  long long shift_iters = 0;
  int max_it = 0, n_real = 0;
  int status = TEM_OK;
  for (int s = 0; s < S; ++s) {
    if (iters) iters[s] = st[s].iters;
    if (relres) relres[s] = st[s].relres;
    shift_iters += st[s].iters;
    max_it = std::max(max_it, st[s].iters);
    n_real += st[s].real ? 1 : 0;
    if (st[s].status == 2) status = TEM_EBREAKDOWN;
    else if (st[s].status != 1 && status == TEM_OK) status = TEM_ENOCONV;
  }
  c->stats.loop_ms = ms;
  c->stats.kernel_launches = launches;
  c->stats.shift_iterations = shift_iters;
  c->stats.iterations = max_it;
  c->stats.grid = grid;   // with all shifts active
  c->stats.block = block;
  c->stats.real_shifts = n_real;
  c->stats.persistent = c->last_persistent;
  c->last_fnorm = S > 0 ? st[0].fnorm : 0.0;
  if (status == TEM_EBREAKDOWN) return fail(status, "tem_cocg_solve: COCG breakdown");
  if (status == TEM_ENOCONV) return fail(status, "tem_cocg_solve: not converged within maxit");
  return TEM_OK;
}

// The persistent loop (tem_persist.cuh) only on request: measured on B200
// (scripts/launch_modes.py, profiles/r02/launch_modes.json) it is 2-14%
// slower than the graph path even on grids whose state fits in L2 (tiny,
// block, layered): a pass is bound by the per-SM plane-step rate of the
// 12-warp sweep CTAs, not by launch gaps, and the two grid barriers per
// iteration cost about what the graph's launch gaps do.
constexpr int kPersistIters = 1024;           // iterations per cooperative launch (host polls between)
static bool use_persistent(const tem_ctx* c, int S) {
  if (c->solver != TEM_SOLVER_SPLIT || c->per_sm_persist < 1 || S > tem::kMaxSlots) return false;
  return c->launch_mode == TEM_LAUNCH_PERSISTENT;
}

// clears ShiftState::real of shifts whose right-hand side is complex
__global__ void k_real_mask(tem::ShiftState* st, const int* flag, int S) {
  const int s = threadIdx.x;
  if (s < S && flag[s]) st[s].real = 0;
}

// Snapshot request of a solve (tem_forward's per-shift refinement targets,
// reading R13): when shift s is first seen at a graph boundary with relative
// residual <= tol, its x (complete there: graphs end on an odd iteration) is
// copied to buf (raw, in the shift's layout during the solve).
struct SolveSnap {
  double tol = 0.0;
  double2* buf = nullptr;
  std::vector<double> relres;   // at the snapshot
  std::vector<int> mode;        // 0 none, 1 complex, 2 real layout (tem::SnapArgs::mode)
};

// One batched solve.  Right-hand side: f (real, every shift) or rhs (a
// complex shift block, one per shift).  Tolerance: tols[s] (host) or tol.
static int solve(tem_ctx* c, const double* mass, const double* f, const double2* rhs, int S,
                 const double* shifts, double tol, const double* tols, int maxit, double* x, char* w,
                 const WorkLayout& L, int* iters, double* relres, cudaStream_t stream,
                 SolveSnap* snap = nullptr) {
  const bool split = c->solver == TEM_SOLVER_SPLIT;
  if (snap) {
    snap->relres.assign(S, 0.0);
    snap->mode.assign(S, 0);
  }
  using T2 = tem::Tile<tem::kTYTwoSweep>;
  using TS = tem::Tile<tem::kTYSplit>;
  const int ty = split ? tem::kTYSplit : tem::kTYTwoSweep;
  const int nt = split ? TS::NT : T2::NT;
  double2* Z[2] = {reinterpret_cast<double2*>(w + L.z), reinterpret_cast<double2*>(w + L.z1)};
  double2* P[2] = {reinterpret_cast<double2*>(w + L.p0), reinterpret_cast<double2*>(w + L.p1)};
  CUtensorMap tmZ[2], tmP[2], tmZr[2], tmPr[2];
  for (int q = 0; q < 2; ++q) {
    if (int rc = make_tmap(c, S, Z[q], &tmZ[q], ty)) return rc;
    if (int rc = make_tmap(c, S, P[q], &tmP[q], ty)) return rc;
    if (int rc = make_tmap(c, S, Z[q], &tmZr[q], ty, true)) return rc;
    if (int rc = make_tmap(c, S, P[q], &tmPr[q], ty, true)) return rc;
  }
  tem::SweepArgs base{};
  int grid = 0;
  sweep_geometry(c, S, S, base, &grid, ty);
  base.mass = mass;
  base.x = reinterpret_cast<double2*>(x);
  base.z = Z[0];
  base.rhs = rhs;
  base.st = reinterpret_cast<tem::ShiftState*>(w + L.st);
  base.ctl = reinterpret_cast<tem::Control*>(w + L.ctl);
  base.part_c = reinterpret_cast<double2*>(w + L.part_c);
  base.part_r = reinterpret_cast<double*>(w + L.part_r);
  base.part = reinterpret_cast<double*>(w + L.part9);
  base.pstride = (int)L.nparts;
  if (const char* env = getenv("TEM_XDIRECT")) base.force_xdirect = atoi(env);   // tests

  struct Cfg {
    tem::SweepArgs a1[2], a2[2];   // first / second kernel of an iteration, per parity
    int grid;
  };
  auto make_cfg = [&](int nslot) {
    Cfg k{};
    tem::SweepArgs g0 = base;
    sweep_geometry(c, S, nslot, g0, &k.grid, ty);
    for (int q = 0; q < 2; ++q) {
      k.a1[q] = g0;
      k.a1[q].out = P[1 - q];
      if (split) {
        k.a1[q].zin = Z[q];
        k.a1[q].z = Z[1 - q];
        k.a1[q].pold = P[q];
      }
      k.a2[q] = g0;
    }
    return k;
  };
  auto launch_iter = [&](const Cfg& k, int q, cudaStream_t st_) {
    if (split) {
      if (q == 0)
        tem::k_sweep<3><<<k.grid, TS::NT, TS::kSmemUpd, st_>>>(k.a1[0], tmP[0], tmZ[0], tmPr[0], tmZr[0]);
      else
        tem::k_sweep<4><<<k.grid, TS::NT, TS::kSmemDirap, st_>>>(k.a1[1], tmP[1], tmZ[1], tmPr[1], tmZr[1]);
      tem::k_delta<false><<<k.grid, TS::NT, TS::kSmemDelta, st_>>>(k.a2[q], tmZ[1 - q], tmZr[1 - q]);
    } else {
      tem::k_sweep<1><<<k.grid, T2::NT, T2::kSmemDirap, st_>>>(k.a1[q], tmP[q], tmZ[0], tmP[q], tmZ[0]);
      tem::k_sweep<2><<<k.grid, T2::NT, T2::kSmemDirect, st_>>>(k.a2[q], tmP[1 - q], tmP[1 - q], tmP[1 - q],
                                                                  tmP[1 - q]);
    }
  };
  // graphs of kChunk iterations, cached per (slots, z-chunks) for these buffers and this scheme
  const std::vector<const void*> key = {mass, x, w, f, rhs, reinterpret_cast<const void*>((uintptr_t)c->solver),
                                        reinterpret_cast<const void*>((uintptr_t)S)};
  if (!c->graphs.count(key) && c->graphs.size() >= 4) {
    for (auto& set : c->graphs)
      for (auto& kv : set.second) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
  }
  auto& gset = c->graphs[key];
  auto get_graph = [&](const Cfg& k, int nslot, cudaGraphExec_t* out) -> int {
    const long long id = (long long)nslot * 4096 + k.a1[0].nzc;
    auto it = gset.find(id);
    if (it != gset.end()) {
      *out = it->second;
      return TEM_OK;
    }
    cudaGraph_t gr;
    TEM_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < kChunk; ++i) launch_iter(k, i & 1, c->cap_stream);
    TEM_CUDA(cudaStreamEndCapture(c->cap_stream, &gr));
    cudaGraphExec_t ex;
    cudaError_t e = cudaGraphInstantiate(&ex, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) return fail(TEM_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    gset[id] = ex;
    *out = ex;
    return TEM_OK;
  };

  // per-shift state + control (host -> device, small)
  std::vector<tem::ShiftState> st(S);
  bool any_real = false;
  for (int s = 0; s < S; ++s) {
    memset(&st[s], 0, sizeof(tem::ShiftState));
    st[s].s = make_double2(shifts[2 * s], shifts[2 * s + 1]);
    st[s].tol = tols ? tols[s] : tol;
    st[s].real = (split && c->real_arith && shifts[2 * s + 1] == 0.0) ? 1 : 0;
    any_real |= st[s].real != 0;
  }
  tem::Control ctl{};
  TEM_CUDA(cudaMemcpyAsync(base.st, st.data(), sizeof(tem::ShiftState) * S, cudaMemcpyHostToDevice, stream));
  TEM_CUDA(cudaMemcpyAsync(base.ctl, &ctl, sizeof(tem::Control), cudaMemcpyHostToDevice, stream));

  TEM_CUDA(cudaEventRecord(c->ev0, stream));
  long long launches = 0;
  if (rhs && any_real) {   // a real shift with a complex right-hand side runs in complex arithmetic
    int* flags = reinterpret_cast<int*>(w + L.flags);
    TEM_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * TEM_MAX_SHIFTS, stream));
    k_rhs_imag<<<dim3(64, S), 256, 0, stream>>>(rhs, 3 * c->g.Nn, flags);
    k_real_mask<<<1, 32, 0, stream>>>(base.st, flags, S);
    TEM_CUDA(cudaGetLastError());
    launches += 2;
  }
  // pairs of real shifts share a slot (R16); the persistent path runs them singly
  const bool persistent = split && use_persistent(c, S);
  const int pairing = split && c->real_arith && any_real && !persistent && !getenv("TEM_NO_PAIR");
  k_pair<<<1, 32, 0, stream>>>(base.st, S, pairing);
  launches += 1;
  const bool dbg = getenv("TEM_DEBUG_SYNC") != nullptr;   // debugging: locate a failing launch
#define TEM_DBG(name)                                                                               \
  if (dbg) {                                                                                        \
    cudaError_t e_ = cudaStreamSynchronize(stream);                                                 \
    if (e_ != cudaSuccess) return fail(TEM_ECUDA, std::string(name) + ": " + cudaGetErrorString(e_)); \
  }
  const int vec_grid = S * std::max(1, std::min(64, (int)((3 * c->g.Nn + 255) / 256)));
  k_init<<<vec_grid, 256, 0, stream>>>(base, P[0], P[1], split ? Z[1] : nullptr, f);
  TEM_CUDA(cudaGetLastError());
  TEM_DBG("k_init");
  launches += 1;
  int nslot = S;
  Cfg cfg = make_cfg(nslot);
  if (split) {
    tem::k_delta<true><<<cfg.grid, TS::NT, TS::kSmemDelta, stream>>>(cfg.a2[0], tmZ[0], tmZr[0]);   // delta_0
    TEM_CUDA(cudaGetLastError());
    TEM_DBG("k_delta<true>");
    launches += 1;
  }

  const bool trace = getenv("TEM_TRACE") != nullptr;
  auto t_prev = std::chrono::steady_clock::now();
  int done = 0;
  c->last_persistent = persistent ? 1 : 0;
  if (c->last_persistent) {
    // one cooperative launch runs up to kPersistIters iterations; z-chunking
    // per active-slot count for one resident CTA per SM (latency regime)
    tem::PersistArgs PA{};
    PA.A = base;
    for (int q = 0; q < 2; ++q) {
      PA.Z[q] = Z[q];
      PA.P[q] = P[q];
    }
    for (int ns = 1; ns <= S; ++ns) {
      tem::SweepArgs g0 = base;
      int gr = 0;
      sweep_geometry(c, S, ns, g0, &gr, ty, c->per_sm_persist);
      PA.nzc[ns] = g0.nzc;
      PA.kchunk[ns] = g0.kchunk;
    }
    PA.gbar = reinterpret_cast<unsigned*>(w + L.gbar);
    TEM_CUDA(cudaMemsetAsync(PA.gbar, 0, 2 * sizeof(unsigned), stream));
    const int pgrid = c->num_sms * c->per_sm_persist;
    while (done < maxit) {
      PA.it0 = done;
      PA.n_iter = std::min(kPersistIters, maxit - done);
      void* args[] = {&PA, &tmZ[0], &tmZ[1], &tmP[0], &tmP[1], &tmZr[0], &tmZr[1], &tmPr[0], &tmPr[1]};
      TEM_CUDA(cudaLaunchCooperativeKernel((const void*)tem::k_persist<>, dim3(pgrid), dim3(TS::NT), args,
                                           TS::kSmemUpd, stream));
      TEM_DBG("k_persist");
      launches += 1;
      done += PA.n_iter;
      TEM_CUDA(cudaMemcpyAsync(c->pinned_active, &base.ctl->n_active, sizeof(int), cudaMemcpyDeviceToHost, stream));
      TEM_CUDA(cudaStreamSynchronize(stream));
      if (trace) {
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[tem trace] persistent it<=%d grid=%d active=%d launch_ms=%.3f\n", done, pgrid,
                *c->pinned_active, std::chrono::duration<double, std::milli>(now - t_prev).count());
        t_prev = now;
      }
      if (*c->pinned_active == 0) break;
    }
  }
  bool snap_pending = snap != nullptr;
  cudaGraphExec_t graph = nullptr;
  if (!c->last_persistent)
    if (int rc = get_graph(cfg, nslot, &graph)) return rc;
  while (!c->last_persistent && done < maxit) {
    const int chunk = std::min(kChunk, maxit - done);
    if (chunk == kChunk && !dbg) {  // kChunk is even: parity returns to 0
      TEM_CUDA(cudaGraphLaunch(graph, stream));
    } else {
      for (int i = 0; i < chunk; ++i) {
        launch_iter(cfg, (done + i) & 1, stream);
        TEM_CUDA(cudaGetLastError());
        TEM_DBG(((done + i) & 1) ? "iteration (odd)" : "iteration (even)");
      }
    }
    launches += 2LL * chunk;
    done += chunk;
    TEM_CUDA(cudaMemcpyAsync(c->pinned_active, &base.ctl->n_active, sizeof(int), cudaMemcpyDeviceToHost, stream));
    TEM_CUDA(cudaStreamSynchronize(stream));
    const int n_active = *c->pinned_active;
    if (trace) {
      const auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "[tem trace] it=%d slots=%d nzc=%d grid=%d active=%d chunk_ms=%.3f\n", done, nslot,
              cfg.a1[0].nzc, cfg.grid, n_active,
              std::chrono::duration<double, std::milli>(now - t_prev).count());
      t_prev = now;
    }
    if (snap && snap_pending && split && chunk == kChunk && !dbg) {
      std::vector<tem::ShiftState> hs(S);
      TEM_CUDA(cudaMemcpy(hs.data(), base.st, sizeof(tem::ShiftState) * S, cudaMemcpyDeviceToHost));
      const size_t vb = (size_t)3 * c->g.Nn * sizeof(double2);
      snap_pending = false;
      for (int s = 0; s < S; ++s) {
        if (!snap->mode[s] && hs[s].active && hs[s].relres <= snap->tol) {
          // a pair's x is packed in its leader's block (component x: leader, y: partner)
          const int src = hs[s].pair && !hs[s].lead ? hs[s].pair - 1 : s;
          TEM_CUDA(cudaMemcpyAsync(snap->buf + (size_t)s * 3 * c->g.Nn, reinterpret_cast<double2*>(x) +
                                   (size_t)src * 3 * c->g.Nn, vb, cudaMemcpyDeviceToDevice, stream));
          snap->mode[s] = hs[s].pair ? (hs[s].lead ? 3 : 4) : hs[s].real ? 2 : 1;
          snap->relres[s] = hs[s].relres;
        }
        snap_pending |= !snap->mode[s] && hs[s].active;   // still to be taken
      }
    }
    if (n_active == 0) break;
    if (n_active < nslot) {  // shifts converged: fewer slots, possibly more z-chunks
      nslot = n_active;
      cfg = make_cfg(nslot);
      if (int rc = get_graph(cfg, nslot, &graph)) return rc;
    }
  }
  if (split) {
    k_xfix<<<vec_grid, 256, 0, stream>>>(base, P[1]);
    launches += 1;
    TEM_DBG("k_xfix");
    if (any_real) {   // real-layout / pair-packed x of real shifts -> complex ABI layout (Z[0] as scratch)
      if (pairing) {
        k_pair_out<<<vec_grid, 256, 0, stream>>>(base);
        launches += 1;
      }
      k_real_out<<<vec_grid, 256, 0, stream>>>(base, Z[0], 0);
      k_real_out<<<vec_grid, 256, 0, stream>>>(base, Z[0], 1);
      launches += 2;
    }
    TEM_CUDA(cudaGetLastError());
    TEM_DBG("k_real_out");
#undef TEM_DBG
  }
  TEM_CUDA(cudaEventRecord(c->ev1, stream));
  return finish_solve(c, S, st, base.st, stream, launches, grid, nt, iters, relres);
}

int tem_cocg_solve(tem_ctx* c, const double* mass, const double* f, int S, const double* shifts,
                   double tol, int maxit, double* x, void* work, size_t work_bytes, int* iters,
                   double* relres, void* stream_) {
  if (!c || !mass || !f || !shifts || !x || !work) return fail(TEM_EINVAL, "tem_cocg_solve: null pointer");
  if (int rc = check_S(S)) return rc;
  if (!(tol > 0.0) || maxit < 1) return fail(TEM_EINVAL, "tem_cocg_solve: need tol > 0, maxit >= 1");
  if (int rc = check_device(c)) return rc;
  const WorkLayout L = work_layout(c, S);
  if (work_bytes < L.total) return fail(TEM_EINVAL, "tem_cocg_solve: workspace too small");
  return solve(c, mass, f, nullptr, S, shifts, tol, nullptr, maxit, x, static_cast<char*>(work), L, iters,
               relres, (cudaStream_t)stream_);
}

int tem_cocg_solve_rhs(tem_ctx* c, const double* mass, const double* rhs, int S, const double* shifts,
                       const double* tols, int maxit, double* x, void* work, size_t work_bytes, int* iters,
                       double* relres, void* stream_) {
  if (!c || !mass || !rhs || !shifts || !tols || !x || !work)
    return fail(TEM_EINVAL, "tem_cocg_solve_rhs: null pointer");
  if (int rc = check_S(S)) return rc;
  if (int rc = check_device(c)) return rc;
  if (int rc = check_index(c, S)) return rc;
  if (maxit < 1) return fail(TEM_EINVAL, "tem_cocg_solve_rhs: need maxit >= 1");
  for (int s = 0; s < S; ++s)
    if (!(tols[s] > 0.0)) return fail(TEM_EINVAL, "tem_cocg_solve_rhs: need tols[s] > 0");
  if (rhs == x) return fail(TEM_EINVAL, "tem_cocg_solve_rhs: rhs and x must not alias");
  const WorkLayout L = work_layout(c, S);
  if (work_bytes < L.total) return fail(TEM_EINVAL, "tem_cocg_solve_rhs: workspace too small");
  return solve(c, mass, nullptr, reinterpret_cast<const double2*>(rhs), S, shifts, 0.0, tols, maxit, x,
               static_cast<char*>(work), L, iters, relres, (cudaStream_t)stream_);
}

int tem_set_solver(tem_ctx* c, int solver) {
  if (!c) return fail(TEM_EINVAL, "tem_set_solver: null context");
  if (solver != TEM_SOLVER_SPLIT && solver != TEM_SOLVER_TWO_SWEEP)
    return fail(TEM_EINVAL, "tem_set_solver: unknown solver " + std::to_string(solver));
  c->solver = solver;
  return TEM_OK;
}

int tem_get_solver(const tem_ctx* c) { return c ? c->solver : TEM_EINVAL; }

int tem_set_launch_mode(tem_ctx* c, int mode) {
  if (!c) return fail(TEM_EINVAL, "tem_set_launch_mode: null context");
  if (mode != TEM_LAUNCH_AUTO && mode != TEM_LAUNCH_GRAPHS && mode != TEM_LAUNCH_PERSISTENT)
    return fail(TEM_EINVAL, "tem_set_launch_mode: unknown mode " + std::to_string(mode));
  if (mode == TEM_LAUNCH_PERSISTENT && c->per_sm_persist < 1)
    return fail(TEM_EINVAL, "tem_set_launch_mode: k_persist cannot be made resident on this device");
  c->launch_mode = mode;
  return TEM_OK;
}
int tem_get_launch_mode(const tem_ctx* c) { return c ? c->launch_mode : TEM_EINVAL; }

int tem_last_solve_stats(const tem_ctx* c, tem_solve_stats* out) {
  if (!c || !out) return fail(TEM_EINVAL, "tem_last_solve_stats: null pointer");
  *out = c->stats;
  return TEM_OK;
}

// Small host arrays (residues, receivers) reach the device through a
// context-owned pinned staging buffer: the copy is asynchronous on the
// caller's stream and the pageable caller array may be reused on return.
// The staging buffer is rewritten only after the previous copy out of it
// has completed (stage_ev); the device scratch is stream-ordered (calls on
// one context are issued on one stream, include/tem_b200.h).
static int stage_to_device(tem_ctx* c, const void* const* src, const size_t* bytes, int n, cudaStream_t stream) {
  size_t total = 0;
  for (int i = 0; i < n; ++i) total += align_up(bytes[i], 256);
  if (c->stage_ev) TEM_CUDA(cudaEventSynchronize(c->stage_ev));
  if (c->pin_bytes < total) {
    if (c->pin) cudaFreeHost(c->pin);
    c->pin = nullptr;
    c->pin_bytes = 0;
    TEM_CUDA(cudaMallocHost(&c->pin, total));
    c->pin_bytes = total;
  }
  if (c->scratch_bytes < total) {
    if (c->scratch) {
      TEM_CUDA(cudaStreamSynchronize(stream));   // a queued kernel may still read the old scratch
      cudaFree(c->scratch);
    }
    c->scratch = nullptr;
    c->scratch_bytes = 0;
    TEM_CUDA(cudaMalloc(&c->scratch, total));
    c->scratch_bytes = total;
  }
  size_t o = 0;
  for (int i = 0; i < n; ++i) {
    memcpy(static_cast<char*>(c->pin) + o, src[i], bytes[i]);
    o += align_up(bytes[i], 256);
  }
  TEM_CUDA(cudaMemcpyAsync(c->scratch, c->pin, total, cudaMemcpyHostToDevice, stream));
  TEM_CUDA(cudaEventRecord(c->stage_ev, stream));
  return TEM_OK;
}

// u = sum_s w_s Re(res[k][s] x_s), residues [K][S] complex on the host.
static int synth(tem_ctx* c, int S, int K, const double* residues, const int* is_pair, const double2* x,
                 double* u, cudaStream_t stream) {
  const size_t res_bytes = (size_t)K * S * sizeof(double2);
  const size_t smem = res_bytes;
  if (smem > 200 * 1024) return fail(TEM_EINVAL, "tem_synthesize: K*S too large for shared memory");
  double wts[TEM_MAX_SHIFTS];
  for (int s = 0; s < S; ++s) wts[s] = is_pair[s] ? 2.0 : 1.0;
  const void* src[2] = {residues, wts};
  const size_t bytes[2] = {res_bytes, S * sizeof(double)};
  if (int rc = stage_to_device(c, src, bytes, 2, stream)) return rc;
  char* sc = static_cast<char*>(c->scratch);
  const double2* res_d = reinterpret_cast<const double2*>(sc);
  const double* w_d = reinterpret_cast<const double*>(sc + align_up(res_bytes, 256));
  const long long nslots = 3 * c->g.Nn;
  const int block = 128;
  const int grid = (int)std::min<long long>((nslots + block - 1) / block, (long long)c->num_sms * 16);
#define TEM_SYNTH(SM)                                                                      \
  do {                                                                                     \
    if (smem > 48 * 1024)                                                                  \
      TEM_CUDA(cudaFuncSetAttribute(k_synth<SM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_synth<SM><<<grid, block, smem, stream>>>(c->g, S, K, res_d, w_d, x, u);              \
  } while (0)
  if (S <= 8) TEM_SYNTH(8);
  else if (S <= 16) TEM_SYNTH(16);
  else if (S <= 24) TEM_SYNTH(24);
  else TEM_SYNTH(32);
#undef TEM_SYNTH
  TEM_CUDA(cudaGetLastError());
  return TEM_OK;
}

int tem_synthesize(tem_ctx* c, int S, int K, const double* residues, const int* is_pair,
                   const double* x, double* u, void* stream_) {
  if (!c || !residues || !is_pair || !x || !u) return fail(TEM_EINVAL, "tem_synthesize: null pointer");
  if (int rc = check_S(S)) return rc;
  if (int rc = check_device(c)) return rc;
  if (int rc = check_index(c, S)) return rc;
  if (K < 1) return fail(TEM_EINVAL, "tem_synthesize: K must be >= 1");
  return synth(c, S, K, residues, is_pair, reinterpret_cast<const double2*>(x), u, (cudaStream_t)stream_);
}

int tem_curl_z(tem_ctx* c, int K, const double* u, int R, const int* receivers, double* out, void* stream_) {
  if (!c || !u || !receivers || !out) return fail(TEM_EINVAL, "tem_curl_z: null pointer");
  if (K < 1 || R < 1) return fail(TEM_EINVAL, "tem_curl_z: need K >= 1, R >= 1");
  if (int rc = check_device(c)) return rc;
  for (int r = 0; r < R; ++r) {
    const int i = receivers[3 * r], j = receivers[3 * r + 1], k = receivers[3 * r + 2];
    if (i < 0 || i >= c->g.n[0] || j < 0 || j >= c->g.n[1] || k < 0 || k > c->g.n[2])
      return fail(TEM_EINVAL, "tem_curl_z: receiver " + std::to_string(r) + " outside the grid");
  }
  cudaStream_t stream = (cudaStream_t)stream_;
  const void* src[1] = {receivers};
  const size_t bytes[1] = {(size_t)3 * R * sizeof(int)};
  if (int rc = stage_to_device(c, src, bytes, 1, stream)) return rc;
  const int n = K * R, block = 256;
  k_curl_z<<<(n + block - 1) / block, block, 0, stream>>>(c->g, K, R, static_cast<const int*>(c->scratch),
                                                          u, out);
  TEM_CUDA(cudaGetLastError());
  return TEM_OK;
}

// ------------------------------------------------------------ forward
// tem_forward: solve, synthesise, and (opts->max_refine > 0) refine until
// the channels are converged (reading R13).
struct FwdLayout {
  size_t cocg, r, d, part, out, total;
  int nblk;
};

static FwdLayout fwd_layout(const tem_ctx* c, int S, int K) {
  FwdLayout L{};
  const size_t vec = (size_t)3 * c->g.Nn * S * sizeof(double2);
  L.nblk = 2 * std::max(1, c->num_sms);
  const size_t rows = (size_t)std::max(4 * S, K);
  size_t o = 0;
  L.cocg = o;  o = align_up(o + work_layout(c, S).total, 256);
  L.r = o;     o = align_up(o + vec, 256);
  L.d = o;     o = align_up(o + vec, 256);
  L.part = o;  o = align_up(o + rows * L.nblk * sizeof(double), 256);
  L.out = o;   o = align_up(o + rows * sizeof(double), 256);
  L.total = o;
  return L;
}

// device rows -> host: out[row] = sum_b part[row][b]
static int rows_to_host(tem_ctx* c, const double* part, int nrow, int ncol, double* dev_out, double* host,
                        cudaStream_t stream) {
  k_rows_sum<<<(nrow + 7) / 8, 256, 0, stream>>>(part, nrow, ncol, dev_out);
  TEM_CUDA(cudaGetLastError());
  TEM_CUDA(cudaMemcpyAsync(host, dev_out, nrow * sizeof(double), cudaMemcpyDeviceToHost, stream));
  TEM_CUDA(cudaStreamSynchronize(stream));
  return TEM_OK;
}

static int resid_dd(tem_ctx* c, const double* mass, const double* f, int S, const double* shifts,
                    const std::vector<int>& list, const double2* x, double2* r, const FwdLayout& L, char* w,
                    std::vector<double>& res2, cudaStream_t stream, std::vector<double>* abs2 = nullptr) {
  tem::ResidArgs A{};
  A.g = c->g;
  A.mass = mass;
  A.f = f;
  A.x = x;
  A.r = r;
  A.part = reinterpret_cast<double*>(w + L.part);
  const int n = (int)list.size();
  A.part_abs = abs2 ? A.part + (size_t)n * L.nblk : nullptr;
  for (int y = 0; y < n; ++y) {
    A.list[y] = list[y];
    A.shifts[y] = make_double2(shifts[2 * list[y]], shifts[2 * list[y] + 1]);
  }
  tem::k_resid_dd<<<dim3(L.nblk, n), 256, 0, stream>>>(A);
  TEM_CUDA(cudaGetLastError());
  std::vector<double> both(abs2 ? 2 * n : n, 0.0);
  if (int rc = rows_to_host(c, A.part, (int)both.size(), L.nblk, reinterpret_cast<double*>(w + L.out), both.data(),
                           stream))
    return rc;
  res2.assign(both.begin(), both.begin() + n);
  if (abs2) abs2->assign(both.begin() + n, both.end());
  return TEM_OK;
}

static int forward(tem_ctx* c, const double* mass, const double* f, int S, const double* shifts, int K,
                   const double* residues, const int* is_pair, const tem_forward_opts& o, double* x, double* u,
                   char* w, const FwdLayout& L, int* iters, double* relres, tem_forward_stats* fst,
                   cudaStream_t stream) {
  const WorkLayout WL = work_layout(c, S);
  char* wc = w + L.cocg;
  double2* xc = reinterpret_cast<double2*>(x);
  double2* r = reinterpret_cast<double2*>(w + L.r);
  double2* d = reinterpret_cast<double2*>(w + L.d);
  const size_t vec1 = (size_t)3 * c->g.Nn * sizeof(double2);
  std::vector<int> it(S, 0), it1(S, 0);
  std::vector<double> rr(S, 0.0);
  tem_forward_stats F{};
  // with refinement: snapshot each shift's x at 10x the first-solve
  // tolerance (into r, unused until the first residual) for its refinement target
  SolveSnap snap;
  snap.tol = 10.0 * o.tol;
  snap.buf = r;
  const bool targets = o.max_refine > 0 && c->solver == TEM_SOLVER_SPLIT && !getenv("TEM_UNIFORM_REFINE");
  int rc_solve = solve(c, mass, f, nullptr, S, shifts, o.tol, nullptr, o.maxit, x, wc, WL, it.data(), rr.data(),
                       stream, targets ? &snap : nullptr);
  if (rc_solve == TEM_ECUDA || rc_solve == TEM_EINVAL) return rc_solve;
  std::string solve_msg = g_last_error;
  F.shift_iterations = c->stats.shift_iterations;
  F.loop_ms = c->stats.loop_ms;
  F.kernel_launches = c->stats.kernel_launches + 1;   // + synthesis
  F.initial_shift_iterations = c->stats.shift_iterations;
  const double fnorm = c->last_fnorm;
  if (int rc = synth(c, S, K, residues, is_pair, xc, u, stream)) return rc;
  F.channel_bound = -1.0;   // not estimated (no refinement)
  if (o.max_refine > 0 && rc_solve == TEM_OK && fnorm > 0.0) {
    // ||u_k||_M per channel (the yardstick of the channel-aware rule)
    double* part = reinterpret_cast<double*>(w + L.part);
    double* dout = reinterpret_cast<double*>(w + L.out);
    k_channel_mnorm<<<dim3(L.nblk, K), 256, 0, stream>>>(3 * c->g.Nn, mass, u, part);
    TEM_CUDA(cudaGetLastError());
    F.kernel_launches += 4;   // channel norms, first residual, their two reductions
    std::vector<double> unorm(K);
    if (int rc = rows_to_host(c, part, K, L.nblk, dout, unorm.data(), stream)) return rc;
    for (auto& v : unorm) v = sqrt(v);
    std::vector<int> list(S);
    for (int s = 0; s < S; ++s) list[s] = s;
    std::vector<double> tols(S, o.refine_tol);
    // Per-shift targets: the error left in x_s after the first solve is
    // estimated from how far x_s moved between the snapshot (relative
    // residual rho_snap ~ 10 tol) and the end (rho_end ~ tol):
    //   E_s = safety * (rho_end / rho_snap) * max_k ||w_s Re(alpha_ks (x_s - snap_s))||_M / ||u_k||_M
    // (the error contracts with the residual, measured ~1x per decade).
    // Shift s is asked for the reduction that leaves it at most a quarter of
    // its share of the target, eta_s = channel_tol / (4 S E_s), but never
    // for less than refine_tol (the slow shifts, whose E_s the snapshot
    // overestimates by 10^2-10^3, get exactly refine_tol), and a shift whose
    // eta_s is >= 1/2 is not refined.  Measured on `large` (R13) the estimate
    // is 1.2-12x above the true error for the fast shifts it decides about.
    bool any_snap = false;
    for (int s = 0; s < S; ++s) any_snap |= targets && snap.mode[s] != 0;
    if (any_snap) {
      tem::SnapArgs SA{};
      SA.g = c->g;
      SA.mass = mass;
      SA.x = xc;
      SA.snap = r;
      SA.d = d;
      SA.part = part;
      for (int s = 0; s < S; ++s) SA.mode[s] = snap.mode[s];
      tem::k_snap_delta<<<dim3(L.nblk, S), 256, 0, stream>>>(SA);
      TEM_CUDA(cudaGetLastError());
      F.kernel_launches += 2;
      std::vector<double> mom(3 * S);
      if (int rc = rows_to_host(c, part, 3 * S, L.nblk, dout, mom.data(), stream)) return rc;
      std::vector<double> E(S, -1.0);
      for (int s = 0; s < S; ++s) {
        if (!snap.mode[s] || !(snap.relres[s] > 0.0)) continue;
        const double ratio = rr[s] / snap.relres[s];
        const double wgt = is_pair[s] ? 2.0 : 1.0;
        double e = 0.0;
        for (int k = 0; k < K; ++k) {
          const double ar = residues[2 * ((size_t)k * S + s)], ai = residues[2 * ((size_t)k * S + s) + 1];
          const double q = ar * ar * mom[3 * s] + ai * ai * mom[3 * s + 1] - 2.0 * ar * ai * mom[3 * s + 2];
          e = std::max(e, wgt * sqrt(std::max(q, 0.0)) / std::max(unorm[k], 1e-300));
        }
        E[s] = o.safety * ratio * e;
      }
      std::vector<int> keep;
      for (int s = 0; s < S; ++s) {
        double eta = o.refine_tol;
        if (E[s] >= 0.0)
          eta = std::max(o.refine_tol, std::min(1.0, o.channel_tol / (4.0 * S * std::max(E[s], 1e-300))));
        if (getenv("TEM_TRACE"))
          fprintf(stderr, "[tem trace] refine target shift %d E %.3e eta %.3e%s\n", s, E[s], eta,
                  eta >= 0.5 ? " (not refined)" : "");
        if (eta < 0.5) {
          keep.push_back(s);
          tols[s] = eta;
        }
      }
      list = keep;
      F.kernel_launches += 0;
    }
    std::vector<double> res_prev(S), res_now;
    for (int s = 0; s < S; ++s) res_prev[s] = rr[s] * fnorm;   // unrefined shifts: the solve's own residual
    if (!list.empty())
      if (int rc = resid_dd(c, mass, f, S, shifts, list, xc, r, L, w, res_now, stream)) return rc;
    for (size_t y = 0; y < list.size(); ++y) res_prev[list[y]] = sqrt(res_now[y]);
    for (int round = 1; round <= o.max_refine && !list.empty(); ++round) {
      // right-hand sides: r for the refined shifts (written by resid_dd), 0 for the others
      std::vector<char> on(S, 0);
      for (int s : list) on[s] = 1;
      for (int s = 0; s < S; ++s)
        if (!on[s]) TEM_CUDA(cudaMemsetAsync(r + (size_t)s * 3 * c->g.Nn, 0, vec1, stream));
      std::vector<double> eta(S, 0.0);   // residual reduction each correction solve achieved
      const int rc2 = solve(c, mass, nullptr, r, S, shifts, 0.0, tols.data(), o.maxit, reinterpret_cast<double*>(d),
                            wc, WL, it1.data(), eta.data(), stream);
      if (rc2 == TEM_ECUDA || rc2 == TEM_EINVAL) return rc2;
      if (rc2 != TEM_OK && rc_solve == TEM_OK) {
        rc_solve = rc2;
        solve_msg = g_last_error;
      }
      for (int s = 0; s < S; ++s) it[s] += it1[s];
      F.shift_iterations += c->stats.shift_iterations;
      F.loop_ms += c->stats.loop_ms;
      F.kernel_launches += c->stats.kernel_launches + 4;   // + update, residual and their two reductions
      F.refine_rounds = round;
      // x += d, and the M-weighted statistics of d
      tem::UpdateArgs U{};
      U.Nn = c->g.Nn;
      U.mass = mass;
      U.x = xc;
      U.d = d;
      U.part = part;
      const int n = (int)list.size();
      for (int y = 0; y < n; ++y) U.list[y] = list[y];
      tem::k_refine_update<<<dim3(L.nblk, n), 256, 0, stream>>>(U);
      TEM_CUDA(cudaGetLastError());
      std::vector<double> dst(4 * n);
      if (int rc = rows_to_host(c, part, 4 * n, L.nblk, dout, dst.data(), stream)) return rc;
      std::vector<double> abs_now;
      if (int rc = resid_dd(c, mass, f, S, shifts, list, xc, r, L, w, res_now, stream, &abs_now)) return rc;
      // per shift: the contraction this round achieved, c_s = min(1, safety *
      // residual ratio) (an allowance for the error-to-residual
      // amplification), and the triangle-inequality size of its correction
      // in each channel
      std::vector<double> worst(S, 0.0), contr(S, 0.0);
      for (int y = 0; y < n; ++y) {
        const int s = list[y];
        const double rho_after = sqrt(res_now[y]);
        // the part of ||r after|| explained by the rounding of x itself,
        // 2^-52 || |A| |x| ||, carries no error in the directions the channels
        // see (its preimage is the rounding of x); what the correction solve
        // left beyond it is max(eta_s, (||r after|| - floor) / ||r before||)
        const double floor_s = 0x1p-52 * sqrt(std::max(abs_now[y], 0.0));
        const double ratio = std::max(eta[s], (rho_after - floor_s) / std::max(res_prev[s], 1e-300));
        contr[s] = std::min(1.0, o.safety * ratio);
        const double wgt = is_pair[s] ? 2.0 : 1.0;
        for (int k = 0; k < K; ++k) {
          const double ar = residues[2 * ((size_t)k * S + s)], ai = residues[2 * ((size_t)k * S + s) + 1];
          const double q = ar * ar * dst[4 * y] + ai * ai * dst[4 * y + 1] - 2.0 * ar * ai * dst[4 * y + 2];
          worst[s] = std::max(worst[s], wgt * sqrt(std::max(q, 0.0)) / std::max(unorm[k], 1e-300));
        }
        res_prev[s] = rho_after;
      }
      // the error left in channel k is estimated as the round's correction of
      // every shift scaled by that shift's contraction, synthesised with
      // cancellation: ||sum_s w_s c_s Re(alpha_ks d_s)||_M / ||u_k||_M (per-shift
      // terms cancel in late channels as the fields do, eq:rmj)
      {
        double wts[TEM_MAX_SHIFTS];
        for (int s = 0; s < S; ++s) wts[s] = (is_pair[s] ? 2.0 : 1.0) * contr[s];
        const void* src[2] = {residues, wts};
        const size_t bytes[2] = {(size_t)K * S * sizeof(double2), S * sizeof(double)};
        if (int rc = stage_to_device(c, src, bytes, 2, stream)) return rc;
        const char* sc = static_cast<const char*>(c->scratch);
        const double2* res_d = reinterpret_cast<const double2*>(sc);
        const double* w_d = reinterpret_cast<const double*>(sc + align_up(bytes[0], 256));
        tem::k_dsynth_mnorm<<<dim3(L.nblk, (K + tem::kCB - 1) / tem::kCB), 256, 0, stream>>>(
            3 * c->g.Nn, mass, S, K, res_d, w_d, d, part);
        TEM_CUDA(cudaGetLastError());
        F.kernel_launches += 2;
      }
      std::vector<double> dch(K);
      if (int rc = rows_to_host(c, part, K, L.nblk, dout, dch.data(), stream)) return rc;
      double bound = 0.0;
      for (int k = 0; k < K; ++k) bound = std::max(bound, sqrt(std::max(dch[k], 0.0)) / std::max(unorm[k], 1e-300));
      F.channel_bound = bound;
      if (bound <= o.channel_tol) break;
      // next round: every shift whose own correction could still matter
      // (triangle size above its share of the target), each asked for the
      // residual reduction that brings the estimate to half the target
      const double eta_next = std::min(o.refine_tol, std::max(1e-9, 0.5 * o.channel_tol / (o.safety * bound)));
      std::vector<int> next;
      for (int s : list)
        if (worst[s] * contr[s] > o.channel_tol / S) {
          next.push_back(s);
          tols[s] = eta_next;
        }
      list = next;
      if (list.empty()) break;
    }
    for (int s = 0; s < S; ++s) rr[s] = res_prev[s] / fnorm;
    if (int rc = synth(c, S, K, residues, is_pair, xc, u, stream)) return rc;
    F.kernel_launches += 1;
  }
  double rmax = 0.0;
  for (int s = 0; s < S; ++s) {
    if (iters) iters[s] = it[s];
    if (relres) relres[s] = rr[s];
    rmax = std::max(rmax, rr[s]);
  }
  F.relres_max = rmax;
  if (fst) *fst = F;
  c->fstats = F;
  if (rc_solve != TEM_OK) return fail(rc_solve, solve_msg);
  return TEM_OK;
}

static int check_opts(const tem_forward_opts* o) {
  if (!(o->tol > 0.0) || o->maxit < 1 || o->max_refine < 0)
    return fail(TEM_EINVAL, "tem_forward: need tol > 0, maxit >= 1, max_refine >= 0");
  if (o->max_refine > 0 && !(o->refine_tol > 0.0 && o->refine_tol < 1.0 && o->channel_tol > 0.0 && o->safety >= 1.0))
    return fail(TEM_EINVAL, "tem_forward: need 0 < refine_tol < 1, channel_tol > 0, safety >= 1");
  return TEM_OK;
}

size_t tem_forward_workspace_bytes(const tem_ctx* c, int S, int K) {
  if (!c || S < 1 || S > TEM_MAX_SHIFTS || K < 1) return 0;
  return fwd_layout(c, S, K).total;
}

void tem_forward_default_opts(tem_forward_opts* o) {
  if (!o) return;
  o->tol = 1e-10;
  o->maxit = 200000;
  o->max_refine = 0;
  o->refine_tol = 1e-4;
  o->channel_tol = 1e-7;
  o->safety = 1.5;
}

int tem_forward(tem_ctx* c, const double* mass, const double* f, int S, const double* shifts, int K,
                const double* residues, const int* is_pair, const tem_forward_opts* opts, double* x, double* u,
                void* work, size_t work_bytes, int* iters, double* relres, tem_forward_stats* fst,
                void* stream) {
  if (!c || !mass || !f || !shifts || !residues || !is_pair || !opts || !x || !u || !work)
    return fail(TEM_EINVAL, "tem_forward: null pointer");
  if (int rc = check_S(S)) return rc;
  if (int rc = check_device(c)) return rc;
  if (int rc = check_index(c, S)) return rc;
  if (K < 1) return fail(TEM_EINVAL, "tem_forward: K must be >= 1");
  if (int rc = check_opts(opts)) return rc;
  const FwdLayout L = fwd_layout(c, S, K);
  if (work_bytes < L.total) return fail(TEM_EINVAL, "tem_forward: workspace too small");
  return forward(c, mass, f, S, shifts, K, residues, is_pair, *opts, x, u, static_cast<char*>(work), L, iters,
                 relres, fst, (cudaStream_t)stream);
}

int tem_residual(tem_ctx* c, const double* mass, const double* f, int S, const double* shifts, const double* x,
                 double* r, double* rnorm, void* stream_) {
  if (!c || !mass || !f || !shifts || !x || !r) return fail(TEM_EINVAL, "tem_residual: null pointer");
  if (int rc = check_S(S)) return rc;
  if (int rc = check_device(c)) return rc;
  if (int rc = check_index(c, S)) return rc;
  if (x == r) return fail(TEM_EINVAL, "tem_residual: x and r must not alias");
  cudaStream_t stream = (cudaStream_t)stream_;
  const int nblk = 2 * std::max(1, c->num_sms);
  const size_t need = ((size_t)S * nblk + TEM_MAX_SHIFTS) * sizeof(double);
  if (c->red_bytes < need) {
    if (c->red) {
      TEM_CUDA(cudaStreamSynchronize(stream));
      cudaFree(c->red);
    }
    c->red = nullptr;
    c->red_bytes = 0;
    TEM_CUDA(cudaMalloc(&c->red, need));
    c->red_bytes = need;
  }
  tem::ResidArgs A{};
  A.g = c->g;
  A.mass = mass;
  A.f = f;
  A.x = reinterpret_cast<const double2*>(x);
  A.r = reinterpret_cast<double2*>(r);
  A.part = static_cast<double*>(c->red);
  for (int y = 0; y < S; ++y) {
    A.list[y] = y;
    A.shifts[y] = make_double2(shifts[2 * y], shifts[2 * y + 1]);
  }
  tem::k_resid_dd<<<dim3(nblk, S), 256, 0, stream>>>(A);
  TEM_CUDA(cudaGetLastError());
  if (!rnorm) return TEM_OK;
  double* dout = static_cast<double*>(c->red) + (size_t)S * nblk;
  std::vector<double> rr(S);
  if (int rc = rows_to_host(c, A.part, S, nblk, dout, rr.data(), stream)) return rc;
  for (int y = 0; y < S; ++y) rnorm[y] = sqrt(rr[y]);
  return TEM_OK;
}

int tem_last_forward_stats(const tem_ctx* c, tem_forward_stats* out) {
  if (!c || !out) return fail(TEM_EINVAL, "tem_last_forward_stats: null pointer");
  *out = c->fstats;
  return TEM_OK;
}

int tem_forward_host(tem_ctx* c, const double* sigma, const double* f, int S, const double* shifts,
                     int K, const double* residues, const int* is_pair, const tem_forward_opts* opts,
                     double* u, int* iters, double* relres) {
  if (!c || !sigma || !f || !shifts || !residues || !is_pair || !opts || !u)
    return fail(TEM_EINVAL, "tem_forward_host: null pointer");
  if (int rc = check_S(S)) return rc;
  if (int rc = check_device(c)) return rc;
  if (int rc = check_index(c, S)) return rc;
  if (K < 1) return fail(TEM_EINVAL, "tem_forward_host: K must be >= 1");
  if (int rc = check_opts(opts)) return rc;
  const size_t ncell = (size_t)c->g.n[0] * c->g.n[1] * c->g.n[2];
  const size_t nsl = (size_t)3 * c->g.Nn;
  const FwdLayout FL = fwd_layout(c, S, K);
  size_t o = 0;
  const size_t o_sig = o;  o = align_up(o + ncell * sizeof(double), 256);
  const size_t o_f = o;    o = align_up(o + nsl * sizeof(double), 256);
  const size_t o_m = o;    o = align_up(o + nsl * sizeof(double), 256);
  const size_t o_x = o;    o = align_up(o + nsl * S * sizeof(double2), 256);
  const size_t o_u = o;    o = align_up(o + (size_t)K * nsl * sizeof(double), 256);
  const size_t o_w = o;    o = align_up(o + FL.total, 256);
  if (c->e2e_bytes < o) {
    if (c->e2e) cudaFree(c->e2e);
    c->e2e = nullptr;
    c->e2e_bytes = 0;
    cudaError_t e = cudaMalloc(&c->e2e, o);
    if (e != cudaSuccess) return fail(TEM_ENOMEM, std::string("tem_forward_host: ") + cudaGetErrorString(e));
    c->e2e_bytes = o;
  }
  char* b = static_cast<char*>(c->e2e);
  cudaStream_t stream = c->cap_stream;  // private non-blocking stream
  TEM_CUDA(cudaMemcpyAsync(b + o_sig, sigma, ncell * sizeof(double), cudaMemcpyHostToDevice, stream));
  TEM_CUDA(cudaMemcpyAsync(b + o_f, f, nsl * sizeof(double), cudaMemcpyHostToDevice, stream));
  if (int rc = tem_edge_mass(c, (const double*)(b + o_sig), (double*)(b + o_m), stream)) return rc;
  const int rc_fwd = forward(c, (const double*)(b + o_m), (const double*)(b + o_f), S, shifts, K, residues, is_pair,
                             *opts, (double*)(b + o_x), (double*)(b + o_u), b + o_w, FL, iters, relres, nullptr,
                             stream);
  if (rc_fwd == TEM_ECUDA || rc_fwd == TEM_EINVAL) return rc_fwd;
  const std::string msg = g_last_error;
  TEM_CUDA(cudaMemcpyAsync(u, b + o_u, (size_t)K * nsl * sizeof(double), cudaMemcpyDeviceToHost, stream));
  TEM_CUDA(cudaStreamSynchronize(stream));
  if (rc_fwd != TEM_OK) return fail(rc_fwd, msg);
  return TEM_OK;
}

}  // extern "C"
