// tem_b200.cu -- B200 (sm_100a) kernels and C ABI of the TEM forward hot path.
//
//   tem_edge_mass       lumped conductivity mass per edge          (§2.2, R1)
//   tem_apply_shifted   y_s = (K + s M) x_s for all shifts, one pass (north star (2))
//   tem_cocg_solve      batched multi-shift Jacobi-COCG               (north star (3))
//   tem_synthesize      u(t_k) = sum_s w_s Re(alpha_ks x_s)          (§3.2 eq:rmj, north star (4))
//   tem_forward_host    all of the above from host buffers
//
// Data layout: see include/tem_b200.h.  A shift block keeps the S shifts of
// one edge contiguous, so a warp's 32 lanes read 32 consecutive complex
// numbers (512 B, fully coalesced) and every per-edge coefficient (mass,
// face weights) is loaded once per edge and broadcast to the S lanes that
// share it: "each coefficient and edge load serves every pole".
//
// COCG iteration = three fused sweeps:
//   k_dir : p = D^-1 r + beta p                               (elementwise)
//   k_ap  : q = A p on the fly, mu = p^T q                     (stencil + reduction)
//   k_upd : q = A p again, x += alpha p, r -= alpha q,
//           z = D^-1 r, rho' = r^T z, ||r||^2                    (stencil + 2 reductions)
// q is recomputed rather than stored (re-reading p from L2/L1 halo is cheaper
// than a 16 B/unknown/shift write + read).  Each reduction ends in the last
// CTA to finish (atomic ticket), which updates the per-shift scalars in
// device memory; no host round trip per iteration.  The iteration loop is
// a CUDA graph of `kChunk` iterations; the host checks the active-shift
// count once per chunk.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/tem_b200.h"
#include "tem_device.cuh"

using tem::Grid;

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
constexpr int kMaxGridMult = 16;    // partials sized for numSMs * kMaxGridMult CTAs
constexpr int kTargetThreads = 256; // CTA size target (tile = floor(256/S) nodes x S shifts)

struct ShiftState {
  double2 s;        // shift
  double2 rho;      // r^T z
  double2 alpha;
  double2 beta;
  double fnorm;     // ||f||_2
  double relres;    // ||r||_2 / ||f||_2
  int active;
  int iters;
  int status;       // 0 running, 1 converged, 2 breakdown
  int pad;
};

struct Control {
  double tol;
  int n_active;
  unsigned int ticket[4];
};

struct SolveArgs {
  Grid g;
  int S;
  int tile_nodes;
  long long ntiles;
  const double* mass;   // [3][Nn]
  const double* f;      // [3][Nn]
  double2* x;           // [3][Nn][S]
  double2* r;
  double2* p;
  ShiftState* st;       // [S]
  Control* ctl;
  double2* part_c;      // [grid][S]
  double* part_r;       // [grid][S]
};

// ------------------------------------------------------------------ helpers

// Per-shift block reduction of one value per thread (thread = node_local*S + s).
// Threads s < S end up with the block sum for shift s (deterministic order).
template <typename T>
__device__ __forceinline__ T block_sum_per_shift(T v, T* buf, int S, int tile_nodes) {
  buf[threadIdx.x] = v;
  __syncthreads();
  T acc{};
  if ((int)threadIdx.x < S) {
    for (int nl = 0; nl < tile_nodes; ++nl) acc += buf[nl * S + threadIdx.x];
  }
  __syncthreads();
  return acc;
}
__device__ __forceinline__ double2& operator+=(double2& a, const double2& b) {
  a.x += b.x;
  a.y += b.y;
  return a;
}

// The last CTA of a launch (atomic ticket) reduces the per-CTA partials per
// shift: warp w handles shifts w, w + nwarps, ...; lanes stride over CTAs;
// fixed shuffle tree.  Returns true in the finalising CTA.
__device__ bool last_block(unsigned int* ticket) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(ticket, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

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

struct ShiftList {
  double2 s[TEM_MAX_SHIFTS];
};

template <int A>
__device__ __forceinline__ void apply_one(const Grid& g, const double* __restrict__ mass,
                                          const double2* __restrict__ x, double2* __restrict__ y,
                                          long long n, int s, int S, double2 sh) {
  const long long slot = (long long)A * g.Nn + n;
  const double m = __ldg(mass + slot);
  double2 out = tem::czero();
  if (m > 0.0) {
    int pos[3];
    tem::node_pos(g, n, pos);
    const tem::EdgeWeights w = tem::edge_weights<A>(g, pos);
    const double2 a0 = __ldg(x + slot * S + s);
    out = tem::curlcurl<A>(g, x, n, s, S, w, a0);
    out = tem::cfma(sh, tem::cscale(m, a0), out);
  }
  y[slot * S + s] = out;
}

__global__ void k_apply(Grid g, int S, int tile_nodes, long long ntiles, ShiftList sl,
                        const double* __restrict__ mass, const double2* __restrict__ x,
                        double2* __restrict__ y) {
  const int s = threadIdx.x % S;
  const int nl = threadIdx.x / S;
  if (nl >= tile_nodes) return;
  const double2 sh = sl.s[s];
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int a = (int)(t % 3);
    const long long n = (t / 3) * tile_nodes + nl;
    if (n >= g.Nn) continue;
    if (a == 0) apply_one<0>(g, mass, x, y, n, s, S, sh);
    else if (a == 1) apply_one<1>(g, mass, x, y, n, s, S, sh);
    else apply_one<2>(g, mass, x, y, n, s, S, sh);
  }
}

// COCG init: x = 0, p = 0, r = f, rho = r^T D^-1 r, ||f||.
__global__ void k_init(SolveArgs A) {
  extern __shared__ unsigned char smem_raw[];
  double* buf = reinterpret_cast<double*>(smem_raw);
  const Grid& g = A.g;
  const int S = A.S;
  const int s = threadIdx.x % S;
  const int nl = threadIdx.x / S;
  const bool lane_ok = nl < A.tile_nodes;
  const double2 sh = A.st[s].s;
  double2 rho = tem::czero();
  double rr = 0.0;
  for (long long t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
    const int a = (int)(t % 3);
    const long long n = (t / 3) * A.tile_nodes + nl;
    if (!lane_ok || n >= g.Nn) continue;
    const long long slot = (long long)a * g.Nn + n;
    const long long e = slot * S + s;
    const double m = __ldg(A.mass + slot);
    double2 r0 = tem::czero();
    if (m > 0.0) {
      r0 = make_double2(__ldg(A.f + slot), 0.0);
      int pos[3];
      tem::node_pos(g, n, pos);
      double kd;
      if (a == 0) kd = tem::edge_weights<0>(g, pos).diag();
      else if (a == 1) kd = tem::edge_weights<1>(g, pos).diag();
      else kd = tem::edge_weights<2>(g, pos).diag();
      const double2 D = make_double2(kd + m * sh.x, m * sh.y);
      rho += tem::cmul(r0, tem::cdiv(r0, D));
      rr += r0.x * r0.x;
    }
    A.x[e] = tem::czero();
    A.p[e] = tem::czero();
    A.r[e] = r0;
  }
  // per-shift block sums -> partials
  double2* bufc = reinterpret_cast<double2*>(smem_raw);
  const double2 bc = block_sum_per_shift<double2>(lane_ok ? rho : tem::czero(), bufc, S, A.tile_nodes);
  const double br = block_sum_per_shift<double>(lane_ok ? rr : 0.0, buf, S, A.tile_nodes);
  if ((int)threadIdx.x < S) {
    A.part_c[blockIdx.x * S + threadIdx.x] = bc;
    A.part_r[blockIdx.x * S + threadIdx.x] = br;
  }
  if (!last_block(&A.ctl->ticket[0])) return;
  // only full warps take part (blockDim may not be a multiple of 32)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int q = warp; warp < nw && q < S; q += nw) {
    double cx = 0, cy = 0, cr = 0;
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      const double2 v = __ldcg(A.part_c + b * S + q);
      cx += v.x;
      cy += v.y;
      cr += __ldcg(A.part_r + b * S + q);
    }
    cx = warp_sum(cx);
    cy = warp_sum(cy);
    cr = warp_sum(cr);
    if (lane == 0) {
      ShiftState& st = A.st[q];
      st.rho = make_double2(cx, cy);
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
  if (threadIdx.x == 0) {
    int na = 0;
    for (int q = 0; q < S; ++q) na += A.st[q].active;
    A.ctl->n_active = na;
    A.ctl->ticket[0] = 0;
  }
}

// p = D^-1 r + beta p  (elementwise; active shifts only)
template <int AX>
__device__ __forceinline__ void dir_one(const SolveArgs& A, long long n, int s, double2 sh, double2 beta) {
  const Grid& g = A.g;
  const long long slot = (long long)AX * g.Nn + n;
  const double m = __ldg(A.mass + slot);
  if (m <= 0.0) return;
  int pos[3];
  tem::node_pos(g, n, pos);
  const double kd = tem::edge_weights<AX>(g, pos).diag();
  const double2 D = make_double2(kd + m * sh.x, m * sh.y);
  const long long e = slot * A.S + s;
  const double2 z = tem::cdiv(A.r[e], D);
  A.p[e] = tem::cfma(beta, A.p[e], z);
}

__global__ void k_dir(SolveArgs A) {
  if (A.ctl->n_active == 0) return;
  const int S = A.S;
  const int s = threadIdx.x % S;
  const int nl = threadIdx.x / S;
  if (nl >= A.tile_nodes) return;
  const ShiftState st = A.st[s];
  if (!st.active) return;
  for (long long t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
    const int a = (int)(t % 3);
    const long long n = (t / 3) * A.tile_nodes + nl;
    if (n >= A.g.Nn) continue;
    if (a == 0) dir_one<0>(A, n, s, st.s, st.beta);
    else if (a == 1) dir_one<1>(A, n, s, st.s, st.beta);
    else dir_one<2>(A, n, s, st.s, st.beta);
  }
}

// mu partial: p^T (A p)
template <int AX>
__device__ __forceinline__ double2 ap_one(const SolveArgs& A, long long n, int s, double2 sh) {
  const Grid& g = A.g;
  const long long slot = (long long)AX * g.Nn + n;
  const double m = __ldg(A.mass + slot);
  if (m <= 0.0) return tem::czero();
  int pos[3];
  tem::node_pos(g, n, pos);
  const tem::EdgeWeights w = tem::edge_weights<AX>(g, pos);
  const double2 p0 = __ldg(A.p + slot * A.S + s);
  double2 q = tem::curlcurl<AX>(g, A.p, n, s, A.S, w, p0);
  q = tem::cfma(sh, tem::cscale(m, p0), q);
  return tem::cmul(p0, q);
}

__global__ void k_ap(SolveArgs A) {
  extern __shared__ unsigned char smem_raw[];
  if (A.ctl->n_active == 0) return;
  const int S = A.S;
  const int s = threadIdx.x % S;
  const int nl = threadIdx.x / S;
  const bool lane_ok = nl < A.tile_nodes;
  const ShiftState st = A.st[s];
  double2 mu = tem::czero();
  if (lane_ok && st.active) {
    for (long long t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
      const int a = (int)(t % 3);
      const long long n = (t / 3) * A.tile_nodes + nl;
      if (n >= A.g.Nn) continue;
      if (a == 0) mu += ap_one<0>(A, n, s, st.s);
      else if (a == 1) mu += ap_one<1>(A, n, s, st.s);
      else mu += ap_one<2>(A, n, s, st.s);
    }
  }
  double2* bufc = reinterpret_cast<double2*>(smem_raw);
  const double2 bc = block_sum_per_shift<double2>(mu, bufc, S, A.tile_nodes);
  if ((int)threadIdx.x < S) A.part_c[blockIdx.x * S + threadIdx.x] = bc;
  if (!last_block(&A.ctl->ticket[1])) return;
  // only full warps take part (blockDim may not be a multiple of 32)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int q = warp; warp < nw && q < S; q += nw) {
    if (!A.st[q].active) continue;
    double cx = 0, cy = 0;
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      const double2 v = __ldcg(A.part_c + b * S + q);
      cx += v.x;
      cy += v.y;
    }
    cx = warp_sum(cx);
    cy = warp_sum(cy);
    if (lane == 0) {
      ShiftState& sq = A.st[q];
      const double2 mu_q = make_double2(cx, cy);
      if (mu_q.x == 0.0 && mu_q.y == 0.0) {
        sq.status = 2;  // breakdown
        sq.active = 0;
        sq.alpha = tem::czero();
      } else {
        sq.alpha = tem::cdiv(sq.rho, mu_q);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int na = 0;
    for (int q = 0; q < S; ++q) na += A.st[q].active;
    A.ctl->n_active = na;
    A.ctl->ticket[1] = 0;
  }
}

// x += alpha p ; r -= alpha A p ; rho' = r^T D^-1 r ; rr = ||r||^2
template <int AX>
__device__ __forceinline__ void upd_one(const SolveArgs& A, long long n, int s, double2 sh,
                                        double2 alpha, double2& rho, double& rr) {
  const Grid& g = A.g;
  const long long slot = (long long)AX * g.Nn + n;
  const double m = __ldg(A.mass + slot);
  if (m <= 0.0) return;
  int pos[3];
  tem::node_pos(g, n, pos);
  const tem::EdgeWeights w = tem::edge_weights<AX>(g, pos);
  const long long e = slot * A.S + s;
  const double2 p0 = __ldg(A.p + e);
  double2 q = tem::curlcurl<AX>(g, A.p, n, s, A.S, w, p0);
  q = tem::cfma(sh, tem::cscale(m, p0), q);
  A.x[e] = tem::cfma(alpha, p0, A.x[e]);
  const double2 r = tem::cfma(make_double2(-alpha.x, -alpha.y), q, A.r[e]);
  A.r[e] = r;
  const double2 D = make_double2(w.diag() + m * sh.x, m * sh.y);
  rho += tem::cmul(r, tem::cdiv(r, D));
  rr += r.x * r.x + r.y * r.y;
}

__global__ void k_upd(SolveArgs A) {
  extern __shared__ unsigned char smem_raw[];
  if (A.ctl->n_active == 0) return;
  const int S = A.S;
  const int s = threadIdx.x % S;
  const int nl = threadIdx.x / S;
  const bool lane_ok = nl < A.tile_nodes;
  const ShiftState st = A.st[s];
  double2 rho = tem::czero();
  double rr = 0.0;
  if (lane_ok && st.active) {
    for (long long t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
      const int a = (int)(t % 3);
      const long long n = (t / 3) * A.tile_nodes + nl;
      if (n >= A.g.Nn) continue;
      if (a == 0) upd_one<0>(A, n, s, st.s, st.alpha, rho, rr);
      else if (a == 1) upd_one<1>(A, n, s, st.s, st.alpha, rho, rr);
      else upd_one<2>(A, n, s, st.s, st.alpha, rho, rr);
    }
  }
  double2* bufc = reinterpret_cast<double2*>(smem_raw);
  double* bufr = reinterpret_cast<double*>(smem_raw);
  const double2 bc = block_sum_per_shift<double2>(rho, bufc, S, A.tile_nodes);
  const double br = block_sum_per_shift<double>(rr, bufr, S, A.tile_nodes);
  if ((int)threadIdx.x < S) {
    A.part_c[blockIdx.x * S + threadIdx.x] = bc;
    A.part_r[blockIdx.x * S + threadIdx.x] = br;
  }
  if (!last_block(&A.ctl->ticket[2])) return;
  // only full warps take part (blockDim may not be a multiple of 32)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int q = warp; warp < nw && q < S; q += nw) {
    if (!A.st[q].active) continue;
    double cx = 0, cy = 0, cr = 0;
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      const double2 v = __ldcg(A.part_c + b * S + q);
      cx += v.x;
      cy += v.y;
      cr += __ldcg(A.part_r + b * S + q);
    }
    cx = warp_sum(cx);
    cy = warp_sum(cy);
    cr = warp_sum(cr);
    if (lane == 0) {
      ShiftState& sq = A.st[q];
      const double2 rho_new = make_double2(cx, cy);
      sq.iters += 1;
      sq.relres = sqrt(cr) / sq.fnorm;
      if (sq.relres <= A.ctl->tol) {
        sq.active = 0;
        sq.status = 1;
      } else if (sq.rho.x == 0.0 && sq.rho.y == 0.0) {
        sq.active = 0;
        sq.status = 2;
      } else {
        sq.beta = tem::cdiv(rho_new, sq.rho);
        sq.rho = rho_new;
        if (rho_new.x == 0.0 && rho_new.y == 0.0) {
          sq.active = 0;
          sq.status = 2;
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int na = 0;
    for (int q = 0; q < S; ++q) na += A.st[q].active;
    A.ctl->n_active = na;
    A.ctl->ticket[2] = 0;
  }
}

// u[k][slot] = sum_s w_s Re(res[k][s] x[slot][s]); 0 on non-free slots.
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
      xv[s] = (live && s < S) ? __ldg(x + slot * S + s) : tem::czero();
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

}  // namespace

// ====================================================================== C ABI

struct tem_ctx {
  Grid g{};
  int device = 0;
  int num_sms = 0;
  double* dev_h = nullptr;          // ih[3] and hdm[3] packed
  cudaStream_t cap_stream = nullptr;
  int* pinned_active = nullptr;
  // cached graph
  cudaGraphExec_t graph = nullptr;
  SolveArgs graph_args{};
  int graph_grid = 0, graph_block = 0;
  size_t graph_smem = 0;
  // scratch
  void* scratch = nullptr;          // residues etc.
  size_t scratch_bytes = 0;
  // e2e workspace
  void* e2e = nullptr;
  size_t e2e_bytes = 0;
  // stats of the last solve
  tem_solve_stats stats{};
};

static int tile_nodes_for(int S) { return std::max(1, kTargetThreads / S); }

static int check_S(int S) {
  if (S < 1 || S > TEM_MAX_SHIFTS)
    return fail(TEM_EINVAL, "S must be in [1, " + std::to_string(TEM_MAX_SHIFTS) + "]");
  return TEM_OK;
}

extern "C" {

const char* tem_version(void) { return "tem_b200 0.1 sm_100a"; }
const char* tem_last_error(void) { return g_last_error.c_str(); }

int tem_create(int nx, int ny, int nz, const double* hx, const double* hy, const double* hz,
               tem_ctx** out) {
  if (!out || !hx || !hy || !hz) return fail(TEM_EINVAL, "tem_create: null pointer");
  *out = nullptr;
  if (nx < 2 || ny < 2 || nz < 2) return fail(TEM_EINVAL, "tem_create: need nx, ny, nz >= 2");
  const int n[3] = {nx, ny, nz};
  const double* h[3] = {hx, hy, hz};
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < n[a]; ++i)
      if (!(h[a][i] > 0.0)) return fail(TEM_EINVAL, "tem_create: cell widths must be > 0");
  tem_ctx* c = new tem_ctx();
  cudaGetDevice(&c->device);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
  for (int a = 0; a < 3; ++a) c->g.n[a] = n[a];
  c->g.st[0] = 1;
  c->g.st[1] = nx + 1;
  c->g.st[2] = (long long)(nx + 1) * (ny + 1);
  c->g.Nn = (long long)(nx + 1) * (ny + 1) * (nz + 1);
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
  *out = c;
  return TEM_OK;
}

void tem_destroy(tem_ctx* c) {
  if (!c) return;
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->dev_h) cudaFree(c->dev_h);
  if (c->scratch) cudaFree(c->scratch);
  if (c->e2e) cudaFree(c->e2e);
  if (c->pinned_active) cudaFreeHost(c->pinned_active);
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
  ShiftList sl{};
  for (int s = 0; s < S; ++s) sl.s[s] = make_double2(shifts[2 * s], shifts[2 * s + 1]);
  const int tn = tile_nodes_for(S);
  const long long ntiles = 3 * ((c->g.Nn + tn - 1) / tn);
  const int block = tn * S;
  const int grid = (int)std::min<long long>(ntiles, (long long)c->num_sms * 8);
  // zero y first so slots never visited by a thread (tile padding) are 0
  TEM_CUDA(cudaMemsetAsync(y, 0, (size_t)3 * c->g.Nn * S * sizeof(double2), (cudaStream_t)stream));
  k_apply<<<grid, block, 0, (cudaStream_t)stream>>>(c->g, S, tn, ntiles, sl, mass,
                                                    reinterpret_cast<const double2*>(x),
                                                    reinterpret_cast<double2*>(y));
  TEM_CUDA(cudaGetLastError());
  return TEM_OK;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct WorkLayout {
  size_t r, p, st, ctl, part_c, part_r, total;
};

static WorkLayout work_layout(const tem_ctx* c, int S) {
  WorkLayout L{};
  const size_t vec = (size_t)3 * c->g.Nn * S * sizeof(double2);
  const size_t maxgrid = (size_t)c->num_sms * kMaxGridMult;
  size_t o = 0;
  L.r = o;      o = align_up(o + vec, 256);
  L.p = o;      o = align_up(o + vec, 256);
  L.st = o;     o = align_up(o + sizeof(ShiftState) * TEM_MAX_SHIFTS, 256);
  L.ctl = o;    o = align_up(o + sizeof(Control), 256);
  L.part_c = o; o = align_up(o + maxgrid * S * sizeof(double2), 256);
  L.part_r = o; o = align_up(o + maxgrid * S * sizeof(double), 256);
  L.total = o;
  return L;
}

size_t tem_cocg_workspace_bytes(const tem_ctx* c, int S) {
  if (!c || S < 1 || S > TEM_MAX_SHIFTS) return 0;
  return work_layout(c, S).total;
}

static int solve_grid(const tem_ctx* c, int block, size_t smem, const void* kern) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
  per_sm = std::max(1, std::min(per_sm, kMaxGridMult));
  return c->num_sms * per_sm;
}

int tem_cocg_solve(tem_ctx* c, const double* mass, const double* f, int S, const double* shifts,
                   double tol, int maxit, double* x, void* work, size_t work_bytes, int* iters,
                   double* relres, void* stream_) {
  if (!c || !mass || !f || !shifts || !x || !work) return fail(TEM_EINVAL, "tem_cocg_solve: null pointer");
  if (int rc = check_S(S)) return rc;
  if (!(tol > 0.0) || maxit < 1) return fail(TEM_EINVAL, "tem_cocg_solve: need tol > 0, maxit >= 1");
  const WorkLayout L = work_layout(c, S);
  if (work_bytes < L.total) return fail(TEM_EINVAL, "tem_cocg_solve: workspace too small");
  cudaStream_t stream = (cudaStream_t)stream_;
  char* w = static_cast<char*>(work);

  SolveArgs A{};
  A.g = c->g;
  A.S = S;
  A.tile_nodes = tile_nodes_for(S);
  A.ntiles = 3 * ((c->g.Nn + A.tile_nodes - 1) / A.tile_nodes);
  A.mass = mass;
  A.f = f;
  A.x = reinterpret_cast<double2*>(x);
  A.r = reinterpret_cast<double2*>(w + L.r);
  A.p = reinterpret_cast<double2*>(w + L.p);
  A.st = reinterpret_cast<ShiftState*>(w + L.st);
  A.ctl = reinterpret_cast<Control*>(w + L.ctl);
  A.part_c = reinterpret_cast<double2*>(w + L.part_c);
  A.part_r = reinterpret_cast<double*>(w + L.part_r);
  const int block = A.tile_nodes * S;
  const size_t smem = (size_t)block * sizeof(double2);
  int grid = solve_grid(c, block, smem, (const void*)k_upd);
  grid = (int)std::min<long long>(grid, A.ntiles);

  // per-shift state + control (host -> device, small)
  std::vector<ShiftState> st(S);
  for (int s = 0; s < S; ++s) {
    memset(&st[s], 0, sizeof(ShiftState));
    st[s].s = make_double2(shifts[2 * s], shifts[2 * s + 1]);
  }
  Control ctl{};
  ctl.tol = tol;
  TEM_CUDA(cudaMemcpyAsync(A.st, st.data(), sizeof(ShiftState) * S, cudaMemcpyHostToDevice, stream));
  TEM_CUDA(cudaMemcpyAsync(A.ctl, &ctl, sizeof(Control), cudaMemcpyHostToDevice, stream));

  cudaEvent_t ev0, ev1;
  TEM_CUDA(cudaEventCreate(&ev0));
  TEM_CUDA(cudaEventCreate(&ev1));
  TEM_CUDA(cudaEventRecord(ev0, stream));
  k_init<<<grid, block, smem, stream>>>(A);
  TEM_CUDA(cudaGetLastError());
  long long launches = 1;

  // (re)build the cached graph of kChunk iterations if the arguments changed
  const SolveArgs& G = c->graph_args;
  const bool same = c->graph && c->graph_grid == grid && c->graph_block == block &&
                    G.S == A.S && G.mass == A.mass && G.f == A.f && G.x == A.x &&
                    G.r == A.r && G.p == A.p && G.st == A.st && G.ctl == A.ctl &&
                    G.part_c == A.part_c && G.part_r == A.part_r && G.g.Nn == A.g.Nn &&
                    G.g.ih[0] == A.g.ih[0];
  if (!same) {
    if (c->graph) {
      cudaGraphExecDestroy(c->graph);
      c->graph = nullptr;
    }
    cudaGraph_t gr;
    TEM_CUDA(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
    for (int it = 0; it < kChunk; ++it) {
      k_dir<<<grid, block, 0, c->cap_stream>>>(A);
      k_ap<<<grid, block, smem, c->cap_stream>>>(A);
      k_upd<<<grid, block, smem, c->cap_stream>>>(A);
    }
    TEM_CUDA(cudaStreamEndCapture(c->cap_stream, &gr));
    cudaError_t e = cudaGraphInstantiate(&c->graph, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) return fail(TEM_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    c->graph_args = A;
    c->graph_grid = grid;
    c->graph_block = block;
  }
  int done = 0;
  int n_active = S;
  while (done < maxit) {
    const int chunk = std::min(kChunk, maxit - done);
    if (chunk == kChunk) {
      TEM_CUDA(cudaGraphLaunch(c->graph, stream));
    } else {
      for (int it = 0; it < chunk; ++it) {
        k_dir<<<grid, block, 0, stream>>>(A);
        k_ap<<<grid, block, smem, stream>>>(A);
        k_upd<<<grid, block, smem, stream>>>(A);
      }
      TEM_CUDA(cudaGetLastError());
    }
    launches += 3LL * chunk;
    done += chunk;
    TEM_CUDA(cudaMemcpyAsync(c->pinned_active, &A.ctl->n_active, sizeof(int), cudaMemcpyDeviceToHost, stream));
    TEM_CUDA(cudaStreamSynchronize(stream));
    n_active = *c->pinned_active;
    if (n_active == 0) break;
  }
  TEM_CUDA(cudaEventRecord(ev1, stream));
  TEM_CUDA(cudaMemcpyAsync(st.data(), A.st, sizeof(ShiftState) * S, cudaMemcpyDeviceToHost, stream));
  TEM_CUDA(cudaStreamSynchronize(stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);

  long long shift_iters = 0;
  int max_it = 0;
  int status = TEM_OK;
  for (int s = 0; s < S; ++s) {
    if (iters) iters[s] = st[s].iters;
    if (relres) relres[s] = st[s].relres;
    shift_iters += st[s].iters;
    max_it = std::max(max_it, st[s].iters);
    if (st[s].status == 2) status = TEM_EBREAKDOWN;
    else if (st[s].status != 1 && status == TEM_OK) status = TEM_ENOCONV;
  }
  c->stats.loop_ms = ms;
  c->stats.kernel_launches = launches;
  c->stats.shift_iterations = shift_iters;
  c->stats.iterations = max_it;
  c->stats.grid = grid;
  c->stats.block = block;
  if (status == TEM_EBREAKDOWN) return fail(status, "tem_cocg_solve: COCG breakdown");
  if (status == TEM_ENOCONV) return fail(status, "tem_cocg_solve: not converged within maxit");
  return TEM_OK;
}

int tem_last_solve_stats(const tem_ctx* c, tem_solve_stats* out) {
  if (!c || !out) return fail(TEM_EINVAL, "tem_last_solve_stats: null pointer");
  *out = c->stats;
  return TEM_OK;
}

static int ensure_scratch(tem_ctx* c, size_t bytes) {
  if (c->scratch_bytes >= bytes) return TEM_OK;
  if (c->scratch) cudaFree(c->scratch);
  c->scratch = nullptr;
  c->scratch_bytes = 0;
  TEM_CUDA(cudaMalloc(&c->scratch, bytes));
  c->scratch_bytes = bytes;
  return TEM_OK;
}

int tem_synthesize(tem_ctx* c, int S, int K, const double* residues, const int* is_pair,
                   const double* x, double* u, void* stream_) {
  if (!c || !residues || !is_pair || !x || !u) return fail(TEM_EINVAL, "tem_synthesize: null pointer");
  if (int rc = check_S(S)) return rc;
  if (K < 1) return fail(TEM_EINVAL, "tem_synthesize: K must be >= 1");
  const size_t res_bytes = (size_t)K * S * sizeof(double2);
  const size_t smem = res_bytes;
  if (smem > 200 * 1024) return fail(TEM_EINVAL, "tem_synthesize: K*S too large for shared memory");
  // scratch: residues [K][S] complex, then weights [S]
  if (int rc = ensure_scratch(c, res_bytes + TEM_MAX_SHIFTS * sizeof(double))) return rc;
  cudaStream_t stream = (cudaStream_t)stream_;
  std::vector<double> wts(S);
  for (int s = 0; s < S; ++s) wts[s] = is_pair[s] ? 2.0 : 1.0;
  char* sc = static_cast<char*>(c->scratch);
  TEM_CUDA(cudaMemcpyAsync(sc, residues, res_bytes, cudaMemcpyHostToDevice, stream));
  TEM_CUDA(cudaMemcpyAsync(sc + res_bytes, wts.data(), S * sizeof(double), cudaMemcpyHostToDevice, stream));
  const long long nslots = 3 * c->g.Nn;
  const int block = 128;
  const int grid = (int)std::min<long long>((nslots + block - 1) / block, (long long)c->num_sms * 16);
  const double2* res_d = reinterpret_cast<const double2*>(sc);
  const double* w_d = reinterpret_cast<const double*>(sc + res_bytes);
  const double2* xd = reinterpret_cast<const double2*>(x);
#define TEM_SYNTH(SM)                                                                      \
  do {                                                                                     \
    if (smem > 48 * 1024)                                                                  \
      TEM_CUDA(cudaFuncSetAttribute(k_synth<SM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_synth<SM><<<grid, block, smem, stream>>>(c->g, S, K, res_d, w_d, xd, u);             \
  } while (0)
  if (S <= 8) TEM_SYNTH(8);
  else if (S <= 16) TEM_SYNTH(16);
  else if (S <= 24) TEM_SYNTH(24);
  else TEM_SYNTH(32);
#undef TEM_SYNTH
  TEM_CUDA(cudaGetLastError());
  // synchronise so the pageable host buffers above are not reused early
  TEM_CUDA(cudaStreamSynchronize(stream));
  return TEM_OK;
}

int tem_forward_host(tem_ctx* c, const double* sigma, const double* f, int S, const double* shifts,
                     int K, const double* residues, const int* is_pair, double tol, int maxit,
                     double* u, int* iters, double* relres) {
  if (!c || !sigma || !f || !shifts || !residues || !is_pair || !u)
    return fail(TEM_EINVAL, "tem_forward_host: null pointer");
  if (int rc = check_S(S)) return rc;
  if (K < 1) return fail(TEM_EINVAL, "tem_forward_host: K must be >= 1");
  const size_t ncell = (size_t)c->g.n[0] * c->g.n[1] * c->g.n[2];
  const size_t nsl = (size_t)3 * c->g.Nn;
  size_t o = 0;
  const size_t o_sig = o;  o = align_up(o + ncell * sizeof(double), 256);
  const size_t o_f = o;    o = align_up(o + nsl * sizeof(double), 256);
  const size_t o_m = o;    o = align_up(o + nsl * sizeof(double), 256);
  const size_t o_x = o;    o = align_up(o + nsl * S * sizeof(double2), 256);
  const size_t o_u = o;    o = align_up(o + (size_t)K * nsl * sizeof(double), 256);
  const size_t o_w = o;
  const size_t wbytes = tem_cocg_workspace_bytes(c, S);
  o = align_up(o + wbytes, 256);
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
  const int rc_solve = tem_cocg_solve(c, (const double*)(b + o_m), (const double*)(b + o_f), S, shifts,
                                      tol, maxit, (double*)(b + o_x), b + o_w, wbytes, iters, relres,
                                      stream);
  if (rc_solve == TEM_ECUDA || rc_solve == TEM_EINVAL) return rc_solve;
  const std::string solve_msg = g_last_error;
  if (int rc = tem_synthesize(c, S, K, residues, is_pair, (const double*)(b + o_x), (double*)(b + o_u), stream))
    return rc;
  TEM_CUDA(cudaMemcpyAsync(u, b + o_u, (size_t)K * nsl * sizeof(double), cudaMemcpyDeviceToHost, stream));
  TEM_CUDA(cudaStreamSynchronize(stream));
  if (rc_solve != TEM_OK) return fail(rc_solve, solve_msg);
  return TEM_OK;
}

}  // extern "C"
