// tem_sweep.cuh -- the 2.5D z-marching curl-curl sweep (sm_100a).
//
// One CTA owns a TX x TY tile of nodes in the x-y plane, ONE shift s and a
// range of node planes k; it marches upward in k.  The halo-extended plane
// tiles of the swept vector v (x,y components on planes k-1, k, k+1 and the
// z component on layers k-1, k) live in a shared-memory ring, so every
// element is fetched from L2/HBM once per sweep (plus the 1-node halo) and
// the 13-point gather of
//   (K v)_a(m) = W_d(m) C_d(m) - W_d(m-e_b) C_d(m-e_b) - W_b(m) C_b(m) + W_b(m-e_d) C_b(m-e_d)
// (tem_device.cuh; §2.2, reading R1) reads shared memory only.
// The next plane set is loaded into registers one step ahead (software
// pipelining) so its HBM latency overlaps the current step's arithmetic.
//
// MODE 0  apply : y = (K + s M) v                                  (tem_apply_shifted)
// MODE 1  dirap : v = p_new = z + beta p_old formed on load; writes p_new;
//                 mu = p_new^T (K + s M) p_new                      (COCG sweep 1)
// MODE 2  upd   : v = p; x += alpha p; z -= alpha D^-1 (K + s M) p;
//                 rho = (D z)^T z, ||D z||^2                        (COCG sweep 2)
// z = D^-1 r is stored instead of r (reading "z-form"): r = D z
// is recovered where needed, so a COCG iteration streams x, z, p_old, p_new
// at the 128 B / unknown / shift minimum of a two-reduction COCG.
#pragma once
#include "tem_device.cuh"

namespace tem {

constexpr int TX = 32;                    // tile nodes along x (one warp row)
constexpr int TY = 8;                     // tile nodes along y
constexpr int NT = TX * TY;               // threads per CTA
constexpr int HX = TX + 2, HY = TY + 2;   // halo-extended tile
constexpr int H = HX * HY;                // nodes per plane tile
constexpr int LOADS = (3 * H + NT - 1) / NT;  // plane-set elements per thread per step
constexpr size_t kSweepSmem = (size_t)11 * H * sizeof(double2);  // dynamic shared memory

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

struct SweepArgs {
  Grid g;
  int S;
  int ntx, nty, nzc, kchunk;   // tiles along x, y; z-chunks and their length
  const double* mass;          // [3][Nn]
  const double2* v;            // swept vector [S][3][Nn] (MODE 0: x; MODE 1: p_old; MODE 2: p)
  const double2* zin;          // MODE 1: z
  double2* out;                // MODE 0: y; MODE 1: p_new
  double2* x;                  // MODE 2
  double2* z;                  // MODE 2 (in/out)
  ShiftState* st;              // [S]
  Control* ctl;
  double2* part_c;             // [gridDim]
  double* part_r;              // [gridDim]
  double2 shifts[32];          // MODE 0 only
};

__device__ __forceinline__ bool free_x(const Grid& g, int i, int j, int k) {
  return i < g.n[0] && j >= 1 && j <= g.n[1] - 1 && k >= 1 && k <= g.n[2] - 1;
}
__device__ __forceinline__ bool free_y(const Grid& g, int i, int j, int k) {
  return i >= 1 && i <= g.n[0] - 1 && j < g.n[1] && k >= 1 && k <= g.n[2] - 1;
}
__device__ __forceinline__ bool free_z(const Grid& g, int i, int j, int k) {
  return i >= 1 && i <= g.n[0] - 1 && j >= 1 && j <= g.n[1] - 1 && k < g.n[2];
}

// Block-wide sum of a complex and a real value (all NTH threads participate);
// the result is valid in thread 0.  Fixed order -> deterministic.
template <int NTH>
__device__ __forceinline__ void block_sum_n(double2& c, double& r, double* red) {
  for (int o = 16; o > 0; o >>= 1) {
    c.x += __shfl_down_sync(0xffffffffu, c.x, o);
    c.y += __shfl_down_sync(0xffffffffu, c.y, o);
    r += __shfl_down_sync(0xffffffffu, r, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    red[3 * w] = c.x;
    red[3 * w + 1] = c.y;
    red[3 * w + 2] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0, d = 0;
    for (int q = 0; q < NTH / 32; ++q) {
      a += red[3 * q];
      b += red[3 * q + 1];
      d += red[3 * q + 2];
    }
    c = make_double2(a, b);
    r = d;
  }
}

// The last CTA of a launch (atomic ticket) returns true.
__device__ __forceinline__ bool last_block(unsigned int* ticket) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(NT, 3) k_sweep(SweepArgs A) {
  // ring: X, Y planes (4 slots each: k-1, k, k+1 and the one being filled), Z layers (3 slots)
  extern __shared__ double2 smem_ring[];
  double2 (*sX)[H] = reinterpret_cast<double2 (*)[H]>(smem_ring);
  double2 (*sY)[H] = reinterpret_cast<double2 (*)[H]>(smem_ring + 4 * H);
  double2 (*sZ)[H] = reinterpret_cast<double2 (*)[H]>(smem_ring + 8 * H);
  __shared__ double red[3 * NT / 32];

  const Grid& g = A.g;
  const int S = A.S;
  // block -> (z-chunk, xy tile, shift), shift fastest so that the S CTAs of a
  // tile run together and share its coefficients through L2
  const int s = blockIdx.x % S;
  const int xy = (blockIdx.x / S) % (A.ntx * A.nty);
  const int zc = blockIdx.x / (S * A.ntx * A.nty);
  const int tx0 = (xy % A.ntx) * TX, ty0 = (xy / A.ntx) * TY;
  const int kb = zc * A.kchunk;
  const int ke = min(kb + A.kchunk, g.n[2]);

  double2 sh, beta, alpha;
  bool live;
  if (MODE == 0) {
    sh = A.shifts[s];
    live = true;
  } else {
    const ShiftState& st = A.st[s];
    sh = st.s;
    beta = st.beta;
    alpha = st.alpha;
    live = st.active != 0;
  }

  double2 acc_c = czero();
  double acc_r = 0.0;
  const int nx1 = g.n[0] + 1, ny1 = g.n[1] + 1, nz = g.n[2];
  const long long vs = (long long)s * 3 * g.Nn;   // shift offset
  const int tid = threadIdx.x;

  if (live) {
    // per-thread constants of the column (i, j)
    const int i = tx0 + (tid % TX), j = ty0 + (tid / TX);
    const int li = (tid % TX) + 1, lj = (tid / TX) + 1;
    const int c0 = lj * HX + li;          // centre in a plane tile
    const bool in_ij = i < g.n[0] && j < g.n[1];
    const double ihx = in_ij ? __ldg(g.ih[0] + i) : 0.0;
    const double ihxm = (in_ij && i >= 1) ? __ldg(g.ih[0] + i - 1) : 0.0;
    const double ihy = in_ij ? __ldg(g.ih[1] + j) : 0.0;
    const double ihym = (in_ij && j >= 1) ? __ldg(g.ih[1] + j - 1) : 0.0;
    const double hdx = in_ij ? __ldg(g.hdm[0] + i) : 0.0;
    const double hdy = in_ij ? __ldg(g.hdm[1] + j) : 0.0;

    // plane-set loader: element e of {X(kx), Y(kx), Z(kz)} tiles
    auto load_elem = [&](int e, int kx, int kz, const double2* __restrict__ src) -> double2 {
      const int comp = e / H;
      const int r = e - comp * H;
      const int ii = tx0 - 1 + (r % HX), jj = ty0 - 1 + (r / HX);
      const int kk = comp == 2 ? kz : kx;
      if (ii < 0 || ii >= nx1 || jj < 0 || jj >= ny1 || kk < 0 || kk > nz) return czero();
      return __ldg(src + vs + (long long)comp * g.Nn + ((long long)kk * ny1 + jj) * nx1 + ii);
    };
    auto store_elem = [&](int e, int slot_xy, int slot_z, double2 v) {
      const int comp = e / H;
      const int r = e - comp * H;
      if (comp == 0) sX[slot_xy][r] = v;
      else if (comp == 1) sY[slot_xy][r] = v;
      else sZ[slot_z][r] = v;
    };
    auto fetch = [&](int e, int kx, int kz) -> double2 {
      // MODE 1 forms p_new = z + beta p_old on load
      if (MODE == 1) {
        const double2 zv = load_elem(e, kx, kz, A.zin);
        const double2 pv = load_elem(e, kx, kz, A.v);
        return cfma(beta, pv, zv);
      }
      return load_elem(e, kx, kz, A.v);
    };

    // prologue: X,Y planes kb-1, kb ; Z layer kb-1 ; then X,Y kb+1 and Z kb
    for (int e = tid; e < 3 * H; e += NT) store_elem(e, (kb + 3) & 3, (kb + 2) % 3, fetch(e, kb - 1, kb - 1));
    for (int e = tid; e < 2 * H; e += NT) store_elem(e, kb & 3, 0, fetch(e, kb, kb));
    for (int e = tid; e < 3 * H; e += NT) store_elem(e, (kb + 1) & 3, kb % 3, fetch(e, kb + 1, kb));
    __syncthreads();

    for (int k = kb; k < ke; ++k) {
      // 1. issue the loads of the next plane set (X,Y plane k+2, Z layer k+1)
      double2 nxt[LOADS];
#pragma unroll
      for (int q = 0; q < LOADS; ++q) {
        const int e = tid + q * NT;
        nxt[q] = e < 3 * H ? fetch(e, k + 2, k + 1) : czero();
      }
      // 2. compute the three edges of node (i, j, k) from shared memory
      const int xm = (k + 3) & 3, x0 = k & 3, xp = (k + 1) & 3;
      const int zm = (k + 2) % 3, z0 = k % 3;
      const double ihz = __ldg(g.ih[2] + k);
      const double ihzm = k >= 1 ? __ldg(g.ih[2] + k - 1) : 0.0;
      const double hdz = __ldg(g.hdm[2] + k);
      const long long node = ((long long)k * ny1 + j) * nx1 + i;
#define X_(dk, di, dj) sX[dk][c0 + (dj) * HX + (di)]
#define Y_(dk, di, dj) sY[dk][c0 + (dj) * HX + (di)]
#define Z_(dk, di, dj) sZ[dk][c0 + (dj) * HX + (di)]
      double2 q3[3], p3[3];
      double m3[3], kd3[3];
      bool f3[3];
      f3[0] = in_ij && free_x(g, i, j, k);
      f3[1] = in_ij && free_y(g, i, j, k);
      f3[2] = in_ij && free_z(g, i, j, k);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        q3[c] = czero();
        p3[c] = czero();
        m3[c] = 0.0;
        kd3[c] = 0.0;
      }
      if (f3[0]) {  // x-edge: A=x, B=y, D=z
        const double2 a0 = X_(x0, 0, 0);
        const double2 cD0 = csub(cadd(a0, Y_(x0, 1, 0)), cadd(X_(x0, 0, 1), Y_(x0, 0, 0)));
        const double2 cD1 = csub(cadd(X_(x0, 0, -1), Y_(x0, 1, -1)), cadd(a0, Y_(x0, 0, -1)));
        const double2 cB0 = csub(cadd(Z_(z0, 0, 0), X_(xp, 0, 0)), cadd(Z_(z0, 1, 0), a0));
        const double2 cB1 = csub(cadd(Z_(zm, 0, 0), a0), cadd(Z_(zm, 1, 0), X_(xm, 0, 0)));
        const double wD0 = hdz * ihx * ihy, wD1 = hdz * ihx * ihym;
        const double wB0 = hdy * ihx * ihz, wB1 = hdy * ihx * ihzm;
        q3[0] = make_double2(wD0 * cD0.x - wD1 * cD1.x - wB0 * cB0.x + wB1 * cB1.x,
                             wD0 * cD0.y - wD1 * cD1.y - wB0 * cB0.y + wB1 * cB1.y);
        kd3[0] = wD0 + wD1 + wB0 + wB1;
        p3[0] = a0;
      }
      if (f3[1]) {  // y-edge: A=y, B=z, D=x
        const double2 a0 = Y_(x0, 0, 0);
        const double2 cD0 = csub(cadd(a0, Z_(z0, 0, 1)), cadd(Y_(xp, 0, 0), Z_(z0, 0, 0)));
        const double2 cD1 = csub(cadd(Y_(xm, 0, 0), Z_(zm, 0, 1)), cadd(a0, Z_(zm, 0, 0)));
        const double2 cB0 = csub(cadd(X_(x0, 0, 0), Y_(x0, 1, 0)), cadd(X_(x0, 0, 1), a0));
        const double2 cB1 = csub(cadd(X_(x0, -1, 0), a0), cadd(X_(x0, -1, 1), Y_(x0, -1, 0)));
        const double wD0 = hdx * ihy * ihz, wD1 = hdx * ihy * ihzm;
        const double wB0 = hdz * ihy * ihx, wB1 = hdz * ihy * ihxm;
        q3[1] = make_double2(wD0 * cD0.x - wD1 * cD1.x - wB0 * cB0.x + wB1 * cB1.x,
                             wD0 * cD0.y - wD1 * cD1.y - wB0 * cB0.y + wB1 * cB1.y);
        kd3[1] = wD0 + wD1 + wB0 + wB1;
        p3[1] = a0;
      }
      if (f3[2]) {  // z-edge: A=z, B=x, D=y
        const double2 a0 = Z_(z0, 0, 0);
        const double2 cD0 = csub(cadd(a0, X_(xp, 0, 0)), cadd(Z_(z0, 1, 0), X_(x0, 0, 0)));
        const double2 cD1 = csub(cadd(Z_(z0, -1, 0), X_(xp, -1, 0)), cadd(a0, X_(x0, -1, 0)));
        const double2 cB0 = csub(cadd(Y_(x0, 0, 0), Z_(z0, 0, 1)), cadd(Y_(xp, 0, 0), a0));
        const double2 cB1 = csub(cadd(Y_(x0, 0, -1), a0), cadd(Y_(xp, 0, -1), Z_(z0, 0, -1)));
        const double wD0 = hdy * ihz * ihx, wD1 = hdy * ihz * ihxm;
        const double wB0 = hdx * ihz * ihy, wB1 = hdx * ihz * ihym;
        q3[2] = make_double2(wD0 * cD0.x - wD1 * cD1.x - wB0 * cB0.x + wB1 * cB1.x,
                             wD0 * cD0.y - wD1 * cD1.y - wB0 * cB0.y + wB1 * cB1.y);
        kd3[2] = wD0 + wD1 + wB0 + wB1;
        p3[2] = a0;
      }
#undef X_
#undef Y_
#undef Z_
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (!f3[c]) continue;
        const long long slot = (long long)c * g.Nn + node;
        const double m = __ldg(A.mass + slot);
        const double2 q = cfma(sh, cscale(m, p3[c]), q3[c]);   // (K + s M) v
        if (MODE == 0) {
          A.out[vs + slot] = q;
        } else if (MODE == 1) {
          A.out[vs + slot] = p3[c];                          // p_new
          acc_c = cfma(p3[c], q, acc_c);                     // p^T A p
        } else {
          const double2 D = make_double2(kd3[c] + m * sh.x, m * sh.y);
          const long long e = vs + slot;
          A.x[e] = cfma(alpha, p3[c], A.x[e]);
          // z_new = z - alpha D^-1 q ; r_new = D z_new
          const double2 zn = csub(A.z[e], cmul(alpha, cdiv(q, D)));
          A.z[e] = zn;
          const double2 rn = cmul(D, zn);
          acc_c = cfma(rn, zn, acc_c);                       // r^T z
          acc_r += rn.x * rn.x + rn.y * rn.y;                // ||r||^2
        }
      }
      // 3. commit the prefetched plane set into the free ring slots
      const int wx = (k + 2) & 3, wz = (k + 1) % 3;
#pragma unroll
      for (int q = 0; q < LOADS; ++q) {
        const int e = tid + q * NT;
        if (e < 3 * H) store_elem(e, wx, wz, nxt[q]);
      }
      __syncthreads();
    }
  }

  if (MODE == 0) return;
  // ---- per-CTA partial -> last CTA finalises the per-shift scalars
  block_sum_n<NT>(acc_c, acc_r, red);
  if (tid == 0) {
    A.part_c[blockIdx.x] = acc_c;
    A.part_r[blockIdx.x] = acc_r;
  }
  if (!last_block(&A.ctl->ticket[MODE])) return;
  const int warp = tid >> 5, lane = tid & 31;
  const int nblk = gridDim.x;
  for (int q = warp; q < S; q += NT / 32) {
    ShiftState& sq = A.st[q];
    if (!sq.active) continue;
    double cx = 0, cy = 0, cr = 0;
    for (int b = q + lane * S; b < nblk; b += 32 * S) {
      const double2 v = __ldcg(A.part_c + b);
      cx += v.x;
      cy += v.y;
      cr += __ldcg(A.part_r + b);
    }
    cx = warp_sum(cx);
    cy = warp_sum(cy);
    cr = warp_sum(cr);
    if (lane == 0) {
      const double2 sum = make_double2(cx, cy);
      if (MODE == 1) {
        if (sum.x == 0.0 && sum.y == 0.0) {
          sq.status = 2;
          sq.active = 0;
          sq.alpha = czero();
        } else {
          sq.alpha = cdiv(sq.rho, sum);
        }
      } else {
        sq.iters += 1;
        sq.relres = sqrt(cr) / sq.fnorm;
        if (sq.relres <= A.ctl->tol) {
          sq.active = 0;
          sq.status = 1;
        } else if ((sq.rho.x == 0.0 && sq.rho.y == 0.0) || (sum.x == 0.0 && sum.y == 0.0)) {
          sq.active = 0;
          sq.status = 2;
        } else {
          sq.beta = cdiv(sum, sq.rho);
          sq.rho = sum;
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    int na = 0;
    for (int q = 0; q < S; ++q) na += A.st[q].active;
    A.ctl->n_active = na;
    A.ctl->ticket[MODE] = 0;
  }
}

}  // namespace tem
