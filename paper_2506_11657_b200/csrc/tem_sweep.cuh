// tem_sweep.cuh -- the 2.5D z-marching curl-curl sweep, TMA-fed (sm_100a).
//
// One CTA owns a TX x TY tile of nodes in the x-y plane, ONE shift s and a
// range of node planes k; it marches upward in k.  The halo-extended plane
// tiles of the swept vector (x,y components on planes k-1, k, k+1 and the z
// component on layers k-1, k) live in a shared-memory ring filled by TMA
// (cp.async.bulk.tensor, 5-D tensor map over the shift-major vector
// [S][3][nz+1][ny+1][2(nx+1)] fp64; out-of-range halo boxes are zero-filled by
// the TMA unit, which is exactly the Dirichlet boundary n x e = 0 of eq:bc).
// Loads run ahead of the arithmetic through a multi-stage mbarrier pipeline,
// so HBM latency is hidden without per-thread address arithmetic; the
// 13-point gather of
//   (K v)_a(m) = W_d(m) C_d(m) - W_d(m-e_b) C_d(m-e_b) - W_b(m) C_b(m) + W_b(m-e_d) C_b(m-e_d)
// (tem_device.cuh; §2.2, reading R1) reads shared memory only.
//
// MODE 0  apply : y = (K + s M) v                                  (tem_apply_shifted)
// MODE 1  dirap : p_new = z + beta p_old formed from TMA-staged z and p_old
//                 tiles; writes p_new; mu = p_new^T (K + s M) p_new (COCG sweep 1)
// MODE 2  upd   : v = p; x += alpha p; z -= alpha D^-1 (K + s M) p;
//                 rho = (D z)^T z, ||D z||^2                        (COCG sweep 2)
// MODE 3/4 split pass 1 (even / odd iteration): p_i = z_i + beta p_{i-1} as
//                 in MODE 1, then z_{i+1} = z_i - alpha D^-1 A p_i and (odd)
//                 x_{i+1} = x_{i-1} + alpha_{i-1} p_{i-1} + alpha_i p_i;
//                 partials gamma, eps, mu, ||r||^2, s z^T M z (R10, R11)
// k_delta         split pass 2: z^T K z by faces; finalises the split scalars
// z = D^-1 r is stored instead of r (reading "z-form"): r = D z
// is recovered where needed, so the two-sweep iteration streams x, z, p_old,
// p_new at the 128 B / unknown / shift minimum of a two-reduction COCG, and
// the split iteration 96 B.
#pragma once
#include <cuda.h>

#include "tem_device.cuh"

namespace tem {

// Tile geometry, by tile height: a CTA owns TX x TYV nodes (one thread per
// node).  TYV = 8: 256 threads, 2 CTAs/SM at <= 128 registers (two-sweep
// scheme, operator apply); TYV = 12: 384 threads, 1 CTA/SM at <= 168
// registers (split scheme: its pass 1 carries the full update and spills at
// 128 registers; measured -12% on the odd pass).
// ring: sets q = {X(q+1), Y(q+1), Z(q)}; X,Y: 5 slots, Z: 4 slots (+ z staging 2 x 3)
constexpr int R_XY = 5, R_Z = 4;
constexpr int R_D = 4;                    // k_delta ring depth (whole plane sets)
template <int TYV>
struct Tile {
  static constexpr int TX = 32;                    // tile nodes along x (one warp row)
  static constexpr int TY = TYV;
  static constexpr int NT = TX * TY;               // threads per CTA
  static constexpr int kMinBlocks = NT <= 256 ? 2 : 1;
  static constexpr int HX = TX + 2, HY = TY + 2;   // halo-extended tile
  static constexpr int TILE_BYTES = HX * HY * 16;  // one plane tile as delivered by TMA
  static constexpr int TILE_STRIDE = (TILE_BYTES + 127) / 128 * 128;   // slot pitch (128 B aligned)
  static constexpr int TS2 = TILE_STRIDE / 16;     // slot pitch in double2
  static constexpr size_t kSmemDirect = 128 + (size_t)(2 * R_XY + R_Z) * TILE_STRIDE;
  static constexpr size_t kSmemDirap = kSmemDirect + (size_t)6 * TILE_STRIDE;    // + z staging, 2 sets
  // even split pass: 4 staged z sets (own z_i served from them); a tile lower than 12 rows runs
  // 2 CTAs per SM and has room for 2 sets only (own z_i re-read)
  static constexpr int kStageSets = TYV >= 12 ? 4 : 2;
  static constexpr size_t kSmemUpd = kSmemDirect + (size_t)3 * kStageSets * TILE_STRIDE;
  static constexpr size_t kSmemDelta = 128 + (size_t)3 * R_D * TILE_STRIDE;
};
constexpr int kTYTwoSweep = 8;    // tile height of MODE 0, 1, 2
#ifndef TEM_TY_SPLIT
#define TEM_TY_SPLIT 12           // build-variant experiments: -DTEM_TY_SPLIT=6 (192 threads, 2 CTAs per SM)
#endif
constexpr int kTYSplit = TEM_TY_SPLIT;   // tile height of MODE 3, 4 and k_delta
#define TEM_TILE_CONSTANTS(TYV)                                                              \
  constexpr int TX = Tile<TYV>::TX, TY = Tile<TYV>::TY, NT = Tile<TYV>::NT;                 \
  constexpr int HX = Tile<TYV>::HX, HY = Tile<TYV>::HY, TS2 = Tile<TYV>::TS2;               \
  constexpr int TILE_BYTES = Tile<TYV>::TILE_BYTES;                                         \
  (void)TX; (void)TY; (void)NT; (void)HX; (void)HY; (void)TS2; (void)TILE_BYTES

constexpr int kMaxChunk = 128;            // max planes per z-chunk (z tables in smem)

struct ShiftState {
  double2 s;        // shift
  double2 rho;      // r^T z
  double2 alpha;
  double2 beta;
  double2 alpha_prev;   // alpha of the previous iteration (split solver: x every other iteration)
  double2 dm0;          // split solver: s z_0^T M z_0 (mass part of delta_0, from k_init)
  double fnorm;     // ||f||_2
  double relres;    // ||r||_2 / ||f||_2
  double tol;       // stopping tolerance of this shift (relative residual)
  int active;
  int iters;
  int status;       // 0 running, 1 converged, 2 breakdown
  int real;         // 1: real shift and real right-hand side -> real arithmetic (split scheme)
  int pair;         // partner shift + 1 of a pair of real shifts sharing one slot (R16), 0: none
  int lead;         // 1: component x of the pair (its block holds the packed vectors), 0: component y
};

// Control::list entry of a slot: the shift (leader of a pair) in bits 0..7,
// partner + 1 in bits 8..15.
__host__ __device__ __forceinline__ int slot_code(int s, int partner) { return s | ((partner + 1) << 8); }
__host__ __device__ __forceinline__ int slot_shift(int code) { return code & 255; }
__host__ __device__ __forceinline__ int slot_partner(int code) { return (code >> 8) - 1; }

struct Control {
  int n_active;           // number of active shifts
  unsigned int ticket[8];
  int list[32];           // the active shifts, compacted (first n_active entries)
};

struct SweepArgs {
  Grid g;
  int S;
  int nslot;                   // shift slots of the grid (CTA slot a serves shift list[a])
  int ntx, nty, nzc, kchunk;   // tiles along x, y; z-chunks and their length
  const double* mass;          // [3][Nn]
  double2* out;                // MODE 0: y; MODE 1, 3, 4: p_new
  double2* x;                  // MODE 2, 4
  double2* z;                  // MODE 2 (in/out); MODE 3, 4: z_{i+1} (out)
  const double2* zin;          // MODE 4: z_i own values (MODE 3 reads them from its TMA staging)
  const double2* pold;         // MODE 4: p_{i-1} (own values)
  ShiftState* st;              // [S]
  Control* ctl;
  const double2* rhs;          // k_init: per-shift right-hand sides (shift block), or NULL (f for all)
  double2* part_c;             // [gridDim]
  double* part_r;              // [gridDim]
  double* part;                // MODE 3, 4, k_delta: [kSplitPart][pstride] per-CTA partial sums
  int pstride;
  int band;                    // tile rows per band of the block order (block_coords)
  int force_xdirect;           // MODE 4: always re-read p_{i-1} (tests: TEM_XDIRECT=1)
  double2 shifts[32];          // MODE 0 only
};

// Split solver (MODE 3/4 pass 1, k_delta pass 2) per-CTA partials:
// [0..6] pass 1: gamma, eps, mu (re, im), ||r||^2; [7, 8] pass 2: z^T K z;
// [9, 10] pass 1: s sum_e m_e z_e^2 (the mass part of delta, pointwise);
// [11] pass 1: ||r||^2 of shift B of a pair of real shifts ([6]: shift A)
constexpr int kSplitPart = 12;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 5-D tiled TMA load of one plane tile: coords (2(i0-1), j0-1, k, comp, shift)
__device__ __forceinline__ void tma_tile(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                         int c3, int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(smem_u32(bar))
      : "memory");
}

// Per-edge mass loads (8 B per edge, shared by the S shift CTAs of a tile):
// they carry an L2 evict_last policy, so the streamed vectors do not push the
// mass out between the shift slots of a band (measured on `large`: pass 1
// even -0.6 GB of DRAM reads and -3.4% time, odd -1.7%).  The same policy in
// reverse (evict_first) on the TMA loads breaks the halo reuse between
// neighbouring tiles (+25% reads) and is not used.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_mass(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// Result stores of the sweeps are read again only by the next kernel (after
// the whole vector has streamed through L2): streaming, evict-first, so they
// do not displace the plane tiles and halo rows still to be re-read
// (measured: split pass 1 odd -4%).
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double* p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(dpair* p, dpair v) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(v.x, v.y));
}
// own-value loads through L2 (ld.global.cg)
__device__ __forceinline__ double2 ld_cgv(const double2* p) { return __ldcg(p); }
__device__ __forceinline__ double ld_cgv(const double* p) { return __ldcg(p); }
__device__ __forceinline__ dpair ld_cgv(const dpair* p) {
  const double2 v = __ldcg(reinterpret_cast<const double2*>(p));
  return make_dpair(v.x, v.y);
}

// q mod n for q >= -8n (ring slots of plane sets; sets start at kb - 2 >= -2)
__device__ __forceinline__ int pmod(int q, int n) { return (int)((unsigned)(q + 8 * n) % (unsigned)n); }

// 128-byte aligned view of the dynamic shared memory that stays a pointer
// derived from the __shared__ array (so the compiler emits LDS/STS, not
// generic LD/ST).
__device__ __forceinline__ double2* smem_align128(unsigned char* raw) {
  const uint32_t a = smem_u32(raw);
  return reinterpret_cast<double2*>(raw + ((128u - (a & 127u)) & 127u));
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

// Column constants of thread (i, j) of the tile: products of inverse cell
// widths and dual lengths that do not depend on k.
struct Column {
  int i, j, c0;
  bool in_ij;
  double pxy, pxym, pxmy;   // ih_x ih_y, ih_x ih_y(j-1), ih_x(i-1) ih_y
  double cyx, cyxm;         // hd_y ih_x, hd_y ih_x(i-1)
  double cxy, cxym;         // hd_x ih_y, hd_x ih_y(j-1)
  // bit c: edge c of the column is free (not on the boundary n x e = 0, eq:bc)
  // as far as (i, j) decide: x: i < nx, 1 <= j <= ny-1; y: 1 <= i <= nx-1, j < ny;
  // z: 1 <= i <= nx-1, 1 <= j <= ny-1.  The k part (x, y: 1 <= k <= nz-1;
  // z: 0 <= k < nz) is per plane (stencil3p).
  unsigned fm;
};

// Column constants of node column (i, j); i, j may lie outside the grid
// (halo threads of the single-pass sweep): then every weight is 0 and no
// edge of the column is free.
__device__ __forceinline__ Column make_column_ij(const Grid& g, int i, int j) {
  Column C;
  C.i = i;
  C.j = j;
  C.c0 = 0;
  C.in_ij = i >= 0 && j >= 0 && i < g.n[0] && j < g.n[1];
  const double ihx = C.in_ij ? __ldg(g.ih[0] + C.i) : 0.0;
  const double ihxm = (C.in_ij && C.i >= 1) ? __ldg(g.ih[0] + C.i - 1) : 0.0;
  const double ihy = C.in_ij ? __ldg(g.ih[1] + C.j) : 0.0;
  const double ihym = (C.in_ij && C.j >= 1) ? __ldg(g.ih[1] + C.j - 1) : 0.0;
  const double hdx = C.in_ij ? __ldg(g.hdm[0] + C.i) : 0.0;
  const double hdy = C.in_ij ? __ldg(g.hdm[1] + C.j) : 0.0;
  C.pxy = ihx * ihy;
  C.pxym = ihx * ihym;
  C.pxmy = ihxm * ihy;
  C.cyx = hdy * ihx;
  C.cyxm = hdy * ihxm;
  C.cxy = hdx * ihy;
  C.cxym = hdx * ihym;
  const bool ii = i >= 1 && i <= g.n[0] - 1, jj = j >= 1 && j <= g.n[1] - 1;
  C.fm = !C.in_ij ? 0u : ((jj ? 1u : 0u) | (ii ? 2u : 0u) | (ii && jj ? 4u : 0u));
  return C;
}

template <int TYV>
__device__ __forceinline__ Column make_column(const Grid& g, int tx0, int ty0) {
  TEM_TILE_CONSTANTS(TYV);
  const int tid = threadIdx.x;
  Column C = make_column_ij(g, tx0 + (tid % TX), ty0 + (tid / TX));
  C.c0 = ((tid / TX) + 1) * HX + (tid % TX) + 1;
  return C;
}

// K v for the three edges of node (i, j, k) from ring tiles:
// Xm/X0/Xp = x-comp planes k-1/k/k+1, same for Y; Zm/Z0 = z-comp layers k-1/k.
// The 12 (edge, face) pairs touch only 9 distinct faces and 24 distinct tile
// values: each face circulation F is formed once, scaled by its weight
// W = hdual/(mu0 A) (G = W F), and the edges combine G's with the incidence
// signs of K = T^T W T.
template <typename V>
struct Edge3 {
  V q[3], p[3];
  double kd[3];
  bool f[3];
};

// PITCH = row pitch of the tiles (in V), c0 = index of the node in them.
template <int PITCH, typename V>
__device__ __forceinline__ void stencil3p(const Grid& g, const Column& C, int c0, int k, double ihz,
                                          double ihzm, double hdz, const V* Xm, const V* X0, const V* Xp,
                                          const V* Ym, const V* Y0, const V* Yp, const V* Zm, const V* Z0,
                                          Edge3<V>& E) {
  {   // free edges: the (i, j) part is per column (Column::fm), only the k part changes per plane
    const bool kxy = k >= 1 && k <= g.n[2] - 1, kz = k >= 0 && k < g.n[2];
    E.f[0] = kxy && (C.fm & 1u);
    E.f[1] = kxy && (C.fm & 2u);
    E.f[2] = kz && (C.fm & 4u);
  }
#define T_(P, di, dj) P[c0 + (dj) * PITCH + (di)]
  const V x00 = T_(X0, 0, 0), y00 = T_(Y0, 0, 0), z00 = T_(Z0, 0, 0);
  // face weights W = hdual / (mu0 A)
  const double wz = hdz * C.pxy, wz_y = hdz * C.pxym, wz_x = hdz * C.pxmy;      // Fz(m), Fz(m-ey), Fz(m-ex)
  const double wy = C.cyx * ihz, wy_z = C.cyx * ihzm, wy_x = C.cyxm * ihz;      // Fy(m), Fy(m-ez), Fy(m-ex)
  const double wx = C.cxy * ihz, wx_z = C.cxy * ihzm, wx_y = C.cxym * ihz;      // Fx(m), Fx(m-ez), Fx(m-ey)
  // G = W * circulation (right-hand rule about the face normal), accumulated
  // into (K v)_x = Gz - Gz(m-ey) - Gy + Gy(m-ez), (K v)_y = Gx - Gx(m-ez) - Gz + Gz(m-ex),
  // (K v)_z = Gy - Gy(m-ex) - Gx + Gx(m-ey): the three faces at m serve two
  // edges each (weight applied once), the six others one edge each (weight
  // folded into the accumulation, one FMA per component)
  V qx, qy, qz;
  {
    const V Gz = cscale(wz, csub(cadd(x00, T_(Y0, 1, 0)), cadd(T_(X0, 0, 1), y00)));     // Fz(m)
    const V Gy = cscale(wy, csub(cadd(z00, T_(Xp, 0, 0)), cadd(T_(Z0, 1, 0), x00)));     // Fy(m)
    const V Gx = cscale(wx, csub(cadd(y00, T_(Z0, 0, 1)), cadd(T_(Yp, 0, 0), z00)));     // Fx(m)
    qx = csub(Gz, Gy);
    qy = csub(Gx, Gz);
    qz = csub(Gy, Gx);
  }
  qx = sfma(-wz_y, csub(cadd(T_(X0, 0, -1), T_(Y0, 1, -1)), cadd(x00, T_(Y0, 0, -1))), qx);   // Fz(m-ey)
  qx = sfma(wy_z, csub(cadd(T_(Zm, 0, 0), x00), cadd(T_(Zm, 1, 0), T_(Xm, 0, 0))), qx);      // Fy(m-ez)
  qy = sfma(wz_x, csub(cadd(T_(X0, -1, 0), y00), cadd(T_(X0, -1, 1), T_(Y0, -1, 0))), qy);   // Fz(m-ex)
  qy = sfma(-wx_z, csub(cadd(T_(Ym, 0, 0), T_(Zm, 0, 1)), cadd(y00, T_(Zm, 0, 0))), qy);     // Fx(m-ez)
  qz = sfma(-wy_x, csub(cadd(T_(Z0, -1, 0), T_(Xp, -1, 0)), cadd(z00, T_(X0, -1, 0))), qz);   // Fy(m-ex)
  qz = sfma(wx_y, csub(cadd(T_(Y0, 0, -1), z00), cadd(T_(Yp, 0, -1), T_(Z0, 0, -1))), qz);     // Fx(m-ey)
#undef T_
  E.q[0] = qx;
  E.q[1] = qy;
  E.q[2] = qz;
  E.kd[0] = wz + wz_y + wy + wy_z;
  E.kd[1] = wx + wx_z + wz + wz_x;
  E.kd[2] = wy + wy_x + wx + wx_y;
  E.p[0] = x00;
  E.p[1] = y00;
  E.p[2] = z00;
}

template <int TYV, typename V>
__device__ __forceinline__ void stencil3(const Grid& g, const Column& C, int k, double ihz, double ihzm,
                                         double hdz, const V* Xm, const V* X0, const V* Xp, const V* Ym,
                                         const V* Y0, const V* Yp, const V* Zm, const V* Z0, Edge3<V>& E) {
  stencil3p<Tile<TYV>::HX>(g, C, C.c0, k, ihz, ihzm, hdz, Xm, X0, Xp, Ym, Y0, Yp, Zm, Z0, E);
}

// v^T K v restricted to the three faces whose lower corner is this node
// (K = T^T W T, §2.2: v^T K v = sum_f W_f C_f(v)^2 over all faces,
// unconjugated square for the complex-symmetric form).  Summed over all
// nodes every face is counted once; it reads only the +x, +y, +z neighbours.
template <int TYV, typename V>
__device__ __forceinline__ V faces_quad(const Column& C, double ihz, double hdz, const V* X0, const V* Xp,
                                        const V* Y0, const V* Yp, const V* Z0) {
  constexpr int HX = Tile<TYV>::HX;
  const int c0 = C.c0;
  const V x00 = X0[c0], y00 = Y0[c0], z00 = Z0[c0];
  const V Fz = csub(cadd(x00, Y0[c0 + 1]), cadd(X0[c0 + HX], y00));
  const V Fy = csub(cadd(z00, Xp[c0]), cadd(Z0[c0 + 1], x00));
  const V Fx = csub(cadd(y00, Z0[c0 + HX]), cadd(Yp[c0], z00));
  V acc = cscale(hdz * C.pxy, csq(Fz));
  acc = cadd(acc, cscale(C.cyx * ihz, csq(Fy)));
  return cadd(acc, cscale(C.cxy * ihz, csq(Fx)));
}

// Split solver finalisation (last CTA of pass 2): per-shift sums of the pass-1
// partials (gamma, eps, mu, ||r||^2) and the pass-2 partial delta, then
//   beta = gamma / gamma_prev,  p^T A p = delta + beta (2 eps + beta mu),
//   alpha = gamma / p^T A p     (reading R10)
// PRIME (after k_init): alpha_0 = gamma_0 / delta_0.
// ShiftState through L2 (ld.global.cg): a persistent CTA must not see an
// L1 copy of a state another SM's finalisation has since changed.
__device__ __forceinline__ ShiftState ld_state(const ShiftState* p) {
  static_assert(sizeof(ShiftState) % 8 == 0, "ShiftState is copied as 8-byte words");
  ShiftState v;
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(p);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(&v);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(ShiftState) / 8); ++i) dst[i] = __ldcg(src + i);
  return v;
}
__device__ __forceinline__ int ld_cg(const int* p) { return __ldcg(p); }

// One shift's scalar update from its sums (real shifts and the members of a
// pair pass zero imaginary parts): returns with sq updated.
template <bool PRIME>
__device__ __forceinline__ void split_update(ShiftState& sq, double2 gam, double2 eps, double2 mu, double2 dk,
                                             double2 dm, double rr) {
  if (PRIME) {
    const double2 del0 = cadd(dk, sq.dm0);
    if (del0.x == 0.0 && del0.y == 0.0) {
      sq.active = 0;
      sq.status = 2;
    } else {
      sq.alpha = cdiv(sq.rho, del0);
      sq.alpha_prev = czero();
      sq.beta = czero();
    }
    return;
  }
  const double2 del = cadd(dk, dm);   // z^T K z + s z^T M z
  sq.iters += 1;
  sq.relres = sqrt(rr) / sq.fnorm;
  if (sq.relres <= sq.tol) {
    sq.active = 0;
    sq.status = 1;
  } else if ((gam.x == 0.0 && gam.y == 0.0) || (sq.rho.x == 0.0 && sq.rho.y == 0.0)) {
    sq.active = 0;
    sq.status = 2;
  } else {
    const double2 beta = cdiv(gam, sq.rho);
    const double2 den = cadd(del, cmul(beta, cadd(cscale(2.0, eps), cmul(beta, mu))));
    if (den.x == 0.0 && den.y == 0.0) {
      sq.active = 0;
      sq.status = 2;
    } else {
      sq.beta = beta;
      sq.alpha_prev = sq.alpha;
      sq.alpha = cdiv(gam, den);
      sq.rho = gam;
    }
  }
}

// A member of a pair that has stopped while its partner runs on is frozen:
// alpha = beta = 0 (p = z, z unchanged), and its last step length moves to
// alpha_prev once, so the next odd pass (or k_xfix) still adds alpha_i p_i to
// x exactly once (R11, R16).
__device__ __forceinline__ void pair_freeze(ShiftState& sq) {
  sq.alpha_prev = sq.alpha;
  sq.alpha = czero();
  sq.beta = czero();
}

// The active slots: a single shift while it is active, a pair while either
// member is (the leader carries the slot).  Called by the whole first warp
// (S <= 32: one shift per lane, one L2 round trip instead of a serial scan --
// the scan was ~4 us per iteration, a tenth of an iteration of `block`).
__device__ __forceinline__ void rebuild_list(const SweepArgs& A) {
  const int lane = threadIdx.x & 31;
  const bool has = lane < A.S;
  const int partner = has ? ld_cg(&A.st[lane].pair) - 1 : -1;
  const int lead = has ? ld_cg(&A.st[lane].lead) : 0;
  const int act = has ? ld_cg(&A.st[lane].active) : 0;
  const int pact = __shfl_sync(0xffffffffu, act, partner >= 0 ? partner : 0);
  const bool slot = has && (partner < 0 ? act != 0 : (lead && (act || pact)));
  const unsigned mask = __ballot_sync(0xffffffffu, slot);
  if (slot) A.ctl->list[__popc(mask & ((1u << lane) - 1u))] = slot_code(lane, partner);
  if (lane == 0) A.ctl->n_active = __popc(mask);
}

template <bool PRIME, int TYV>
__device__ void finalize_split(const SweepArgs& A, int ns, int per) {
  // ns: shift slots of the pass; per: work units (partials) per slot
  constexpr int NT = Tile<TYV>::NT;
  const int n_list = ld_cg(&A.ctl->n_active);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int a = warp; a < ns && a < n_list; a += NT / 32) {
    const int code = ld_cg(&A.ctl->list[a]);
    const int sidx = slot_shift(code), pidx = slot_partner(code);
    const bool act_a = ld_cg(&A.st[sidx].active) != 0;
    const bool act_b = pidx >= 0 && ld_cg(&A.st[pidx].active) != 0;
    if (!act_a && !act_b) continue;
    double v[kSplitPart];
#pragma unroll
    for (int t = 0; t < kSplitPart; ++t) {
      double acc = 0.0;
      if (!PRIME || t == 7 || t == 8)   // PRIME: the mass part of delta_0 is sq.dm0
        for (int b = a * per + lane; b < (a + 1) * per; b += 32) acc += __ldcg(A.part + t * A.pstride + b);
      v[t] = warp_sum(acc);
    }
    if (lane != 0) continue;
    if (pidx < 0) {
      ShiftState sq = ld_state(&A.st[sidx]);
      split_update<PRIME>(sq, make_double2(v[0], v[1]), make_double2(v[2], v[3]), make_double2(v[4], v[5]),
                          make_double2(v[7], v[8]), make_double2(v[9], v[10]), v[6]);
      A.st[sidx] = sq;
      continue;
    }
    // a pair: component x is shift sidx, component y its partner, both real
    // (one member at a time: one ShiftState live)
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int q = h ? pidx : sidx;
      ShiftState sq = ld_state(&A.st[q]);
      if (h ? act_b : act_a) {
        split_update<PRIME>(sq, make_double2(v[0 + h], 0.0), make_double2(v[2 + h], 0.0),
                            make_double2(v[4 + h], 0.0), make_double2(v[7 + h], 0.0),
                            make_double2(v[9 + h], 0.0), h ? v[11] : v[6]);
        if (!sq.active) pair_freeze(sq);
      } else if (!PRIME) {
        pair_freeze(sq);
      }
      A.st[q] = sq;
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    __threadfence();
    rebuild_list(A);
    if (threadIdx.x == 0) A.ctl->ticket[PRIME ? 6 : 5] = 0;
  }
}

// Finalisation by the last CTA: per-shift sums of the per-CTA partials (the
// CTAs of slot a are blockIdx = a mod nslot and served shift list[a]), COCG
// scalar updates, then the compacted active list for the next launch.
template <int MODE, int TYV>
__device__ void finalize(const SweepArgs& A) {
  constexpr int NT = Tile<TYV>::NT;
  const int S = A.S, ns = A.nslot;
  const int n_list = A.ctl->n_active;   // as read by every CTA of this launch
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = gridDim.x / ns;   // blocks per shift slot (pidx of block_coords)
  for (int a = warp; a < ns && a < n_list; a += NT / 32) {
    ShiftState& sq = A.st[A.ctl->list[a]];
    if (!sq.active) continue;
    double cx = 0, cy = 0, cr = 0;
    for (int b = a * per + lane; b < (a + 1) * per; b += 32) {
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
        if (sq.relres <= sq.tol) {
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
  if (threadIdx.x == 0) {
    int na = 0;
    for (int q = 0; q < S; ++q)
      if (A.st[q].active) A.ctl->list[na++] = q;
    A.ctl->n_active = na;
    A.ctl->ticket[MODE] = 0;
  }
}

// block -> (z-chunk, band of `band` tile rows, shift slot, tile row, tile
// column), column fastest.  The CTAs of one band run together for all shift
// slots, so (i) the S CTAs of a tile share its coefficients (mass) through L2
// and (ii) a tile's +-y halo rows were streamed moments earlier by its
// neighbour in the band (L2 hits instead of DRAM re-reads).  band = 0: the
// slot-fastest order (slot, then column, then row).  pidx: index of the
// block's reduction partials, slot-major ([slot][tile and chunk]).
template <int TYV>
__device__ __forceinline__ void unit_coords(const SweepArgs& A, int idx, int ns, int nzc, int kchunk, int& a,
                                            int& tx0, int& ty0, int& kb, int& ke, int& pidx) {
  constexpr int TX = Tile<TYV>::TX, TY = Tile<TYV>::TY;
  const int ntx = A.ntx, nty = A.nty;
  const int per_z = ns * ntx * nty;
  const int zc = idx / per_z;
  int r = idx - zc * per_z;
  int tx, ty;
  if (A.band <= 0) {
    a = r % ns;
    const int xy = r / ns;
    tx = xy % ntx;
    ty = xy / ntx;
  } else {
    const int per_band = A.band * ntx * ns;
    const int band = r / per_band;
    r -= band * per_band;
    const int rows = min(A.band, nty - band * A.band);
    a = r / (rows * ntx);
    const int t = r - a * rows * ntx;
    ty = band * A.band + t / ntx;
    tx = t % ntx;
  }
  tx0 = tx * TX;
  ty0 = ty * TY;
  kb = zc * kchunk;
  ke = min(kb + kchunk, A.g.n[2]);
  pidx = a * (nzc * ntx * nty) + (zc * nty + ty) * ntx + tx;
}
template <int TYV>
__device__ __forceinline__ void block_coords(const SweepArgs& A, int& a, int& tx0, int& ty0, int& kb,
                                             int& ke, int& pidx) {
  unit_coords<TYV>(A, blockIdx.x, A.nslot, A.nzc, A.kchunk, a, tx0, ty0, kb, ke, pidx);
}

// ---------------------------------------------------------------- layouts
// Shift s's vectors in a shift block: complex -> [3][Nn] double2 at
// s * 3 Nn (include/tem_b200.h); real -> [3][NnP] double at the start of the
// same region (Grid::px, NnP).
template <typename V>
__device__ __forceinline__ V* vbase(const double2* p, int s, const Grid& g) {
  if constexpr (VT<V>::kReal)
    return reinterpret_cast<V*>(const_cast<double2*>(p)) + (long long)s * 6 * g.Nn;
  else
    return const_cast<double2*>(p) + (long long)s * 3 * g.Nn;
}
template <typename V>
__device__ __forceinline__ long long vcomp(const Grid& g) {
  if constexpr (VT<V>::kReal) return g.NnP; else return g.Nn;
}
template <typename V>
__device__ __forceinline__ int vrow(const Grid& g) {
  if constexpr (VT<V>::kReal) return g.px; else return g.n[0] + 1;
}
// column of node i in a row of this layout is i + vofs
template <typename V>
__device__ __forceinline__ constexpr int vofs() {
  return VT<V>::kReal ? 1 : 0;
}

// ---------------------------------------------------------------- sweeps
// One kernel for all modes.  Plane sets q = {X(q+1), Y(q+1), Z(q)} of the
// swept vector v live in a ring: X,Y slots q mod 5, Z slots q mod 4,
// mbarrier q mod 5.  MODE 0/2: v is read as is, three sets run ahead of the
// arithmetic.  MODE 1/3/4: v = p_old is loaded into the ring and z into a
// staging area; when set q has landed it is combined IN PLACE into
// p_new = z + beta p_old (at the end of step q-1, two sets ahead).
// The split modes run a real shift (ShiftState::real) in real arithmetic:
// the same body over V = double, half-size tiles in the same ring slots.
struct Partials {
  double2 c, e, m;   // gamma (MODE 1: p^T A p), eps, mu; a pair of real shifts: (A, B) in (x, y)
  double2 dm;        // split: s z^T M z (the mass part of delta)
  double r, r2;      // ||r||^2 (r2: shift B of a pair)
};

// The vectors one sweep reads and writes (per iteration parity).
struct Bufs {
  double2* out;          // MODE 0: y; MODE 1, 3, 4: p_new
  double2* z;            // MODE 2 (in/out); MODE 3, 4: z_{i+1}
  const double2* zin;    // MODE 4: z_i own values
  const double2* pold;   // MODE 4: p_{i-1} own values
};
__host__ __device__ __forceinline__ Bufs bufs_of(const SweepArgs& A) { return Bufs{A.out, A.z, A.zin, A.pold}; }

template <int MODE, int TYV, typename V>
__device__ __forceinline__ void sweep_body(const SweepArgs& A, const CUtensorMap* tmv, const CUtensorMap* tmz,
                                           int s, int tx0, int ty0, int kb, int ke, double2 sh2, double2 alpha2,
                                           double2 beta2, double2 alpha_prev2, double2* ring2, uint64_t* bar,
                                           uint32_t& phase, bool init_bars, double* zih, double* zhd, Partials& P,
                                           const Bufs& B) {
  TEM_TILE_CONSTANTS(TYV);
  constexpr bool kZ = (MODE == 1 || MODE == 3 || MODE == 4);   // p_new = z + beta p_old formed in smem
  constexpr bool kUpd = (MODE == 3 || MODE == 4);               // split pass 1: full update
  constexpr int kW = sizeof(V) / 8;                             // doubles per value
  constexpr int TSV = TS2 * 2 / kW;                             // slot pitch in V
  constexpr int TILE_V = HX * HY * (int)sizeof(V);              // bytes of one TMA plane tile
  V* ring = reinterpret_cast<V*>(ring2);
  V* rX = ring;                        // [R_XY] slots
  V* rY = ring + R_XY * TSV;           // [R_XY]
  V* rZ = ring + 2 * R_XY * TSV;       // [R_Z]
  // z staging [RS][3 tiles]: 2 sets (MODE 1, 4); 4 sets (MODE 3), so that the
  // node's own z_i (X, Y of set k-1, Z of set k) is still staged at step k
  // own z_i from the staging (else re-read from global memory)
  constexpr bool kZOwn = MODE == 3 && Tile<TYV>::kStageSets == 4;
  constexpr int RS = kZOwn ? 4 : 2;
  V* zs = ring + (2 * R_XY + R_Z) * TSV;
  const Grid& g = A.g;
  const int tid = threadIdx.x;
  const V sh = VT<V>::from(sh2), alpha = VT<V>::from(alpha2), beta = VT<V>::from(beta2);
  const V alpha_prev = VT<V>::from(alpha_prev2);
  V acc_c = VT<V>::zero(), acc_e = VT<V>::zero(), acc_m = VT<V>::zero(), acc_q = VT<V>::zero();
  typename VT<V>::R acc_r = VT<V>::rzero();
  // MODE 4: x_{i+1} = x_{i-1} + (alpha_i + a/beta_i) p_i - (a/beta_i) z_i, a = alpha_{i-1}
  // (exact rewrite of alpha_{i-1} p_{i-1} + alpha_i p_i).  Its rounding error,
  // relative to the x increment, grows like |z_i| / |beta_i p_{i-1}|; when
  // |beta_i| < 1/32 (about 2% of iterations) p_{i-1} is re-read instead (x_direct).
  const bool x_direct =
      MODE == 4 && (A.force_xdirect || VT<V>::small_beta(beta, alpha, alpha_prev, 1.0 / 1024.0));
  // x_{i+1} = x_{i-1} + xc_p p_i + xc_z (z_i, or p_{i-1} when x_direct)
  V xc_p = alpha, xc_z = alpha_prev;
  if (MODE == 4 && !x_direct) {
    xc_z = VT<V>::div0(alpha_prev, beta);
    xc_p = cadd(alpha, xc_z);
    xc_z = cscale(-1.0, xc_z);
  }

  const Column C = make_column<TYV>(g, tx0, ty0);
  // element indices inside one shift's vector are 32-bit (3 NnP < 2^31), and
  // with the shift's offset unsigned 32-bit (check_index in tem_b200.cu): an
  // address is a kernel-parameter base + one widening multiply-add instead of
  // a 64-bit index chain per access (-8..-15% instructions in the split pass 1)
  typedef int idx_t;
  const idx_t cst = (idx_t)vcomp<V>(g);              // component stride of this layout
  const int rowp = vrow<V>(g);                       // node row pitch of this layout
  const int nx1 = g.n[0] + 1, ny1 = g.n[1] + 1;
  const unsigned sb = (unsigned)s * (unsigned)((VT<V>::kReal ? 6 : 3) * g.Nn);   // the shift's offset
  V* out = reinterpret_cast<V*>(B.out);
  V* xv = reinterpret_cast<V*>(A.x);
  V* zv = reinterpret_cast<V*>(B.z);
  const V* zin = reinterpret_cast<const V*>(B.zin);
  const V* pold = reinterpret_cast<const V*>(B.pold);
#define TEM_EI(e) ((unsigned)(e) + sb)
  for (int q = tid; q <= ke - kb; q += NT) {
    const int k = kb - 1 + q;
    zih[q] = k >= 0 ? __ldg(g.ih[2] + k) : 0.0;
    if (q < ke - kb) zhd[q] = __ldg(g.hdm[2] + kb + q);
  }
  // Set kb-2 carries no Z tile: Z(kb-2) is never read, and with five sets in
  // flight its Z slot is the one set kb+2 fills (two TMAs into one slot race).
  auto issue = [&](int q) {
    const int sx = pmod(q, R_XY), sz = pmod(q, R_Z);
    const bool with_z = q > kb - 2;
    const int ntile = (with_z ? 3 : 2) * (kZ ? 2 : 1);
    mbar_expect_tx(&bar[sx], ntile * TILE_V);
    const int cx = kW * (tx0 - 1) + vofs<V>(), cy = ty0 - 1;   // even: 16-byte aligned box origin
    tma_tile(rX + sx * TSV, tmv, cx, cy, q + 1, 0, s, &bar[sx]);
    tma_tile(rY + sx * TSV, tmv, cx, cy, q + 1, 1, s, &bar[sx]);
    if (with_z) tma_tile(rZ + sz * TSV, tmv, cx, cy, q, 2, s, &bar[sx]);
    if (kZ) {
      V* d = zs + pmod(q, RS) * 3 * TSV;
      tma_tile(d, tmz, cx, cy, q + 1, 0, s, &bar[sx]);
      tma_tile(d + TSV, tmz, cx, cy, q + 1, 1, s, &bar[sx]);
      if (with_z) tma_tile(d + 2 * TSV, tmz, cx, cy, q, 2, s, &bar[sx]);
    }
  };
  // phase: bit b = parity of the next wait on bar[b] (kept across the work
  // units of a persistent CTA; every unit waits for every set it issues)
  auto wait_set = [&](int q) {
    const int b = pmod(q, R_XY);
    mbar_wait(&bar[b], (phase >> b) & 1u);
    phase ^= 1u << b;
  };
  // MODE 1/3/4: wait for set q and form p_new = z + beta p_old in its ring slots
  auto combine = [&](int q) {
    wait_set(q);
    const V* d = zs + pmod(q, RS) * 3 * TSV;
    V* dX = rX + pmod(q, R_XY) * TSV;
    V* dY = rY + pmod(q, R_XY) * TSV;
    V* dZ = rZ + pmod(q, R_Z) * TSV;
    const bool with_z = q > kb - 2;
    for (int e = tid; e < HX * HY; e += NT) {
      dX[e] = cfma(beta, dX[e], d[e]);
      dY[e] = cfma(beta, dY[e], d[TSV + e]);
      if (with_z) dZ[e] = cfma(beta, dZ[e], d[2 * TSV + e]);
    }
  };
  if (tid == 0) {
    if (init_bars) {
      for (int q = 0; q < R_XY; ++q) mbar_init(&bar[q], 1);
      fence_barrier_init();
    }
    fence_proxy_async();   // persistent CTA: the previous unit's generic smem accesses before the TMA writes
  }
  __syncthreads();
  if (!kZ) {
    if (tid == 0)
      for (int q = kb - 2; q <= min(kb + 2, ke - 1); ++q) issue(q);
    wait_set(kb - 2);
    wait_set(kb - 1);
  } else {
    // z staging has 2 slots: sets enter two at a time
    if (tid == 0) {
      issue(kb - 2);
      issue(kb - 1);
    }
    for (int q = kb - 2; q <= kb; ++q) {
      combine(q);
      __syncthreads();
      if (tid == 0 && q + 2 <= ke - 1) {
        fence_proxy_async();
        issue(q + 2);
      }
    }
  }

  // centre operands (mass; MODE 2: x, z; MODE 4: x, z) of the next step, loaded a step ahead
  double mN[3];
  V xN[3], zN[3];
  const uint64_t mass_pol = l2_policy_evict_last();
  // threads outside the grid (partial tiles) load column (0, 0): valid memory,
  // values unused (none of their edges is free) -- no predicates, no zero fill
  const int ci = C.in_ij ? C.i : 0, cj = C.in_ij ? C.j : 0;
  auto load_centre = [&](int k) {   // kb <= k < ke <= nz
    const idx_t node = ((idx_t)k * ny1 + cj) * nx1 + ci;
    const idx_t nodeV = ((idx_t)k * ny1 + cj) * rowp + ci + vofs<V>();
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      mN[c] = ld_mass(A.mass + (unsigned)(c * (idx_t)g.Nn + node), mass_pol);
      const idx_t slot = c * cst + nodeV;
      if (MODE == 2) {
        xN[c] = xv[TEM_EI(slot)];
        zN[c] = zv[TEM_EI(slot)];
      }
      if (MODE == 4) xN[c] = ld_cgv(xv + TEM_EI(slot));
      if (kUpd && !kZOwn) zN[c] = ld_cgv(zin + TEM_EI(slot));
    }
  };
  load_centre(kb);

  // ring slots of the planes the stencil reads: X, Y of k-1, k, k+1 (sets
  // k-2, k-1, k), Z of k-1, k (sets k-1, k); rotated once per step
  int sxm = pmod(kb - 2, R_XY), sx0 = pmod(kb - 1, R_XY), sxp = pmod(kb, R_XY);
  int szm = pmod(kb - 1, R_Z), sz0 = pmod(kb, R_Z);
  const idx_t col = (idx_t)C.j * rowp + C.i + vofs<V>();   // own column, component 0, plane 0
  const idx_t plane = (idx_t)rowp * ny1;
#pragma unroll 1
  for (int k = kb; k < ke; ++k) {
    if (!kZ) wait_set(k);
    Edge3<V> E;
    stencil3<TYV>(g, C, k, zih[k - kb + 1], zih[k - kb], zhd[k - kb], rX + sxm * TSV, rX + sx0 * TSV,
                  rX + sxp * TSV, rY + sxm * TSV, rY + sx0 * TSV, rY + sxp * TSV, rZ + szm * TSV,
                  rZ + sz0 * TSV, E);
    sxm = sx0;
    sx0 = sxp;
    sxp = sxp + 1 == R_XY ? 0 : sxp + 1;
    szm = sz0;
    sz0 = sz0 + 1 == R_Z ? 0 : sz0 + 1;
    const idx_t ek = col + (idx_t)k * plane;
    if (kZOwn) {   // own z_i from the staging tiles: X, Y of set k-1, Z of set k
      const V* zk1 = zs + pmod(k - 1, RS) * 3 * TSV;
      const V* zk = zs + pmod(k, RS) * 3 * TSV;
      zN[0] = zk1[C.c0];
      zN[1] = zk1[TSV + C.c0];
      zN[2] = zk[2 * TSV + C.c0];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (!E.f[c]) continue;
      const auto e = TEM_EI(ek + c * cst);
      const V q = cfma(sh, cscale(mN[c], E.p[c]), E.q[c]);   // (K + s M) v
      if (kUpd) {
        const V D = VT<V>::diag(E.kd[c], mN[c], sh);
        typename VT<V>::R nD;                                           // |D|^2
        const V zn = csub(zN[c], cmul(alpha, cmul(q, crcp(D, nD))));   // z_i - alpha D^-1 A p_i
        st_stream(out + e, E.p[c]);                                     // p_i
        st_stream(zv + e, zn);                                          // z_{i+1}
        if (MODE == 4) {   // x_{i+1} = x_{i-1} + alpha_{i-1} p_{i-1} + alpha_i p_i
          if (x_direct)
            st_stream(xv + e, cfma(xc_p, E.p[c], cfma(xc_z, ld_cgv(pold + e), xN[c])));
          else   // p_{i-1} = (p_i - z_i) / beta_i: no re-read of p_{i-1}
            st_stream(xv + e, cfma(xc_z, zN[c], cfma(xc_p, E.p[c], xN[c])));
        }
        const V zq = csq(zn);                                           // z_{i+1}^2
        acc_c = sfma(E.kd[c], zq, acc_c);            // gamma_{i+1} = (D z)^T z = sum kd z^2 + s z^T M z
        acc_r = VT<V>::rfma(nD, VT<V>::abs2(zn), acc_r);   // ||D z||^2
        acc_q = sfma(mN[c], zq, acc_q);              // z^T M z
        acc_e = cfma(zn, q, acc_e);                  // z_{i+1}^T A p_i
        acc_m = cfma(E.p[c], q, acc_m);              // p_i^T A p_i
      } else if (MODE == 0) {
        out[e] = q;
      } else if (MODE == 1) {
        st_stream(out + e, E.p[c]);      // p_new
        acc_c = cfma(E.p[c], q, acc_c);  // p^T A p
      } else {
        const V D = VT<V>::diag(E.kd[c], mN[c], sh);
        st_stream(xv + e, cfma(alpha, E.p[c], xN[c]));
        const V zn = csub(zN[c], cmul(alpha, cdiv(q, D)));   // z - alpha D^-1 q
        st_stream(zv + e, zn);
        const V rn = cmul(D, zn);                           // r = D z
        acc_c = cfma(rn, zn, acc_c);
        acc_r = VT<V>::rfma(VT<V>::abs2(rn), VT<V>::rone(), acc_r);
      }
    }
    // centre operands of step k+1: issued now, consumed after step k+1's stencil
    if (k + 1 < ke) load_centre(k + 1);
    // MODE 1/3/4: set k+1's ring slots held set k-4/k-3 (no longer read): combine it now
    if (kZ && k + 1 <= ke - 1) combine(k + 1);
    __syncthreads();   // all reads of set k-2 done -> its slots may be refilled
    if (tid == 0 && k + 3 <= ke - 1) {
      fence_proxy_async();
      issue(k + 3);
    }
  }
  // gamma = sum (kd + s m) z^2: the mass part s z^T M z is acc_q (MODE 3/4)
  const V dm = cmul(sh, acc_q);   // s z^T M z
  P.c = VT<V>::cplx(kUpd ? cadd(acc_c, dm) : acc_c);
  P.e = VT<V>::cplx(acc_e);
  P.m = VT<V>::cplx(acc_m);
  P.dm = VT<V>::cplx(dm);
  P.r = VT<V>::r0(acc_r);
  P.r2 = VT<V>::r1(acc_r);
#undef TEM_EI
}

// Split pass 1: the CTA's partial sums (gamma, eps, mu, ||r||^2, s z^T M z)
// -> A.part[t][pidx] (fixed-order block reduction, deterministic).
template <int NT>
__device__ __forceinline__ void write_split_partials(const SweepArgs& A, const Partials& P, int pidx) {
  __shared__ double red9[kSplitPart * NT / 32];
  const int tid = threadIdx.x;
  double v[kSplitPart] = {P.c.x, P.c.y, P.e.x, P.e.y, P.m.x, P.m.y, P.r, 0.0, 0.0, P.dm.x, P.dm.y, P.r2};
#pragma unroll
  for (int t = 0; t < kSplitPart; ++t)
    if (t < 7 || t > 8)
      for (int o = 16; o > 0; o >>= 1) v[t] += __shfl_down_sync(0xffffffffu, v[t], o);
  const int w = tid >> 5, l = tid & 31;
  __syncthreads();
  if (l == 0)
    for (int t = 0; t < kSplitPart; ++t) red9[kSplitPart * w + t] = v[t];
  __syncthreads();
  if (tid < kSplitPart && (tid < 7 || tid > 8)) {
    double acc = 0.0;
    for (int q = 0; q < NT / 32; ++q) acc += red9[kSplitPart * q + tid];
    A.part[tid * A.pstride + pidx] = acc;
  }
}

// tmv/tmz: tensor maps of the swept vector and of z over complex shift
// blocks; tmvr/tmzr: the same buffers in the real layout (split modes).
template <int MODE, int TYV = (MODE >= 3 ? kTYSplit : kTYTwoSweep)>
__global__ void __launch_bounds__(Tile<TYV>::NT, Tile<TYV>::kMinBlocks)
    k_sweep(const __grid_constant__ SweepArgs A, const __grid_constant__ CUtensorMap tmv,
            const __grid_constant__ CUtensorMap tmz, const __grid_constant__ CUtensorMap tmvr,
            const __grid_constant__ CUtensorMap tmzr) {
  constexpr int NT = Tile<TYV>::NT;
  constexpr bool kUpd = (MODE == 3 || MODE == 4);
  extern __shared__ unsigned char smem_raw[];
  double2* ring = smem_align128(smem_raw);
  __shared__ __align__(8) uint64_t bar[R_XY];
  __shared__ double red[3 * NT / 32];
  __shared__ double zih[kMaxChunk + 1];     // ih_z[k] for k = kb-1 .. ke-1
  __shared__ double zhd[kMaxChunk];         // hdual_z[k]/mu0 for k = kb .. ke-1

  int a, tx0, ty0, kb, ke;
  int pidx;
  block_coords<TYV>(A, a, tx0, ty0, kb, ke, pidx);
  const int tid = threadIdx.x;

  double2 sh = czero(), alpha = czero(), beta = czero(), alpha_prev = czero();
  bool live, real = false, pair = false;
  int s = a;
  if (MODE == 0) {
    sh = A.shifts[s];
    live = true;
  } else {
    // n_active and list[a] share a cache line: both loads go out together (one L2
    // round trip instead of two dependent ones ahead of every CTA's first TMA)
    const int n_act = A.ctl->n_active, code = A.ctl->list[a & 31];
    live = a < n_act;
    if (live) {
      s = slot_shift(code);
      const ShiftState& st = A.st[s];
      sh = st.s;
      alpha = st.alpha;
      beta = st.beta;
      alpha_prev = st.alpha_prev;
      live = st.active != 0;
      real = kUpd && st.real;
      if (kUpd && slot_partner(code) >= 0) {   // two real shifts: scalars packed (A, B) component-wise
        const ShiftState& sb = A.st[slot_partner(code)];
        pair = true;
        sh.y = sb.s.x;
        alpha.y = sb.alpha.x;
        beta.y = sb.beta.x;
        alpha_prev.y = sb.alpha_prev.x;
        live = live || sb.active != 0;
      }
    }
  }
  Partials P{};
  uint32_t phase = 0;
  const Bufs B = bufs_of(A);
  if (live) {
    if constexpr (kUpd) {
      if (pair)
        sweep_body<MODE, TYV, dpair>(A, &tmv, &tmz, s, tx0, ty0, kb, ke, sh, alpha, beta, alpha_prev, ring,
                                     bar, phase, true, zih, zhd, P, B);
      else if (real)
        sweep_body<MODE, TYV, double>(A, &tmvr, &tmzr, s, tx0, ty0, kb, ke, sh, alpha, beta, alpha_prev,
                                      ring, bar, phase, true, zih, zhd, P, B);
      else
        sweep_body<MODE, TYV, double2>(A, &tmv, &tmz, s, tx0, ty0, kb, ke, sh, alpha, beta, alpha_prev,
                                       ring, bar, phase, true, zih, zhd, P, B);
    } else {
      sweep_body<MODE, TYV, double2>(A, &tmv, &tmz, s, tx0, ty0, kb, ke, sh, alpha, beta, alpha_prev, ring,
                                     bar, phase, true, zih, zhd, P, B);
    }
  }
  if (MODE == 0) return;
  if (kUpd) {
    write_split_partials<NT>(A, P, pidx);
    return;
  }
  double2 acc_c = P.c;
  double acc_r = P.r;
  block_sum_n<NT>(acc_c, acc_r, red);
  if (tid == 0) {
    A.part_c[pidx] = acc_c;
    A.part_r[pidx] = acc_r;
  }
  if (!last_block(&A.ctl->ticket[MODE])) return;
  finalize<MODE, TYV>(A);
}

// ---------------------------------------------------------------- pass 2
// k_delta: z^T K z of the split solver, per shift, from the node's own faces
// (faces_quad); the mass term s z^T M z is pointwise and comes with pass 1
// (k_init for z_0).  It reads z once (16 B per unknown per shift; 8 B for a
// real shift) with a +1 halo; plane sets q = {X(q), Y(q), Z(q)} in a 4-deep
// ring (step k reads sets k and k+1, sets k+2 and k+3 in flight): 12 tiles,
// 90 KB at TY = 12, two CTAs per SM.
template <int TYV, typename V>
__device__ __forceinline__ double2 delta_body(const SweepArgs& A, const CUtensorMap* tmv, int s, int tx0,
                                              int ty0, int kb, int ke, double2* ring2, uint64_t* bar,
                                              uint32_t& phase, bool init_bars, double* zih, double* zhd) {
  TEM_TILE_CONSTANTS(TYV);
  constexpr int kW = sizeof(V) / 8;
  constexpr int TSV = TS2 * 2 / kW;
  constexpr int TILE_V = HX * HY * (int)sizeof(V);
  V* ring = reinterpret_cast<V*>(ring2);
  const Grid& g = A.g;
  const int tid = threadIdx.x;
  V acc = VT<V>::zero();
  const Column C = make_column<TYV>(g, tx0, ty0);
  for (int q = tid; q < ke - kb; q += NT) {
    zih[q] = __ldg(g.ih[2] + kb + q);
    zhd[q] = __ldg(g.hdm[2] + kb + q);
  }
  auto issue = [&](int q) {
    const int b = q % R_D;
    mbar_expect_tx(&bar[b], 3 * TILE_V);
    const int cx = kW * (tx0 - 1) + vofs<V>(), cy = ty0 - 1;
#pragma unroll
    for (int c = 0; c < 3; ++c) tma_tile(ring + (b * 3 + c) * TSV, tmv, cx, cy, q, c, s, &bar[b]);
  };
  auto wait_set = [&](int q) {
    const int b = q % R_D;
    mbar_wait(&bar[b], (phase >> b) & 1u);
    phase ^= 1u << b;
  };
  if (tid == 0) {
    if (init_bars) {
      for (int q = 0; q < R_D; ++q) mbar_init(&bar[q], 1);
      fence_barrier_init();
    }
    fence_proxy_async();
  }
  __syncthreads();
  if (tid == 0)
    for (int q = kb; q <= min(kb + 3, ke); ++q) issue(q);
  wait_set(kb);
#pragma unroll 1
  for (int k = kb; k < ke; ++k) {
    wait_set(k + 1);
    const V* S0 = ring + (k % R_D) * 3 * TSV;
    const V* S1 = ring + ((k + 1) % R_D) * 3 * TSV;
    acc = cadd(acc, faces_quad<TYV>(C, zih[k - kb], zhd[k - kb], S0, S1, S0 + TSV, S1 + TSV, S0 + 2 * TSV));
    __syncthreads();   // set k no longer read
    if (tid == 0 && k + 4 <= ke) {
      fence_proxy_async();
      issue(k + 4);
    }
  }
  return VT<V>::cplx(acc);
}

template <bool PRIME, int TYV = kTYSplit>
__global__ void __launch_bounds__(Tile<TYV>::NT, 768 / Tile<TYV>::NT)
    k_delta(const __grid_constant__ SweepArgs A, const __grid_constant__ CUtensorMap tmv,
            const __grid_constant__ CUtensorMap tmvr) {
  constexpr int NT = Tile<TYV>::NT;
  extern __shared__ unsigned char smem_raw[];
  double2* ring = smem_align128(smem_raw);   // [R_D][3] tiles
  __shared__ __align__(8) uint64_t bar[R_D];
  __shared__ double red[3 * NT / 32];
  __shared__ double zih[kMaxChunk];         // ih_z[k]   for k = kb .. ke-1
  __shared__ double zhd[kMaxChunk];         // hdm_z[k]  for k = kb .. ke-1

  int a, tx0, ty0, kb, ke;
  int pidx;
  block_coords<TYV>(A, a, tx0, ty0, kb, ke, pidx);
  const int tid = threadIdx.x;
  const int n_act = A.ctl->n_active, code = A.ctl->list[a & 31];   // one cache line, one round trip
  bool live = a < n_act;
  int s = 0;
  bool real = false, pair = false;
  if (live) {
    s = slot_shift(code);
    live = A.st[s].active != 0;
    real = A.st[s].real != 0;
    if (slot_partner(code) >= 0) {
      pair = true;
      live = live || A.st[slot_partner(code)].active != 0;
    }
  }
  double2 acc = czero();
  uint32_t phase = 0;
  if (live) {
    if (pair)
      acc = delta_body<TYV, dpair>(A, &tmv, s, tx0, ty0, kb, ke, ring, bar, phase, true, zih, zhd);
    else if (real)
      acc = delta_body<TYV, double>(A, &tmvr, s, tx0, ty0, kb, ke, ring, bar, phase, true, zih, zhd);
    else
      acc = delta_body<TYV, double2>(A, &tmv, s, tx0, ty0, kb, ke, ring, bar, phase, true, zih, zhd);
  }
  double rdum = 0.0;
  block_sum_n<NT>(acc, rdum, red);
  if (tid == 0) {
    A.part[7 * A.pstride + pidx] = acc.x;
    A.part[8 * A.pstride + pidx] = acc.y;
  }
  if (!last_block(&A.ctl->ticket[PRIME ? 6 : 5])) return;
  finalize_split<PRIME, TYV>(A, A.nslot, gridDim.x / A.nslot);
}

}  // namespace tem
