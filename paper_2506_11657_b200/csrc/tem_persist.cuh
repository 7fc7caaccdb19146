// tem_persist.cuh -- the split COCG iteration loop as ONE cooperative kernel
// (sm_100a), for grids whose whole COCG state stays in the 126 MB L2.
//
// On such grids (BASELINE configs[0-2]; the paper's own experiment has 81 k
// unknowns) an iteration of the graph path is two kernels
// of a few microseconds each, and launch gaps, pipeline fill and the
// last-CTA reductions dominate.  k_persist keeps one CTA per SM resident
// for many iterations and replaces the kernel boundaries by grid barriers:
//
//   per iteration i (parity q = i & 1), n = active shifts:
//     pass 1  units (slot, tile, z-chunk) of the n active shifts, dealt
//             round-robin to the CTAs: sweep_body<3 | 4> (the same code as
//             k_sweep<3|4>), partials -> part[.][unit]
//     grid barrier
//     pass 2  the same units: delta_body (z^T K z) -> part[7, 8][unit]
//     grid barrier; the LAST CTA to arrive runs finalize_split (alpha,
//             beta, stop test, compacted active list) before releasing it
//
// The z-chunking is re-chosen per active-slot count from a host table
// (latency regime of sweep_geometry: fewest plane steps on the critical
// path), so the last slow shifts spread over every SM.  The arithmetic, the
// partial sums and their fixed reduction order are those of the graph path.
//
// Memory ordering: results are written with generic stores and read by
// other SMs through TMA (async proxy) after a barrier: every CTA fences
// (__threadfence) before arriving, the waiting thread acquires the barrier
// generation and then issues fence.proxy.async.global before its next TMA.
// Mutable state (ShiftState, Control, x) is read through L2 (ld.global.cg),
// never from a possibly stale L1 line.
#pragma once
#include "tem_sweep.cuh"

namespace tem {

constexpr int kMaxSlots = 32;   // TEM_MAX_SHIFTS

struct PersistArgs {
  SweepArgs A;              // grid, tiles, band, mass, x, st, ctl, part (nslot/nzc/kchunk unused)
  double2* Z[2];            // z_i ping-pong (iteration parity)
  double2* P[2];            // p_i ping-pong
  int nzc[kMaxSlots + 1];      // z-chunks for n active slots
  int kchunk[kMaxSlots + 1];   // planes per chunk
  int it0;                  // global index of this launch's first iteration (parity)
  int n_iter;               // iterations at most
  unsigned int* gbar;       // [2]: arrivals, generation
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Arrive at the grid barrier; true (in every thread) in the CTA that
// arrived last -- it runs the serial step and then calls grid_release.
// gen (thread 0 only): the generation this barrier completes.
__device__ __forceinline__ bool grid_arrive(unsigned* gbar, unsigned& gen) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    gen = ld_acquire_u32(gbar + 1);   // cannot advance before this CTA arrives
    __threadfence();
    s_last = atomicAdd(gbar, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  return s_last != 0;
}
__device__ __forceinline__ void grid_release(unsigned* gbar, unsigned gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    gbar[0] = 0;
    __threadfence();
    st_release_u32(gbar + 1, gen + 1);
    fence_proxy_async_global();
  }
  __syncthreads();
}
__device__ __forceinline__ void grid_wait(unsigned* gbar, unsigned gen) {
  if (threadIdx.x == 0) {
    while (ld_acquire_u32(gbar + 1) == gen) __nanosleep(20);
    fence_proxy_async_global();
  }
  __syncthreads();
}
__device__ __forceinline__ void grid_sync(unsigned* gbar) {
  unsigned gen = 0;
  if (grid_arrive(gbar, gen))
    grid_release(gbar, gen);
  else
    grid_wait(gbar, gen);
}

// tmZ*/tmP*: tensor maps of Z[q] / P[q], complex and real (r) layouts.
template <int TYV = kTYSplit>
__global__ void __launch_bounds__(Tile<TYV>::NT, 1)
    k_persist(const __grid_constant__ PersistArgs PA, const __grid_constant__ CUtensorMap tmZ0,
              const __grid_constant__ CUtensorMap tmZ1, const __grid_constant__ CUtensorMap tmP0,
              const __grid_constant__ CUtensorMap tmP1, const __grid_constant__ CUtensorMap tmZ0r,
              const __grid_constant__ CUtensorMap tmZ1r, const __grid_constant__ CUtensorMap tmP0r,
              const __grid_constant__ CUtensorMap tmP1r) {
  constexpr int NT = Tile<TYV>::NT;
  extern __shared__ unsigned char smem_raw[];
  double2* ring = smem_align128(smem_raw);
  __shared__ __align__(8) uint64_t bar_s[R_XY];   // sweep ring
  __shared__ __align__(8) uint64_t bar_d[R_D];    // delta ring
  __shared__ double red[3 * NT / 32];
  __shared__ double zih[kMaxChunk + 1];
  __shared__ double zhd[kMaxChunk];
  const SweepArgs& A = PA.A;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < R_XY; ++q) mbar_init(&bar_s[q], 1);
    for (int q = 0; q < R_D; ++q) mbar_init(&bar_d[q], 1);
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t ph_s = 0, ph_d = 0;   // mbarrier phases, carried across units
  const int tiles = A.ntx * A.nty;
#pragma unroll 1
  for (int i = 0; i < PA.n_iter; ++i) {
    const int par = (PA.it0 + i) & 1;
    const int ns = ld_cg(&A.ctl->n_active);
    if (ns == 0) break;
    const int nzc = PA.nzc[ns], kch = PA.kchunk[ns];
    const int units = tiles * nzc * ns;
    const Bufs B{PA.P[1 - par], PA.Z[1 - par], PA.Z[par], PA.P[par]};
    // ---- pass 1: p_i, z_{i+1} (and x on odd i); partials
#pragma unroll 1
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int a, tx0, ty0, kb, ke, pidx;
      unit_coords<TYV>(A, u, ns, nzc, kch, a, tx0, ty0, kb, ke, pidx);
      const int s = ld_cg(&A.ctl->list[a]);
      const ShiftState st = ld_state(&A.st[s]);
      Partials P{};
      if (st.active) {
        if (par == 0) {
          if (st.real)
            sweep_body<3, TYV, double>(A, &tmP0r, &tmZ0r, s, tx0, ty0, kb, ke, st.s, st.alpha, st.beta,
                                       st.alpha_prev, ring, bar_s, ph_s, false, zih, zhd, P, B);
          else
            sweep_body<3, TYV, double2>(A, &tmP0, &tmZ0, s, tx0, ty0, kb, ke, st.s, st.alpha, st.beta,
                                        st.alpha_prev, ring, bar_s, ph_s, false, zih, zhd, P, B);
        } else {
          if (st.real)
            sweep_body<4, TYV, double>(A, &tmP1r, &tmZ1r, s, tx0, ty0, kb, ke, st.s, st.alpha, st.beta,
                                       st.alpha_prev, ring, bar_s, ph_s, false, zih, zhd, P, B);
          else
            sweep_body<4, TYV, double2>(A, &tmP1, &tmZ1, s, tx0, ty0, kb, ke, st.s, st.alpha, st.beta,
                                        st.alpha_prev, ring, bar_s, ph_s, false, zih, zhd, P, B);
        }
      }
      write_split_partials<NT>(A, P, pidx);
    }
    grid_sync(PA.gbar);
    // ---- pass 2: delta = z_{i+1}^T K z_{i+1}
#pragma unroll 1
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int a, tx0, ty0, kb, ke, pidx;
      unit_coords<TYV>(A, u, ns, nzc, kch, a, tx0, ty0, kb, ke, pidx);
      const int s = ld_cg(&A.ctl->list[a]);
      const int real = ld_cg(&A.st[s].real);
      double2 acc = czero();
      if (par == 0) {
        if (real)
          acc = delta_body<TYV, double>(A, &tmZ1r, s, tx0, ty0, kb, ke, ring, bar_d, ph_d, false, zih, zhd);
        else
          acc = delta_body<TYV, double2>(A, &tmZ1, s, tx0, ty0, kb, ke, ring, bar_d, ph_d, false, zih, zhd);
      } else {
        if (real)
          acc = delta_body<TYV, double>(A, &tmZ0r, s, tx0, ty0, kb, ke, ring, bar_d, ph_d, false, zih, zhd);
        else
          acc = delta_body<TYV, double2>(A, &tmZ0, s, tx0, ty0, kb, ke, ring, bar_d, ph_d, false, zih, zhd);
      }
      double rdum = 0.0;
      block_sum_n<NT>(acc, rdum, red);
      if (tid == 0) {
        A.part[7 * A.pstride + pidx] = acc.x;
        A.part[8 * A.pstride + pidx] = acc.y;
      }
    }
    // ---- scalars: the last CTA to arrive finalises, then releases
    unsigned gen = 0;
    if (grid_arrive(PA.gbar, gen)) {
      finalize_split<false, TYV>(A, ns, tiles * nzc);
      grid_release(PA.gbar, gen);
    } else {
      grid_wait(PA.gbar, gen);
    }
  }
}

}  // namespace tem
