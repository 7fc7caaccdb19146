/*
 * tem_b200.h -- C ABI of the B200-native TEM forward hot path.
 *
 * What it computes (PAPER.md, arxiv 2506.11657):
 *   u(t_j) = exp(-t_j M^-1 K) b,  b = M^-1 f                       (§2.2 eq:expm)
 * approximated by the shared-pole family (§3.2 eq:ratfam) and evaluated as
 *   u(t_j) ~ sum_i w_i Re( alpha_ij (K - xi_i M)^-1 f )              (§3.2 eq:rmj)
 * i.e. one complex-shifted sparse solve (K + s_i M) x_i = f per representative
 * pole (s_i = -xi_i; w_i = 2 for a conjugate-pair representative, 1 for a real
 * pole, footnote to eq:rmj) and the tall-skinny product u = 2 Re(S R) (§3.2).
 *
 * Discretisation (reading R1): the staggered Yee / finite-
 * integration grid = lowest-order Nedelec edge elements on a tensor-product
 * hexahedral grid with lumped masses.  Unknowns are edge line integrals of e;
 *   K = T^T W T,  (T u)_f = circulation of u around face f,
 *   W_f = hdual_f / (mu0 A_f),  mu0 = 4 pi 1e-7  (§2.1);
 *   M_e = (sum_{cells c touching e} sigma_c V_c / 4) / l_e^2;
 *   f_e = +-I on the transmitter's edges.
 * Boundary edges (tangential to the outer surface) are fixed to 0 (eq:bc).
 *
 * LAYOUTS (all fp64; "device" = CUDA global memory of the current device):
 *   Nn = (nx+1)(ny+1)(nz+1) nodes, node(i,j,k) = (k*(ny+1)+j)*(nx+1)+i,
 *   i fastest, z up.  Node (i,j,k) owns edge c (c = 0:x, 1:y, 2:z) from
 *   node (i,j,k) to node (i,j,k)+e_c.
 *   - edge vector  (real):    double[3][Nn]            slot = c*Nn + node
 *   - shift block  (complex): double[S][3][Nn][2]      (re, im) interleaved,
 *                             s*3*Nn + slot (shift-major: one edge vector per
 *                             shift, so a CTA sweeping one shift streams it
 *                             contiguously and converged shifts cost nothing)
 *   - channel fields (real):  double[K][3][Nn]
 *   - conductivity:           double[nz][ny][nx]       cell (i,j,k) at [(k*ny+j)*nx+i]
 *   - complex scalars on the host: double[2*n] (re, im) interleaved
 *   Slots of non-existent edges (node index == n_c along their own axis) and
 *   of boundary edges always hold 0 on output.
 *
 * OWNERSHIP: every pointer is owned by the caller.  Device buffers are
 * caller-allocated (PyTorch in the Python binding); the library allocates
 * only its context (grid spacings, per-shift scalars, reduction scratch, a
 * cached CUDA graph) and, for tem_forward_host, a device workspace cached in
 * the context.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream).  Calls are asynchronous on `stream` unless stated.
 *
 * ERRORS: every call returns 0 on success or a negative TEM_E* code; the
 * message of the last error on the calling thread is tem_last_error().
 * Argument errors are detected before any launch; CUDA errors are reported
 * from the launch that raised them.
 */
#ifndef TEM_B200_H
#define TEM_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TEM_OK 0
#define TEM_EINVAL -1      /* bad argument (sizes, null pointers, S out of range) */
#define TEM_ECUDA -2       /* a CUDA runtime call failed */
#define TEM_ENOMEM -3      /* allocation failed */
#define TEM_ENOCONV -4     /* tem_cocg_solve: a shift did not converge within maxit */
#define TEM_EBREAKDOWN -5  /* tem_cocg_solve: COCG breakdown (p^T A p or r^T z == 0) */

#define TEM_MAX_SHIFTS 32  /* S <= 32 representative poles (degree <= 64) */

typedef struct tem_ctx tem_ctx;

/* Library version string, e.g. "tem_b200 0.1 sm_100a". */
const char* tem_version(void);
/* Message of the last failed call on this thread ("" if none). */
const char* tem_last_error(void);

/* Create a context for an nx x ny x nz cell grid with cell widths hx[nx],
 * hy[ny], hz[nz] (HOST arrays, metres, > 0), on the current CUDA device.
 * Requires nx, ny, nz >= 2 (at least one interior node plane per axis).
 * PAPER.md §2.2 (the space V^h): the grid fixes K entirely. */
int tem_create(int nx, int ny, int nz, const double* hx, const double* hy,
               const double* hz, tem_ctx** out);
void tem_destroy(tem_ctx* ctx);

/* Nn = (nx+1)(ny+1)(nz+1), and the number of free (interior) edges N. */
size_t tem_num_nodes(const tem_ctx* ctx);
size_t tem_num_unknowns(const tem_ctx* ctx);

/* M_e for every edge from the cell conductivity (§2.2 [M]_ij =
 * (sigma Phi_j, Phi_i), lumped; reading R1).  sigma: device double[nz][ny][nx]
 * (> 0); mass: device double[3][Nn] output, 0 on non-free slots. */
int tem_edge_mass(tem_ctx* ctx, const double* sigma, double* mass, void* stream);

/* Matrix-free multi-shift operator, all shifts in one pass:
 *   y[:, s] = (K + shifts[s] M) x[:, s],  s = 0..S-1
 * (§4 "A_i := K - xi_i M", with s = -xi).  x, y: device shift
 * blocks (complex, [S][3][Nn]); mass from tem_edge_mass; shifts: HOST
 * complex[S].  Non-free slots of y are written 0.  x's non-free slots MUST
 * hold 0 (they are the Dirichlet values of eq:bc and enter the stencil of
 * neighbouring free edges). */
int tem_apply_shifted(tem_ctx* ctx, const double* mass, int S, const double* shifts,
                      const double* x, double* y, void* stream);

/* Bytes of device workspace tem_cocg_solve needs for S shifts. */
size_t tem_cocg_workspace_bytes(const tem_ctx* ctx, int S);

/* Batched multi-shift Jacobi-preconditioned COCG (BASELINE north star (3)):
 * solves (K + shifts[s] M) x_s = f for every s at once, each shift with its
 * own COCG scalars and the Jacobi preconditioner D_s = diag(K) + shifts[s] M;
 * the unconjugated bilinear form a^T b is used for the complex-symmetric
 * system.  Shift s stops when ||f - A_s x_s||_2 / ||f||_2 <= tol (recursive
 * residual) or after maxit iterations.
 *   f:      device edge vector (real, [3][Nn]); only free slots are read
 *   x:      device shift block output ([S][3][Nn] complex)
 *   work:   device workspace of >= tem_cocg_workspace_bytes(ctx, S) bytes
 *   iters, relres (HOST, may be NULL): per-shift iteration count and final
 *           recursive relative residual.
 * Returns after the solve has finished (synchronises `stream`).
 * TEM_ENOCONV if some shift did not reach tol (x still holds its iterate).
 * TEM_EINVAL if S * 6 * nodes >= 2^32 (the sweeps index a shift block with
 * unsigned 32-bit element indices; HBM capacity is the tighter limit).
 * Real shifts (imag == 0; footnote to eq:rmj) run in real
 * arithmetic in the split scheme, two to a slot where there are two
 * (readings R14, R16); their x has imaginary part exactly 0. */
int tem_cocg_solve(tem_ctx* ctx, const double* mass, const double* f, int S,
                   const double* shifts, double tol, int maxit, double* x,
                   void* work, size_t work_bytes, int* iters, double* relres,
                   void* stream);

/* Iteration scheme of tem_cocg_solve.  Both are Jacobi-COCG: the same Krylov
 * iterates in exact arithmetic, the same stopping rule, the same outputs.
 *   TEM_SOLVER_SPLIT (default): COCG with the inner product p^T A p of the
 *     step length expanded into three inner products of the previous
 *     iteration (Chronopoulos-Gear arrangement, exact expansion: DESIGN.md
 *     reading R10), so each iteration is ONE full update sweep (p, z and,
 *     every second iteration, x) plus one read-only sweep for z^T A z:
 *     96 B per unknown per shift per iteration.
 *   TEM_SOLVER_TWO_SWEEP: the textbook recursion, alpha = r^T z / p^T A p;
 *     128 B per unknown per shift per iteration.
 * tem_set_solver returns TEM_EINVAL for any other value; tem_get_solver
 * returns the current scheme (TEM_EINVAL for a NULL context). */
#define TEM_SOLVER_SPLIT 0
#define TEM_SOLVER_TWO_SWEEP 1
int tem_set_solver(tem_ctx* ctx, int solver);
int tem_get_solver(const tem_ctx* ctx);

/* How the split scheme's iterations are launched (the same per-element
 * arithmetic; the reduction partials are grouped by each path's own
 * z-chunking, so iterates agree to rounding, not bit for bit):
 *   TEM_LAUNCH_GRAPHS: two kernels per iteration (k_sweep<3|4>, k_delta),
 *     captured as CUDA graphs of 16 iterations -- the bandwidth path;
 *   TEM_LAUNCH_PERSISTENT: one cooperative kernel (one CTA per SM) runs up
 *     to 1024 iterations with grid barriers between the passes and the
 *     per-shift scalar update in the last CTA to arrive -- built for grids
 *     whose COCG state stays in L2 (the paper's own experiment has 81 174
 *     unknowns);
 *   TEM_LAUNCH_AUTO (default): graphs -- measured faster than the persistent
 *     kernel on every BASELINE grid ("Launch paths").
 * The two-sweep scheme always uses graphs.  TEM_EINVAL for other values. */
#define TEM_LAUNCH_AUTO 0
#define TEM_LAUNCH_GRAPHS 1
#define TEM_LAUNCH_PERSISTENT 2
int tem_set_launch_mode(tem_ctx* ctx, int mode);
int tem_get_launch_mode(const tem_ctx* ctx);

/* Statistics of the last tem_cocg_solve on this context. */
typedef struct {
  double loop_ms;             /* GPU time (CUDA events) of init + iteration loop */
  long long kernel_launches;  /* kernels launched by the solve */
  long long shift_iterations; /* sum over shifts of COCG iterations */
  int iterations;             /* max over shifts */
  int grid, block;            /* launch configuration of the sweep kernels */
  int real_shifts;            /* shifts solved in real arithmetic (split scheme) */
  int persistent;             /* 1: the iterations ran in k_persist (TEM_LAUNCH_PERSISTENT) */
} tem_solve_stats;
int tem_last_solve_stats(const tem_ctx* ctx, tem_solve_stats* out);

/* Batched solve with one right-hand side PER SHIFT and per-shift tolerances
 * (the correction solves of tem_forward's refinement, reading R13):
 *   (K + shifts[s] M) x_s = rhs_s,  stop when ||rhs_s - A_s x_s|| / ||rhs_s|| <= tols[s]
 *   rhs:  device shift block (complex, [S][3][Nn]); non-free slots must hold 0.
 *         A shift with rhs_s = 0 does no iteration and returns x_s = 0.
 *   tols: HOST double[S] (> 0).  Other arguments as tem_cocg_solve.
 * A real shift (imag == 0) whose rhs_s is real runs in real arithmetic. */
int tem_cocg_solve_rhs(tem_ctx* ctx, const double* mass, const double* rhs, int S,
                       const double* shifts, const double* tols, int maxit, double* x,
                       void* work, size_t work_bytes, int* iters, double* relres,
                       void* stream);

/* Channel synthesis, the tall-skinny product of §3.2 (eq:rmj):
 *   u[k][slot] = sum_s w_s Re( residues[k*S + s] * x[s][slot] ),
 *   w_s = 2 if is_pair[s] else 1,   k = 0..K-1
 * residues: HOST complex[K][S]; is_pair: HOST int[S]; x: device shift block;
 * u: device double[K][3][Nn] (non-free slots written 0).  Asynchronous: the
 * host arrays are staged through context-owned pinned memory and may be
 * reused on return.  Calls on one context must be issued on one stream. */
int tem_synthesize(tem_ctx* ctx, int S, int K, const double* residues, const int* is_pair,
                   const double* x, double* u, void* stream);

/* Receiver observation (§5): -d_t b_z(r_0, t_k) =
 * e_z . curl e(r_0, t_k) ~ Q^T(r_0) u(t_k).  On the tensor grid (DESIGN.md
 * reading R12) e_z . curl e is constant on each z-normal face: the
 * circulation of u around the face divided by its area hx_i hy_j.
 *   u:          device channel fields double[K][3][Nn] (tem_synthesize)
 *   receivers:  HOST int[R][3], the lower-corner node (i, j, k) of the face
 *               holding each receiver (0 <= i < nx, 0 <= j < ny, 0 <= k <= nz;
 *               receivers on the surface: k = the air-earth node plane)
 *   out:        device double[K][R]
 * TEM_EINVAL for a receiver outside the grid.  Asynchronous (as
 * tem_synthesize). */
int tem_curl_z(tem_ctx* ctx, int K, const double* u, int R, const int* receivers,
               double* out, void* stream);

/* Residual of the shifted systems in double-double arithmetic, rounded to
 * fp64 (reading R13): r_s = f - (K + shifts[s] M) x_s on every free
 * edge, 0 elsewhere.  The face weights are the fp64 products the sweeps use,
 * so K is the operator tem_cocg_solve iterates with; sums and products are
 * carried to ~1e-32 relative, so r is accurate even when it is 1e-16 of the
 * terms that cancel in it.  f: device real edge vector; x, r: device shift
 * blocks (must not alias); rnorm: HOST double[S] (may be NULL) receives
 * ||r_s||_2 (then the call synchronises `stream`). */
int tem_residual(tem_ctx* ctx, const double* mass, const double* f, int S, const double* shifts,
                 const double* x, double* r, double* rnorm, void* stream);

/* The forward of the north star in one call: all shifted solves, channel
 * synthesis, and -- with max_refine > 0 -- iterative refinement until the
 * channels are converged (reading R13):
 *   x_s <- COCG(f) to tol;  u = synthesis(x);  then per round, for the shifts
 *   still refined: r_s = f - (K + s M) x_s in double-double arithmetic,
 *   d_s = COCG(r_s) to refine_tol (relative to ||r_s||), x_s += d_s.
 * Per-shift targets (split scheme): the first solve snapshots each shift's x
 * when its residual first reaches 10 tol; the change of x_s from there to the
 * end, scaled by the residual ratio and safety, estimates the error E_s left
 * in x_s as max_k ||w_s Re(alpha_ks dx_s)||_M / ||u_k||_M.  Shift s is asked
 * for the reduction channel_tol / (4 S E_s), at least refine_tol, and a shift
 * whose target is >= 1/2 is not refined.
 * Channel-aware stopping: after a round, shift s's contraction is
 * c_s = min(1, safety * max(eta_s, (||r_s after|| - floor_s) / ||r_s before||))
 * -- eta_s the reduction its correction solve achieved, floor_s =
 * 2^-52 || |K + s M| |x_s| || the part of the residual explained by the
 * rounding of x_s itself, safety an allowance for the error-to-residual
 * amplification -- and the error left
 * in channel k is estimated as ||sum_s w_s c_s Re(alpha_ks d_s)||_M / ||u_k||_M
 * -- the round's corrections scaled by their contractions and synthesised
 * with the cancellation of eq:rmj (the M-norm of the paper's bound,
 * P:210-217).  The first round asks every shift for a residual reduction of
 * refine_tol; while some channel's estimate exceeds channel_tol, the shifts
 * whose own correction could still matter are refined again, asked for the
 * reduction that brings the estimate to half the target.  The loop ends
 * when every channel's estimate is <= channel_tol (or after max_refine
 * rounds).  u is re-synthesised from the refined x. */
typedef struct {
  double tol;          /* COCG tolerance of the first solve (relative residual), e.g. 1e-10 */
  int maxit;           /* COCG iterations per solve, at most */
  int max_refine;      /* refinement rounds at most (0: plain solve + synthesis) */
  double refine_tol;   /* residual reduction asked of each correction solve, in (0, 1) */
  double channel_tol;  /* target: estimated relative M-norm error of every channel */
  double safety;       /* >= 1: error-to-residual amplification allowance of the estimate */
} tem_forward_opts;
typedef struct {
  int refine_rounds;                   /* rounds run */
  long long shift_iterations;          /* COCG shift-iterations of all solves */
  long long initial_shift_iterations;  /* of the first solve */
  double loop_ms;                      /* GPU time of all COCG solves */
  double channel_bound;                /* max_k of the final estimate (-1: no refinement) */
  double relres_max;                   /* max_s final relative residual (double-double if refined) */
  long long kernel_launches;           /* kernels launched (solves, synthesis, refinement) */
} tem_forward_stats;
/* tol 1e-10, maxit 200000, max_refine 0, refine_tol 1e-4, channel_tol 1e-7, safety 1.5 */
void tem_forward_default_opts(tem_forward_opts* opts);
size_t tem_forward_workspace_bytes(const tem_ctx* ctx, int S, int K);
/*   mass, f: device (tem_edge_mass; real edge vector); shifts, residues
 *   ([K][S]), is_pair: HOST as tem_synthesize; x: device shift block out;
 *   u: device double[K][3][Nn] out; work: >= tem_forward_workspace_bytes.
 *   iters (HOST, may be NULL): COCG iterations per shift over all solves;
 *   relres (HOST, may be NULL): final relative residual per shift
 *   (double-double evaluation when refined); fst (HOST, may be NULL).
 * Synchronises `stream`.  Same error codes as tem_cocg_solve (ENOCONV if a
 * solve did not converge; x and u still hold the iterate). */
int tem_forward(tem_ctx* ctx, const double* mass, const double* f, int S, const double* shifts,
                int K, const double* residues, const int* is_pair, const tem_forward_opts* opts,
                double* x, double* u, void* work, size_t work_bytes, int* iters,
                double* relres, tem_forward_stats* fst, void* stream);
int tem_last_forward_stats(const tem_ctx* ctx, tem_forward_stats* out);

/* End-to-end forward with HOST buffers: uploads sigma and f, computes the
 * mass, runs tem_forward with `opts` and downloads u (HOST double[K][3][Nn]).
 * Device memory comes from a workspace cached in the context.  Synchronous.
 * Same error codes as tem_forward. */
int tem_forward_host(tem_ctx* ctx, const double* sigma, const double* f, int S,
                     const double* shifts, int K, const double* residues,
                     const int* is_pair, const tem_forward_opts* opts, double* u,
                     int* iters, double* relres);

/* Host-side construction of the shared-pole family, computed once before the
 * solves (§3.2 eq:ratfam, RKFIT objective eq:rkfit with a diagonal
 * surrogate of dense eigenvalues on [0, inf) and v = 1; R3-R5).
 *   K, t:       HOST double[K], time channels in seconds (> 0)
 *   w:          HOST double[K] weights w_j of eq:rkfit, or NULL for unit weights
 *   m:          degree m-hat (2..64); iters: relocation sweeps (<= 0: 12)
 * Outputs (HOST, caller-allocated for the worst case n_rep = m):
 *   n_rep:      number of shifted systems (one per conjugate pair + one per real pole)
 *   shifts:     complex[m]: s_i = -xi_i / t_max (1/s), the shifts of tem_cocg_solve
 *   residues:   complex[m][K]: alpha_ij / t_max, row i = representative pole i
 *   is_pair:    int[m]: 1 if pole i stands for a conjugate pair (weight 2 in eq:rmj)
 *   uniform_error: (may be NULL) eq:uniform_error estimated on a log grid.
 * Deterministic; CPU only; TEM_EINVAL on bad arguments, and when the family
 * would need more than TEM_MAX_SHIFTS systems (m near 64 with real poles). */
int tem_fit_family(int K, const double* t, const double* w, int m, int iters, int* n_rep,
                   double* shifts, double* residues, int* is_pair, double* uniform_error);

#ifdef __cplusplus
}
#endif
#endif /* TEM_B200_H */
