/* liblsb200 -- B200 (sm_100a) kernels for the Arnoldi orthogonalization hot
 * path of low-synchronization GMRES(m) (arXiv 1809.05805).
 *
 * C ABI only: plain pointers (device memory unless stated), 64-bit sizes,
 * an opaque CUDA stream, an int status.  No torch or C++ types cross this
 * boundary; the Python host layer (paper_1809_05805_b200/_abi.py) binds it
 * with ctypes.  The reference package `lowsync` is pure numpy and has no
 * FFI of its own; each entry point names the reference function (file:line
 * under /root/reference/pkg/src/lowsync) whose arithmetic it replaces.
 *
 * Storage conventions
 *   Krylov basis V : column j at V + j*ld (each column contiguous, like the
 *                    reference's Fortran-order KrylovBasis, kernels.py:219);
 *                    V and ld must be 16-byte aligned / even.
 *   small matrices : R, T, L are cap x cap row-major; tri is (m+1) x m
 *                    row-major; rot holds (c, s) pairs.
 *   reductions     : deterministic -- per-CTA partials, then a fixed-order
 *                    sum by the last CTA; bitwise reproducible run to run.
 *   gating         : every cycle kernel takes (flags, it); once the solver
 *                    has stopped at iteration d (flags->stop_iter == d), a
 *                    kernel of iteration it > d returns immediately, so a
 *                    whole restart cycle runs as one CUDA graph without host
 *                    syncs.  Pass flags == NULL for ungated calls.
 *
 * All functions return 0 on success, LSB_E* otherwise.
 */
#ifndef LSB200_H
#define LSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSB_OK 0
#define LSB_EINVAL 1      /* bad sizes / alignment                          */
#define LSB_ECUDA 2       /* CUDA launch error (see lsb_last_error)         */
#define LSB_ERANGE 3      /* p above the kernel's column limit              */

/* status codes written to lsb_flags.status (mirrors gmres.py:58-61) */
#define LSB_RUNNING 0
#define LSB_CONVERGED 1          /* implicit residual <= target          */
#define LSB_BREAKDOWN 2          /* HappyBreakdown inside the cycle      */
#define LSB_STARTUP_BREAKDOWN 3  /* HappyBreakdown outside a solver loop */
#define LSB_SINGULAR 4           /* SingularHessenberg in back-subst.    */
#define LSB_GHYSELS_CHECK 5      /* cgs1_ghysels radicand lost its digits */

#define LSB_NO_STOP 0x7fffffff

/* Device-resident control block of one solve (one per rank). */
typedef struct lsb_flags {
  int32_t stop_iter;   /* LSB_NO_STOP while running; else last iteration   */
  int32_t status;      /* LSB_RUNNING / LSB_CONVERGED / ...                 */
  int32_t broke_iter;  /* iteration whose orthogonalization broke down, -1  */
  int32_t k;           /* columns consumed by the cycle's least squares     */
  int32_t nonfinite;   /* spmv produced NaN/Inf (kernels.py:271)            */
  int32_t restart_ok;  /* restart residual already <= target               */
  int32_t comm_error;  /* LSB_COMM_TIMEOUT: a peer exchange timed out        */
  int32_t pad;
} lsb_flags;

/* slots of the device scalar block `scal` */
#define LSB_S_BETA 0      /* deferred norm / r_diag of the current column   */
#define LSB_S_TARGET 1    /* rel_tol * beta0 (gmres.py:479)                 */
#define LSB_S_DENOM 2     /* beta0 or 1 (gmres.py:474)                      */
#define LSB_S_RNORM 3     /* last true residual norm ||b - A x||            */
#define LSB_S_RELTOL 4
#define LSB_S_BTF 5       /* breakdown_tol_factor                           */
#define LSB_S_AMAX 6      /* norm pass scratch                              */
#define LSB_S_SSQ 7
#define LSB_S_TOL 8       /* last breakdown tolerance (for HappyBreakdown)  */
#define LSB_S_RAD 9       /* cgs1_ghysels radicand ||z||^2 - ||y||^2        */
#define LSB_S_COUNT 16

/* Reduction workspace: partial >= lsb_partial_len() doubles, counter >= 8
 * zero-initialised uint32 (self-resetting), grid 0 = library default. */
typedef struct lsb_workspace {
  double* partial;
  uint32_t* counter;
  int32_t grid;
  int32_t pad;
} lsb_workspace;

/* CSR matrix with 32-bit indices (the reference keeps int64,
 * kernels.py:113-115; nnz < 2^31 here).  col_scale (optional) is a right
 * Jacobi scaling applied to x before the products (gmres.py:121-126). */
typedef struct lsb_csr {
  int64_t n_rows, n_cols, nnz;
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const double* values;
  const double* col_scale;
  int64_t row0;          /* global index of local row 0 (row-block partition) */
  int64_t x_lo;          /* x is indexed by (global col - x_lo)               */
} lsb_csr;

/* Dictionary-coded CSR: the same matrix as an lsb_csr whose values take at
 * most 256 distinct bit patterns and whose column offsets (global col -
 * global row) take at most 256 distinct values.  Entry j of row r:
 * value = val_tab[val_idx[j]], column = row0 + r + off_tab[off_idx[j]].
 * 2 bytes per nonzero instead of 12 (the CSR-VI / CSR-DU idea). */
typedef struct lsb_csr_dict {
  int64_t n_rows, n_cols, nnz;
  const int32_t* row_ptr;
  const uint8_t* val_idx;
  const uint8_t* off_idx;
  const double* val_tab;   /* n_val entries */
  const int32_t* off_tab;  /* n_off entries */
  int32_t n_val, n_off;
  const double* col_scale;
  int64_t row0;
  int64_t x_lo;
} lsb_csr_dict;

/* Constant-coefficient box stencil, row i = (iz*ny + iy)*nx + ix.
 * Offsets MUST be listed in increasing linear offset (= CSR column order).
 * halo_lo/halo_hi: 1 if x holds a ghost z-plane below/above the local slab
 * at x[-nx*ny .. 0) / x[n .. n+nx*ny) (z-slab row partition), else the
 * plane is a Dirichlet boundary. */
#define LSB_MAX_OFF 27
typedef struct lsb_stencil {
  int32_t nx, ny, nz;
  int32_t noff;
  int32_t halo_lo, halo_hi;
  int32_t dx[LSB_MAX_OFF], dy[LSB_MAX_OFF], dz[LSB_MAX_OFF];
  double val[LSB_MAX_OFF];
  const double* col_scale;   /* optional Jacobi scaling, same layout as x */
} lsb_stencil;

/* Everything one Arnoldi cycle touches (one rank). */
typedef struct lsb_arnoldi {
  double* V;            /* basis, cap columns of stride ld                 */
  int64_t ld, n;        /* local rows                                      */
  int64_t n_global;     /* global rows (breakdown tolerance uses sqrt(n))  */
  int32_t cap, m;       /* basis capacity, restart length                  */
  double* R;            /* cap*cap: R (upper); its columns hold Hbar       */
  double* T;            /* cap*cap: compact-WY factor (mgs_lvl2)           */
  double* L;            /* cap*cap: strictly lower Q^T Q (cgs2_lvl2)        */
  double* rot;          /* 2*m Givens (c, s)                               */
  double* g;            /* m+1 rotated rhs                                 */
  double* tri;          /* (m+1)*m rotated triangle                        */
  double* coef;         /* cap: projection coefficients c / r / h          */
  double* coef2;        /* cap: second-pass s / least-squares y            */
  double* G;            /* reduction result(s), see g_parts                */
  int32_t g_parts;      /* number of rank partials stacked in G (1 = local) */
  int32_t g_stride;     /* doubles between two rank partials               */
  double* Gloc;         /* where this rank's local reduction is written    */
  double* scal;         /* LSB_S_COUNT scalars                             */
  double* res;          /* m+1 implicit residual norms |g[i]|              */
  lsb_flags* flags;
  lsb_workspace ws;
} lsb_arnoldi;

/* ---------------------------------------------------------------- tuning */
#define LSB_TUNE_FUSED_OCC3 1   /* fused K1+SpMV: 0 auto (p<=40), 1 on, 2 off */
#define LSB_TUNE_FORCE_PARTS 2  /* K1 row parts per tile column (1/2/4/8), 0 auto */
#define LSB_TUNE_ROW_CTAS_PER_SM 3 /* row-parallel kernels: persistent CTAs/SM, 0 auto */
#define LSB_TUNE_K3_ROWS 4      /* lagged_update_reduce tile rows 64/128/256, 0 auto */
#define LSB_TUNE_K3_STAGES 5    /* lagged_update_reduce ring stages cap (>= 2), 0 auto */
#define LSB_TUNE_CSR_THREAD_ROW 6 /* CSR SpMV: 0 warp-staged (default), 1 thread per row, 2 warp-staged 8 loads/lane at 3 CTAs/SM */
#define LSB_TUNE_PERSIST_TRACE 7  /* 1: lsb_cycle_persistent records phase timestamps */
#define LSB_TUNE_PERSIST_CTAS 8   /* lsb_cycle_persistent cluster size 1..16, 0 auto */
#define LSB_TUNE_FUSED_PIPE 9     /* fused K1+SpMV pipelined stencil: 0 auto (2-4 items/warp), 1 up to 8, 2 off */
#define LSB_TUNE_CSR_DICT 10      /* dictionary-coded CSR: 0 thread per row, 1 warp-staged index bytes */
#define LSB_TUNE_PDL 11           /* programmatic dependent launch of the per-iteration chains (one-sync K1/K5/K2, two-sync K5a/K3/K5b/K4 while p <= 32, lsb_mdot): 0 auto (n < 2^23), 1 on, 2 off */
#define LSB_TUNE_PERSIST_TIMEOUT_S 12  /* persistent cycle: a cluster handoff waits at most this many seconds (0: 30, < 0: unbounded), then marks the mapped report -1.0 and aborts */
#define LSB_TUNE_GRID_OCC 13       /* grid cycle CTAs per SM (0: 1) */
#define LSB_TUNE_GRID_TRACE 14     /* 1: lsb_cycle_grid accumulates per-phase ns (lsb_grid_trace) */
#define LSB_TUNE_S27_MARCH 15      /* 27-point stencil: 0 auto (TMA plane-tile kernel from 2^21 rows, else
                                     row pairs), 2 row-pair kernel, 3 z-marching without its interior fast
                                     path, 4 z-marching (nz >= 32), 5 plane-tile kernel at any size */
#define LSB_TUNE_MGS1_GRID 16     /* lsb_mgs1_passes: 0 cooperative single launch when it fits, 2 per-pass launches */
#define LSB_TUNE_S27_TILE_Z 17    /* 27-point plane-tile kernel: planes per CTA (0: 32) */
#define LSB_TUNE_COUNT 18
/* Set / read a kernel-variant knob (performance only; results unchanged up
 * to the reduction tree of the affected kernel). Returns the old value. */
int lsb_set_tuning(int32_t key, int32_t value);

/* ---------------------------------------------------------------- info */
const char* lsb_version(void);
const char* lsb_last_error(void);
int lsb_sm_count(void);
int64_t lsb_partial_len(int32_t pmax);   /* doubles for lsb_workspace.partial */
int32_t lsb_max_columns(void);           /* largest p one mdot launch takes   */

/* ---------------------------------------------------------------- primitives
 * (kernels.py:256-362)                                                     */

/* y = A x (or y = b - A x when b != NULL), rows summed exactly as
 * numpy add.reduceat (kernels.py:256-272): first product + pairwise(rest).
 * Sets flags->nonfinite on NaN/Inf. */
int lsb_spmv_csr(const lsb_csr* A, const double* x, const double* b, double* y,
                 lsb_flags* flags, int32_t it, void* stream);
/* y = A x (b == NULL) or y = b - A x for a dictionary-coded CSR; bitwise
 * lsb_spmv_csr on the equivalent lsb_csr (same products, same numpy
 * reduceat summation order).  Replaces the same kernels.py:256-272 call. */
int lsb_spmv_csr_dict(const lsb_csr_dict* A, const double* x, const double* b, double* y,
                      lsb_flags* flags, int32_t it, void* stream);
/* Matrix-free constant-coefficient stencil (the CSR a StencilMatrix stands
 * for, kernels.py:256-272; bitwise lsb_spmv_csr on it).  x points at local
 * plane 0; with halo_lo / halo_hi the ghost planes x - nx*ny and
 * x + nz*nx*ny must be readable.  The 27-point box from 2^21 rows runs as
 * TMA plane tiles (cp.async.bulk.tensor via cuTensorMapEncodeTiled from the
 * driver entry point; LSB_TUNE_S27_MARCH picks the other kernels). */
int lsb_spmv_stencil(const lsb_stencil* S, const double* x, const double* b, double* y,
                     lsb_flags* flags, int32_t it, void* stream);

/* out = [X^T u, X^T w] as p x 2 row-major (w != NULL; mdot_pair,
 * kernels.py:328-347) or out = X^T u (w == NULL; mass_inner_product /
 * fused_mdot_norm / dot, kernels.py:275-325).  One pass over X. */
int lsb_mdot(const double* X, int64_t ld, int64_t n, int32_t p, const double* u,
             const double* w, double* out, const lsb_workspace* ws,
             const lsb_flags* flags, int32_t it, void* stream);

/* out = y + X alpha (maxpy, kernels.py:350-362); out may alias y.
 * alpha_sign = -1 applies -alpha (cgs_iterated, gram_schmidt.py:138). */
int lsb_maxpy(const double* y, const double* X, int64_t ld, int64_t n, int32_t p,
              const double* alpha, int32_t alpha_sign, double* out,
              const lsb_flags* flags, int32_t it, void* stream);

/* out2[0] = max|x|, out2[1] = sum x^2 (local, deterministic). */
int lsb_norm_partial(const double* x, int64_t n, double* out2, const lsb_workspace* ws,
                     const lsb_flags* flags, int32_t it, void* stream);
/* *out = ||x||_2 from nparts (amax, ssq) pairs stacked part_stride doubles
 * apart; if max|x| is outside [2^-450, 2^450] it re-reads x with an exact
 * power-of-two scaling (local only, nparts == 1) -- the overflow-safe
 * contract of norm2 (kernels.py:283-298). */
int lsb_norm_finish(const double* parts, int32_t nparts, int32_t part_stride, const double* x,
                    int64_t n, double* out, const lsb_workspace* ws, const lsb_flags* flags,
                    int32_t it, void* stream);

/* Row-partitioned norm across ranks, overflow-safe (the rescaled pass of
 * kernels.py:113-119 with an exact power-of-two scale): after the (amax,
 * ssq) parts of every rank are gathered, lsb_norm_scaled_partial writes
 * this rank's sum of (x * 2^-e)^2 into out2[0] (e from the GLOBAL amax; 0
 * when max|x| lies in [2^-450, 2^450]); after those are gathered too,
 * lsb_norm_finish_scaled writes ||x|| -- sqrt(sum ssq) in range, else
 * sqrt(sum scaled) * 2^e.  Same value on every rank. */
int lsb_norm_scaled_partial(const double* parts, int32_t nparts, int32_t part_stride,
                            const double* x, int64_t n, double* out2, const lsb_workspace* ws,
                            void* stream);
int lsb_norm_finish_scaled(const double* parts, const double* parts2, int32_t nparts,
                           int32_t part_stride, int32_t part2_stride, double* out, void* stream);

/* out = x / (*s) elementwise (device scalar s; e.g. V.push(r / beta)). */
int lsb_scale_div(const double* x, int64_t n, const double* s, double* out,
                  const lsb_flags* flags, int32_t it, void* stream);

/* ---------------------------------------------------------------- lagged kernels
 * mgs_lvl2 (gram_schmidt.py:206-245) = lagged_reduce + mgs_lvl2_small +
 * lagged_update; cgs2_lvl2 (gram_schmidt.py:248-280) = lagged_reduce +
 * cgs2_lvl2_small_a + lagged_update + mdot(second pass) + cgs2_lvl2_small_b
 * + lagged_correct.  `p` = j-1 columns in Q; u = V[:,p-1], w = V[:,p].   */

/* Gloc = [Q^T u, Q^T w] (p x 2): _lagged_reduce (gram_schmidt.py:195-203). */
int lsb_lagged_reduce(const lsb_arnoldi* S, int32_t it, int32_t p, void* stream);

/* Fused V[:,p] = A V[:,p-1] (7-point stencil in laplace3d's canonical
 * column order, bitwise = spmv, kernels.py:256-272) and Gloc = [Q^T u, Q^T w]
 * in one pass: the `V.push(_op(V.column(i)))` + `_lagged_reduce` pair of
 * gmres.py:411-414.  Ghost planes (multi-rank) must already be in place. */
int lsb_lagged_reduce_spmv7(const lsb_arnoldi* S, const lsb_stencil* A, int32_t it, int32_t p,
                            void* stream);
/* The same plus (max|w|, sum w^2) in Gloc[2p], Gloc[2p+1] (norm_partial's
 * per-row update, fixed-order CTA tree): fused_mdot_norm (kernels.py:315-325)
 * of the cgs1_ghysels step with its SpMV, u = v_{i-1}. */
int lsb_lagged_reduce_spmv7_norm(const lsb_arnoldi* S, const lsb_stencil* A, int32_t it, int32_t p,
                            void* stream);

/* Small-state update of the one-reduce MGS-CWY kernel: beta, breakdown test,
 * R/T columns, c = T^T y (/beta).  givens_col > 0 also folds Hessenberg
 * column givens_col-1 = R[0..givens_col, givens_col] into the Givens state
 * and tests convergence (gmres.py:418-435); givens_col < 0 defers that fold
 * to lsb_settle (pipeline2 schedule, gmres.py:444-462). */
int lsb_mgs_lvl2_small(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                       int32_t givens_col, void* stream);
/* Deferred Givens fold + convergence test of Hessenberg column col-1
 * (settle, gmres.py:427-435), for a small-state call made with
 * givens_col = -col; runs on a side stream in the pipeline2 schedule. */
int lsb_settle(const lsb_arnoldi* S, int32_t it, int32_t col, void* stream);

/* One whole lagged one-sync restart cycle (iterations 0..m of
 * gmres.py:389-466 with mgs_lvl2, gram_schmidt.py:206-245: SpMV, fused
 * reduction, K5 small state, K2 update) in ONE launch of one thread-block
 * cluster (<= 16 CTAs, distributed-shared-memory reduction, cluster
 * barriers) for launch-bound sizes.  A is the operator as CSR (a stencil's
 * CSR gives the same bits).  Call between lsb_cycle_begin and
 * lsb_cycle_lsq in place of the per-iteration kernels.  Every CTA keeps its
 * rows of all cap basis columns in shared memory: LSB_ERANGE when they do
 * not fit (lsb_cycle_persistent_fits) or the state is multi-rank. */
int lsb_cycle_persistent(const lsb_arnoldi* S, const lsb_csr* A, int32_t krylov_scale,
                         void* stream);
/* Whole restarted solve in one cluster launch: cycles (iterations as
 * lsb_cycle_persistent) each followed on the device by the cycle
 * epilogue -- least squares (lsb_cycle_lsq), x += M^-1 V y
 * (lsb_cycle_extract), r = b - A x, ||r|| (lsb_norm_partial/finish),
 * restart test (lsb_restart_check) -- and, unless the cycle stopped, the
 * next prologue (V[:,0] = r/||r||, lsb_cycle_begin).  Call after the host
 * prologue and the first lsb_scale_div + lsb_cycle_begin.  x (local rows,
 * updated in place) and b are device vectors; log receives, per cycle run,
 * m + 22 doubles: the 8 flag ints (4 doubles' bytes), res[0..m], the
 * LSB_S_COUNT scalars, then a marker written last behind a system fence:
 * 2.0 when another cycle follows, 1.0 for the last one (unwritten reports
 * stay as the caller left them).  log may be mapped pinned host memory:
 * the host can then consume each report while later cycles run.  The
 * cycles stop exactly where the host restart shell would
 * (gmres.py:470-516). */
int lsb_solve_persistent(const lsb_arnoldi* S, const lsb_csr* A, int32_t krylov_scale, double* x,
                         const double* b, double* log, int32_t max_cycles, void* stream);
/* 1 if an n-row, cap-column cycle fits one cluster's shared memory
 * (n * cap <= ~450K doubles, cap <= 128), else 0.  No device needed. */
int lsb_cycle_persistent_fits(int64_t n, int32_t cap);
/* Iterations 0..m of a one-sync cycle (as lsb_cycle_persistent) in one
 * cooperative launch over every SM, for bases too large for one cluster but
 * small enough that the per-iteration kernels are latency-bound
 * (lsb_cycle_grid_fits: n * cap <= 2^23 doubles): SpMV, partial dots,
 * their fixed-order sum, K5 on CTA 0 and K2 separated by grid barriers.
 * part: reduction scratch of part_len >= 2 * cap * (2 * SMs) doubles. */
int lsb_cycle_grid(const lsb_arnoldi* S, const lsb_csr* A, int32_t krylov_scale, double* part,
                   int64_t part_len, void* stream);
int lsb_cycle_grid_fits(int64_t n, int32_t cap);
/* Diagnostics: ns per phase summed over traced grid-cycle iterations
 * (SpMV, barrier, dots, barrier + sums, K5, barrier, K2, barrier); reads and
 * clears (LSB_TUNE_GRID_TRACE = 1 to record). */
int lsb_grid_trace(int64_t* out, int32_t count);
/* Diagnostics: the last traced persistent cycle's phase timestamps (6 per
 * iteration, globaltimer ns; LSB_TUNE_PERSIST_TRACE = 1 to record). */
int lsb_persist_trace(int64_t* out, int32_t count);
/* cgs2_lvl2 front: beta, breakdown, L row, r = (I - L - L^T) y (/beta). */
int lsb_cgs2_lvl2_small_a(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                          int32_t givens_col, void* stream);
/* cgs2_lvl2 back: s = sum of rank partials in G, R[:p,p] = r + s. */
int lsb_cgs2_lvl2_small_b(const lsb_arnoldi* S, int32_t it, int32_t p, void* stream);

/* u <- u/beta; w <- (krylov_scale ? w/beta : w) - Q coef  (one pass). */
int lsb_lagged_update(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                      void* stream);
/* Two-sync first projection fused with the second reduction
 * (gram_schmidt.py:273-276: w -= Q r; s = mass_inner_product(Q, w)):
 * lsb_lagged_update, then Gloc[0..p) = Q^T w with Q = V[:, :p], reading Q
 * once.  u and w are bitwise those of lsb_lagged_update.  LSB_ERANGE when
 * p + 1 > 110 (use lsb_lagged_update + lsb_mdot). */
int lsb_lagged_update_reduce(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                             void* stream);
/* w <- w - Q coef2 (cgs2_lvl2 second projection, gram_schmidt.py:277). */
int lsb_lagged_correct(const lsb_arnoldi* S, int32_t it, int32_t p, void* stream);

/* ---------------------------------------------------------------- direct kernels
 * mgs_level1 (gram_schmidt.py:144-160) and cgs_iterated (118-141) acting in
 * place on column `col` of V against Q = V[:, :p]. */

/* Level-1 MGS pass k (0 <= k <= p): if k > 0, h_{k-1} = sum of rank
 * partials in G -> coef[k-1] and z -= h_{k-1} q_{k-1} (two roundings, as
 * numpy's `work -= h * q`); then if k < p, Gloc[0] = q_k . z, else
 * Gloc[0..1] = (max|z|, sum z^2).  One pass over z. */
int lsb_mgs1_pass(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t k, int32_t p,
                  void* stream);
/* All passes k = 0..p of lsb_mgs1_pass for one rank alone (g_parts == 1 and
 * G == Gloc, else LSB_EINVAL): the whole level-1 MGS of column col
 * (gram_schmidt.py:154-158) as one cooperative launch with a grid barrier
 * between passes (bitwise the per-pass results), or p + 1 chained per-pass
 * launches when the grid cannot be co-resident. */
int lsb_mgs1_passes(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p, void* stream);
/* Sum the p rank partials in G into coef (accumulate != 0: coef += s, and
 * coef2 = s) -- the r_col bookkeeping of cgs_iterated. */
int lsb_collect_coef(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t accumulate,
                     void* stream);
/* lsb_collect_coef (accumulate 0) from the odd entries of an interleaved
 * [Q^T u, Q^T w] reduction: the direct methods' first pass when the SpMV
 * z = A v_{i-1} is fused into it (lsb_lagged_reduce_spmv7 with u = v_{i-1},
 * the last column of Q = V[:, :i]). */
int lsb_collect_coef_pairs(const lsb_arnoldi* S, int32_t it, int32_t p, void* stream);
/* z <- z + Q (-coef2) and, when want_norm == 1, Gloc[0..1] = (max|z|,
 * sum z^2); want_norm == 2: then z /= scal[BETA] unless flags->broke_iter ==
 * it (lsb_direct_normalize fused, bitwise the same). */
int lsb_cgs_project(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p,
                    int32_t want_norm, void* stream);
/* cgs_iterated's first projection fused with the second pass's reduction
 * (gram_schmidt.py:136-138 then 131-133): z <- z - Q coef2 (bitwise equal to
 * lsb_cgs_project), then Gloc[0..p) = Q^T z, reading Q once.  z must be
 * column p (col == p); LSB_ERANGE when p + 1 > 110. */
int lsb_cgs_project_reduce(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p,
                           void* stream);
/* r_diag from the (amax, ssq) rank partials in G; breakdown test against
 * coef[0..p); Hbar column (R[:, col]); Givens fold of column col-1;
 * convergence. */
int lsb_direct_small(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p, void* stream);
/* cgs1_ghysels small state (gmres.py:325-360): G = [Q^T z (p), max|z|,
 * sum z^2] -> y, h = sqrt(||z||^2 - y.y), Hbar column, Givens fold; stops the
 * cycle with LSB_GHYSELS_CHECK when the radicand cancels. */
int lsb_ghysels_small(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p, void* stream);
/* The same with G = [v.q_0, z.q_0, v.q_1, z.q_1, ..., max|z|, sum z^2] (the
 * pair layout lsb_lagged_reduce_spmv7 writes with u = v_{col-1}; y_j = G[2j+1],
 * norm pair at G[2p], G[2p+1]): the SpMV of the Ghysels step fused into its
 * reduction. */
int lsb_ghysels_small_pairs(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p,
                            void* stream);
/* V[:, col] /= r_diag unless the column broke down. */
int lsb_direct_normalize(const lsb_arnoldi* S, int32_t it, int32_t col, void* stream);

/* ---------------------------------------------------------------- cycle control */
/* Zero R/T/L/rot/tri/g, g[0] = scal[RNORM], flags -> running (gmres.py:392-395). */
int lsb_cycle_begin(const lsb_arnoldi* S, void* stream);
/* y = back-substitution of the rotated k x k triangle into coef2, k from
 * flags (solve_least_squares, gmres.py:184-192). */
int lsb_cycle_lsq(const lsb_arnoldi* S, void* stream);
/* x <- x + Mi (V_k y)   (_extract, gmres.py:294-297); col_scale optional. */
int lsb_cycle_extract(const lsb_arnoldi* S, double* x, const double* col_scale, void* stream);
/* True-residual probe of iteration `it` (true_residual_every,
 * gmres.py:273-283): y = back-substitution of the first `it` rotated
 * columns; xt = x + Mi (V_it y).  The caller then forms ||b - A xt||. */
int lsb_trial_lsq(const lsb_arnoldi* S, int32_t it, double* y, void* stream);
int lsb_trial_combine(const lsb_arnoldi* S, int32_t it, const double* x, const double* y,
                      double* xt, const double* col_scale, void* stream);
/* After the restart residual norm landed in scal[RNORM]:
 * first != 0 : denom/target set from it (gmres.py:472-479);
 * always     : flags->restart_ok = rnorm <= target. */
int lsb_restart_check(const lsb_arnoldi* S, int32_t first, void* stream);

/* Standalone Givens fold of Hessenberg column i (i+1 entries h, device) into
 * (rot, g, tri) of a restart length m; *res_out = |g[i]| (givens_update,
 * gmres.py:153-177).  Same device code as the in-cycle fold. */
int lsb_givens_update(double* rot, double* g, double* tri, int32_t m, const double* h, int32_t i,
                      double* res_out, void* stream);
/* y = back-substitution of the rotated k x k triangle (solve_least_squares,
 * gmres.py:184-192); *status = -1, or the index of a zero diagonal. */
int lsb_back_substitute(const double* tri, const double* g, int32_t m, int32_t k, double* y,
                        int32_t* status, void* stream);

/* ---------------------------------------------------------------- diagnostics */
/* gram[row, 0..ncols) = V[:, :ncols]^T V[:, row] (measurement only). */
int lsb_gram_row(const lsb_arnoldi* S, int32_t it, int32_t row, int32_t ncols, double* gram,
                 int64_t gram_ld, void* stream);

/* ---------------------------------------------------------------- peer exchange
 * The row-partitioned solve's two exchange steps (the
 * reference's single-process equivalent is the reduction inside
 * mdot_pair / mass_inner_product / norm2, kernels.py:283-347, and the
 * SpMV's access to neighbouring rows, kernels.py:256-272) as kernels that
 * store straight into the peers' memory over NVLink/NVSwitch and signal
 * with release/acquire epochs kept on the device: no host call per
 * iteration, capturable in the cycle's CUDA graph.  Pointers in mbox/sig
 * are this process's mappings of each rank's buffers (CUDA IPC across
 * processes, plain device pointers within one); epoch and counter are this
 * rank's own, zero-initialised. */
#define LSB_PEER_MAX 16
#define LSB_COMM_TIMEOUT 1
typedef struct lsb_peer {
  int32_t rank, size;
  int32_t slot;          /* doubles per mailbox slot (>= count + 1)            */
  int32_t pad;
  int64_t timeout_ns;    /* spin-wait limit, <= 0: 60 s                         */
  double* mbox[LSB_PEER_MAX];   /* rank q's mailbox: [2][size][slot] doubles    */
  int64_t* sig[LSB_PEER_MAX];   /* rank q's signal words: [size + 2] int64      */
  int64_t* epoch;        /* this rank: [0] all-gather, [1] halo, [2] error      */
  uint32_t* counter;     /* this rank: grid counter (self-resetting)            */
} lsb_peer;
/* out[q*out_stride + i] = rank q's local[i], i < count, for every rank q
 * (one exchange; ranks must call it the same number of times).  Also ORs
 * every rank's flags->nonfinite into this rank's. */
int lsb_peer_allgather(const lsb_peer* P, const double* local, int32_t count, double* out,
                       int32_t out_stride, lsb_flags* flags, void* stream);
/* Ghost planes: lo_src (this rank's first plane) -> lo_dst (rank-1's upper
 * ghost, NULL on rank 0), hi_src (last plane) -> hi_dst (rank+1's lower
 * ghost, NULL on the last rank); returns on the stream once both
 * neighbours' planes have landed here. */
int lsb_peer_halo(const lsb_peer* P, const double* lo_src, double* lo_dst, const double* hi_src,
                  double* hi_dst, int64_t plane, lsb_flags* flags, void* stream);
/* Ghost exchange fused into the kernels on either side of it (one-sync
 * fused 7-point path): the K2 that finishes column p also stores its first
 * / last `plane` rows straight into the neighbours' ghost rows of the same
 * column and, from its last CTA, releases the neighbours' halo signals with
 * this rank's next halo epoch; the next fused K1+SpMV processes its interior
 * tiles first and waits for its own signals only before the tiles that read
 * ghost rows.  NULL neighbour pointers = no neighbour on that side. */
typedef struct lsb_halo_push {
  double* lo_dst;        /* rank-1's ghost rows above its block (peer-mapped) */
  double* hi_dst;        /* rank+1's ghost rows below its block (peer-mapped) */
  int64_t plane;         /* ghost rows per side (even)                        */
  int64_t* sig_lo;       /* rank-1's "from above" signal word (peer-mapped)   */
  int64_t* sig_hi;       /* rank+1's "from below" signal word (peer-mapped)   */
  int64_t* epoch;        /* this rank's halo epoch (lsb_peer.epoch + 1)       */
  uint32_t* counter;     /* this rank's grid counter (lsb_peer.counter)       */
} lsb_halo_push;
typedef struct lsb_halo_wait {
  const int64_t* sig_lo; /* own "from below" word, NULL without a lower rank   */
  const int64_t* sig_hi; /* own "from above" word, NULL without an upper rank  */
  const int64_t* epoch;  /* own halo epoch                                     */
  int64_t timeout_ns;    /* <= 0: 60 s                                         */
  lsb_flags* flags;      /* comm_error on timeout                              */
} lsb_halo_wait;
/* lsb_lagged_update + the halo push of column p (see lsb_halo_push). */
int lsb_lagged_update_push(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                           const lsb_halo_push* hp, void* stream);
/* lsb_lagged_reduce_spmv7 on a slab whose ghost rows arrive by push:
 * interior tiles first, boundary tiles after the neighbours' signals. */
int lsb_lagged_reduce_spmv7_halo(const lsb_arnoldi* S, const lsb_stencil* A, int32_t it,
                                 int32_t p, const lsb_halo_wait* hw, void* stream);
/* out[e] = sum_q parts[q*stride + e] over the nparts rank partials, in
 * rank order (e < count): completes an all-gathered reduction, e.g. a
 * diagnostics Gram row (diagnostics.py:47-69) on the row-partitioned
 * solve.  Gated like the cycle kernels. */
int lsb_sum_parts(const double* parts, int32_t nparts, int32_t stride, int32_t count,
                  double* out, const lsb_flags* flags, int32_t it, void* stream);
/* CUDA IPC of an arbitrary device pointer: handle (64 bytes) of the
 * allocation that contains ptr, and ptr's offset inside it. */
int lsb_ipc_export(const void* ptr, void* handle64, int64_t* offset);
/* Map a peer allocation (lazy peer access enabled) / unmap it. */
int lsb_ipc_open(const void* handle64, void** base);
int lsb_ipc_close(void* base);
/* Load every kernel of the library into the current context now (instead
 * of at first launch, CUDA lazy loading): returns the number of kernels
 * loaded, or -LSB_ECUDA.  The host layer calls it once per process before
 * the first launch. */
int lsb_preload(void);

#ifdef __cplusplus
}
#endif
#endif /* LSB200_H */
