// K5: the small (p-sized) state of the orthogonalizers and of GMRES, kept on
// device: deferred norm, breakdown test, R/T/L columns, the projection
// coefficients, the Hessenberg column and its Givens fold, the convergence
// test, and the per-cycle back-substitution.  One CTA; O(p^2) flops.
//
// Everything the serial parts touch (the R column, the rotations) is first
// pulled into shared memory by all threads in parallel, so the serial chain
// (hypot, the Givens sweep) runs at shared-memory latency instead of one L2
// round trip per element.
//
// Reference: gram_schmidt.py:96-106 (breakdown), 206-245 (mgs_lvl2),
// 248-280 (cgs2_lvl2), gmres.py:153-192 (Givens / least squares),
// gmres.py:407-435 (Hessenberg column assembly and settle).
#include "small_body.cuh"

namespace lsb {

// ------------------------------------------------------------------ mgs_lvl2
__global__ void __launch_bounds__(kSmall)
mgs_lvl2_small_kernel(lsb_arnoldi S, int it, int p, int ks, int gc, bool use_smem) {
  pdl_enter();
  if (gated_off(S.flags, it)) return;
  __shared__ SmallShared sh;
  extern __shared__ double sT[];
  mgs_small_body(S, sh, sT, it, p, ks, gc, use_smem);
}

// Deferred settle (pipeline2, gmres.py:444-462): the Givens fold of
// Hessenberg column gc-1 = R[0..gc, gc] run apart from the small-state
// kernel (which was launched with givens_col = -gc), on a side stream, so it
// overlaps the next iteration's basis passes.
__global__ void __launch_bounds__(kSmall)
settle_kernel(lsb_arnoldi S, int it, int gc) {
  if (gated_off(S.flags, it)) return;
  __shared__ SmallShared sh;
  const int cap = S.cap;
  for (int j = threadIdx.x; j <= gc; j += blockDim.x) sh.col[j] = S.R[(int64_t)j * cap + gc];
  __syncthreads();
  const bool broke = S.flags->broke_iter == it;
  if (broke && threadIdx.x == 0) sh.col[gc] = 0.0;
  settle_block(S, sh, it, gc, broke);
}

int launch_settle(const lsb_arnoldi& S, int it, int gc, cudaStream_t st) {
  if (gc < 1 || gc > S.m) return LSB_ERANGE;
  settle_kernel<<<1, kSmall, 0, st>>>(S, it, gc);
  return check_launch("settle");
}

// ------------------------------------------------------------------ cgs2_lvl2
__global__ void __launch_bounds__(kSmall)
cgs2_small_a_kernel(lsb_arnoldi S, int it, int p, int ks, int gc, bool use_smem) {
  pdl_enter();
  if (gated_off(S.flags, it)) return;
  __shared__ SmallShared sh;
  extern __shared__ double sL[];   // L[:p-1, :p-1] (row stride p) when use_smem
  const int t = threadIdx.x, cap = S.cap;
  if (use_smem) stage_block(sL, p, S.L, cap, p - 1, p - 1);   // in flight during the front
  const bool broke = lagged_front(S, sh, it, p, gc);
  if (broke) {
    if (gc > 0) settle_block(S, sh, it, gc, true);
    return;
  }
  const double beta = sh.beta;
  // L[p-1, :p-1] = G[:p-1, 0] / beta  (gram_schmidt.py:266-267)
  for (int e = t; e < p - 1; e += blockDim.x) {
    const double v = __ddiv_rn(sh.a[e], beta);
    S.L[(int64_t)(p - 1) * cap + e] = v;
    if (use_smem) sL[(p - 1) * p + e] = v;
  }
  if (t == 0) sh.y[p - 1] = __ddiv_rn(sh.y[p - 1], beta);
  __syncthreads();
  // r = y - Ls y - Ls^T y  (/beta)   (gram_schmidt.py:270-274)
  for (int j = t; j < p; j += blockDim.x) {
    double a = 0.0, b = 0.0;
    if (use_smem) {
      for (int l = 0; l < j; ++l) a = fma(sL[j * p + l], sh.y[l], a);
      for (int l = j + 1; l < p; ++l) b = fma(sL[l * p + j], sh.y[l], b);
    } else {
      for (int l = 0; l < j; ++l) a = fma(S.L[(int64_t)j * cap + l], sh.y[l], a);
      for (int l = j + 1; l < p; ++l) b = fma(S.L[(int64_t)l * cap + j], sh.y[l], b);
    }
    double r = (sh.y[j] - a) - b;
    if (ks) r = __ddiv_rn(r, beta);
    S.coef[j] = r;
  }
  if (gc > 0) settle_block(S, sh, it, gc, false);
}

// s = gathered second-pass products; R[:p, p] = r + s   (gram_schmidt.py:276-278)
__global__ void __launch_bounds__(kSmall)
cgs2_small_b_kernel(lsb_arnoldi S, int it, int p) {
  pdl_enter();
  if (gated_off(S.flags, it)) return;
  if (S.flags->broke_iter == it) return;
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    const double s = gsum(S, j);
    S.coef2[j] = s;
    S.R[(int64_t)j * S.cap + p] = S.coef[j] + s;
  }
}

// ------------------------------------------------------------------ direct kernels
// coef = s (or coef += s) and coef2 = s from the gathered products.
__global__ void __launch_bounds__(kSmall)
collect_coef_kernel(lsb_arnoldi S, int it, int p, int accumulate, int stride, int offset) {
  if (gated_off(S.flags, it)) return;
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    const double s = gsum(S, stride * j + offset);
    S.coef2[j] = s;
    S.coef[j] = accumulate ? S.coef[j] + s : s;
  }
}

// r_diag (already in scal[BETA] from norm_finish), breakdown test, Hbar
// column col-1 = [coef[0..p), r_diag] stored in R[:, col], Givens fold
// (gmres.py:362-381 / gram_schmidt.py:139-141, 158-160).
__global__ void __launch_bounds__(kSmall)
direct_small_kernel(lsb_arnoldi S, int it, int col, int p, int gc) {
  if (gated_off(S.flags, it)) return;
  __shared__ SmallShared sh;
  const int t = threadIdx.x, cap = S.cap;
  for (int j = t; j < p; j += blockDim.x) sh.col[j] = S.coef[j];
  __syncthreads();
  if (t == 0) {
    const double r_diag = S.scal[LSB_S_BETA];
    const double tol = breakdown_tol(S, r_diag, sh.col, p);
    S.scal[LSB_S_TOL] = tol;
    sh.broke = r_diag <= tol;
    if (sh.broke) S.flags->broke_iter = it;
    sh.col[p] = sh.broke ? 0.0 : r_diag;
    if (gc == 0 && sh.broke) { S.flags->stop_iter = it; S.flags->status = LSB_STARTUP_BREAKDOWN; }
  }
  __syncthreads();
  if (gc > 0) {
    for (int j = t; j <= p; j += blockDim.x) S.R[(int64_t)j * cap + col] = sh.col[j];
    settle_block(S, sh, it, gc, sh.broke);
  }
}

// Single-pass classical GS with the Pythagorean norm substitute
// (cgs1_ghysels, gmres.py:325-360).  G holds [Q^T z (p), max|z|, sum z^2]:
// y = Q^T z, h = sqrt(||z||^2 - y.y).  If the radicand keeps its digits the
// column is accepted (H[i, i-1] = h, normal settle); otherwise H[i, i-1] = 0,
// the rotation is still folded, and the cycle stops with status
// LSB_GHYSELS_CHECK so the host can run the true-residual arbitration of
// gmres.py:338-359 before deciding converged / breakdown / cancellation.
// Strided form: y_j at G[stride j + offset] and the norm pair after the 2p
// pair entries of the fused SpMV + reduction (stride 2, offset 1).
__global__ void __launch_bounds__(kSmall)
ghysels_small_kernel(lsb_arnoldi S, int it, int col, int p, int stride, int offset) {
  if (gated_off(S.flags, it)) return;
  __shared__ SmallShared sh;
  const int t = threadIdx.x, cap = S.cap;
  for (int j = t; j < p; j += blockDim.x) {
    const double y = gsum(S, stride * j + offset);
    sh.col[j] = y;
    S.coef[j] = y;
    S.coef2[j] = y;
  }
  __syncthreads();
  if (t == 0) {
    const double ssq = gsum(S, stride * p + 1);
    const double znorm = sqrt(ssq);
    double yy = 0.0;
    for (int j = 0; j < p; ++j) yy = fma(sh.col[j], sh.col[j], yy);
    const double zz = __dmul_rn(znorm, znorm);
    const double rad = __dsub_rn(zz, yy);
    S.scal[LSB_S_RAD] = rad;
    // rad >= 4.0 * EPS * znorm * znorm, evaluated left to right as in Python
    const bool ok = rad > 0.0 && rad >= __dmul_rn(__dmul_rn(__dmul_rn(4.0, kEps), znorm), znorm);
    sh.broke = !ok;
    if (ok) {
      const double h = sqrt(rad);
      S.scal[LSB_S_BETA] = h;
      sh.col[p] = h;
    } else {
      S.flags->broke_iter = it;
      sh.col[p] = 0.0;
    }
  }
  __syncthreads();
  for (int j = t; j <= p; j += blockDim.x) S.R[(int64_t)j * cap + col] = sh.col[j];
  settle_block(S, sh, it, col, false);
  if (t == 0 && sh.broke) {
    // converged-or-not is decided on the host from the true residual
    S.flags->stop_iter = it;
    S.flags->status = LSB_GHYSELS_CHECK;
  }
}

int launch_ghysels_small(const lsb_arnoldi& S, int it, int col, int p, cudaStream_t st,
                         int stride, int offset) {
  if (p + 2 > 2 * S.cap || col < 1) return LSB_ERANGE;
  ghysels_small_kernel<<<1, kSmall, 0, st>>>(S, it, col, p, stride, offset);
  return check_launch("ghysels_small");
}

// ------------------------------------------------------------------ cycle control
__global__ void __launch_bounds__(kSmall)
cycle_begin_kernel(lsb_arnoldi S) {
  const int t = threadIdx.x;
  const int64_t c2 = (int64_t)S.cap * S.cap;
  for (int64_t e = t; e < c2; e += blockDim.x) { S.R[e] = 0.0; S.T[e] = 0.0; if (S.L) S.L[e] = 0.0; }
  for (int64_t e = t; e < (int64_t)(S.m + 1) * S.m; e += blockDim.x) S.tri[e] = 0.0;
  for (int e = t; e < 2 * S.m; e += blockDim.x) S.rot[e] = 0.0;
  for (int e = t; e <= S.m; e += blockDim.x) { S.g[e] = 0.0; S.res[e] = 0.0; }
  for (int e = t; e < S.cap; e += blockDim.x) { S.coef[e] = 0.0; S.coef2[e] = 0.0; }
  __syncthreads();
  if (t == 0) {
    S.g[0] = S.scal[LSB_S_RNORM];
    S.flags->stop_iter = LSB_NO_STOP;
    S.flags->status = LSB_RUNNING;
    S.flags->broke_iter = -1;
    S.flags->k = 0;
    S.flags->restart_ok = 0;
  }
}

// solve_least_squares (gmres.py:184-192) on the rotated k x k triangle:
// row-oriented back substitution, one warp per row dot (fixed lane order).
__global__ void __launch_bounds__(kSmall)
cycle_lsq_kernel(lsb_arnoldi S, int staged) {
  __shared__ double sy[kSmall];
  __shared__ double sg[kSmall];
  extern __shared__ double stri[];          // tri[:k, :k], row stride m (staged)
  const int t = threadIdx.x, lane = t & 31;
  const int stop = S.flags->stop_iter;
  // a cgs1_ghysels cancellation check leaves the extract to the host
  const int k = S.flags->status == LSB_GHYSELS_CHECK ? 0 : (stop == LSB_NO_STOP ? S.m : stop);
  const int m = S.m;
  // the triangle and g into shared memory by the whole CTA, every thread with
  // 8 loads in flight (a warp reading them row by row from L2 inside the
  // serial solve took ~64 us per cycle); the solve itself is unchanged
  const double* tri = S.tri;
  if (staged) {
    stage_block(stri, m, S.tri, m, k, k);
    tri = stri;
  }
  for (int j = t; j < k; j += blockDim.x) sg[j] = S.g[j];
  __syncthreads();
  if (t >= 32) return;
  if (lane == 0) S.flags->k = k;
  for (int i = k - 1; i >= 0; --i) {
    const double d = tri[(int64_t)i * m + i];
    if (d == 0.0) {
      if (lane == 0) { S.flags->status = LSB_SINGULAR; S.flags->k = i; }
      return;
    }
    double acc = 0.0;
    for (int j = i + 1 + lane; j < k; j += 32) acc = fma(tri[(int64_t)i * m + j], sy[j], acc);
    acc = warp_sum(acc);
    if (lane == 0) sy[i] = __ddiv_rn(sg[i] - acc, d);
    __syncwarp();
  }
  for (int j = lane; j < k; j += 32) S.coef2[j] = sy[j];
}

// Trial least squares of iteration `it` (k = it columns) into y, for the
// true-residual probe (gmres.py:273-278); a zero diagonal marks y[0] NaN.
__global__ void __launch_bounds__(32)
trial_lsq_kernel(lsb_arnoldi S, int it, double* y) {
  if (gated_off(S.flags, it)) return;
  __shared__ double sy[kSmall];
  const int lane = threadIdx.x, k = it, m = S.m;
  for (int i = k - 1; i >= 0; --i) {
    const double d = S.tri[(int64_t)i * m + i];
    if (d == 0.0) {
      if (lane == 0) y[0] = nan("");
      return;
    }
    double acc = 0.0;
    for (int j = i + 1 + lane; j < k; j += 32) acc = fma(S.tri[(int64_t)i * m + j], sy[j], acc);
    acc = warp_sum(acc);
    if (lane == 0) sy[i] = __ddiv_rn(S.g[i] - acc, d);
    __syncwarp();
  }
  for (int j = lane; j < k; j += 32) y[j] = sy[j];
}

int launch_trial_lsq(const lsb_arnoldi& S, int it, double* y, cudaStream_t st) {
  if (it < 1 || it > S.m) return LSB_ERANGE;
  trial_lsq_kernel<<<1, 32, 0, st>>>(S, it, y);
  return check_launch("trial_lsq");
}

// First call: denom = beta0 or 1, target = rel_tol * beta0 (gmres.py:472-479).
__global__ void restart_check_kernel(lsb_arnoldi S, int first) {
  if (threadIdx.x != 0) return;
  const double rn = S.scal[LSB_S_RNORM];
  if (first) {
    S.scal[LSB_S_DENOM] = rn > 0.0 ? rn : 1.0;
    S.scal[LSB_S_TARGET] = __dmul_rn(S.scal[LSB_S_RELTOL], rn);
  }
  S.flags->restart_ok = rn <= S.scal[LSB_S_TARGET];
}

// ------------------------------------------------------------------ launchers
int launch_mgs_lvl2_small(const lsb_arnoldi& S, int it, int p, int ks, int gc, cudaStream_t st) {
  if (p < 1 || S.cap > kSmall || p >= S.cap) return LSB_ERANGE;
  constexpr size_t kMaxT = 160 * 1024;   // T block staged in smem up to p = 143
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(mgs_lvl2_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMaxT);
    attr = true;
  }
  const size_t need = sizeof(double) * (size_t)p * p;
  const bool use = need <= kMaxT;
  const cudaError_t le = launch_chain(use_pdl(S.n), mgs_lvl2_small_kernel, dim3(1), dim3(kSmall), use ? need : 0, st, S, it, p, ks, gc,
               use);
  return check_launch("mgs_lvl2_small", le);
}
int launch_cgs2_small_a(const lsb_arnoldi& S, int it, int p, int ks, int gc, cudaStream_t st) {
  if (p < 1 || S.cap > kSmall || p >= S.cap) return LSB_ERANGE;
  constexpr size_t kMaxL = 160 * 1024;   // L block staged in smem up to p = 143
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(cgs2_small_a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMaxL);
    attr = true;
  }
  const size_t need = sizeof(double) * (size_t)p * p;
  const bool use = need <= kMaxL;
  const cudaError_t le = launch_chain(use_pdl(S.n) && p <= 32, cgs2_small_a_kernel, dim3(1),
                                      dim3(kSmall), use ? need : 0, st, S, it, p, ks, gc, use);
  return check_launch("cgs2_small_a", le);
}
int launch_cgs2_small_b(const lsb_arnoldi& S, int it, int p, cudaStream_t st) {
  const cudaError_t le = launch_chain(use_pdl(S.n) && p <= 32, cgs2_small_b_kernel, dim3(1), dim3(kSmall), 0, st, S, it, p);
  return check_launch("cgs2_small_b", le);
}
int launch_collect_coef(const lsb_arnoldi& S, int it, int p, int acc, cudaStream_t st,
                        int stride, int offset) {
  collect_coef_kernel<<<1, kSmall, 0, st>>>(S, it, p, acc, stride, offset);
  return check_launch("collect_coef");
}
int launch_direct_small(const lsb_arnoldi& S, int it, int col, int p, int gc, cudaStream_t st) {
  if (p + 1 > kSmall) return LSB_ERANGE;
  direct_small_kernel<<<1, kSmall, 0, st>>>(S, it, col, p, gc);
  return check_launch("direct_small");
}
int launch_cycle_begin(const lsb_arnoldi& S, cudaStream_t st) {
  if (S.cap > kSmall) return LSB_ERANGE;
  cycle_begin_kernel<<<1, kSmall, 0, st>>>(S);
  return check_launch("cycle_begin");
}
int launch_cycle_lsq(const lsb_arnoldi& S, cudaStream_t st) {
  constexpr size_t kMaxTri = 160 * 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(cycle_lsq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMaxTri);
    attr = true;
  }
  const size_t need = sizeof(double) * (size_t)S.m * S.m;
  const int staged = need <= kMaxTri;
  cycle_lsq_kernel<<<1, kSmall, staged ? need : 0, st>>>(S, staged);
  return check_launch("cycle_lsq");
}
int launch_restart_check(const lsb_arnoldi& S, int first, cudaStream_t st) {
  restart_check_kernel<<<1, 32, 0, st>>>(S, first);
  return check_launch("restart_check");
}

// ------------------------------------------------------------------ standalone Givens / LSQ
// givens_update(state, h_col, i) and solve_least_squares(state, k) of the
// public API (gmres.py:153-192) on device-resident GivensState arrays --
// the same fold the cycle kernels run.
__global__ void givens_update_kernel(double* rot, double* g, double* tri, int m, const double* hin,
                                     int i, double* res_out) {
  __shared__ double h[kSmall + 2];
  __shared__ double r[2 * kSmall];
  for (int j = threadIdx.x; j <= i; j += blockDim.x) h[j] = hin[j];
  for (int j = threadIdx.x; j < 2 * (i - 1); j += blockDim.x) r[j] = rot[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    *res_out = givens_fold(h, r, g, i);
    rot[2 * (i - 1)] = r[2 * (i - 1)];
    rot[2 * (i - 1) + 1] = r[2 * (i - 1) + 1];
  }
  __syncthreads();
  for (int j = threadIdx.x; j <= i; j += blockDim.x) tri[(int64_t)j * m + (i - 1)] = h[j];
}

__global__ void back_substitute_kernel(const double* tri, const double* g, int m, int k, double* y,
                                       int* status) {
  if (threadIdx.x != 0) return;
  *status = -1;
  for (int i = k - 1; i >= 0; --i) {
    const double d = tri[(int64_t)i * m + i];
    if (d == 0.0) { *status = i; return; }
    double acc = 0.0;
    for (int j = i + 1; j < k; ++j) acc = fma(tri[(int64_t)i * m + j], y[j], acc);
    y[i] = __ddiv_rn(g[i] - acc, d);
  }
}

int launch_givens_update(double* rot, double* g, double* tri, int m, const double* h, int i,
                         double* res, cudaStream_t st) {
  if (i < 1 || i > m || m + 1 > kSmall) return LSB_ERANGE;
  givens_update_kernel<<<1, 128, 0, st>>>(rot, g, tri, m, h, i, res);
  return check_launch("givens_update");
}
int launch_back_substitute(const double* tri, const double* g, int m, int k, double* y, int* status,
                           cudaStream_t st) {
  if (k < 0 || k > m) return LSB_ERANGE;
  back_substitute_kernel<<<1, 32, 0, st>>>(tri, g, m, k, y, status);
  return check_launch("back_substitute");
}

// lsb_preload: one kernel of this translation unit (its module)
const void* tu_anchor_small() { return (const void*)mgs_lvl2_small_kernel; }

}  // namespace lsb
