// Row-parallel passes over the basis: MAXPY family (K2/K4/K10), the fused
// level-1 MGS axpy+dot pass (K8), norms and scalings.  All are HBM-bound
// streaming kernels: 128-bit loads of row pairs, coefficients broadcast
// from shared memory, grid-stride persistent CTAs.
#include "tile.cuh"

#include <cooperative_groups.h>

namespace lsb {

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// acc (a row pair) += c[k] X[:, k], k ascending (one fma chain): groups of 8
// columns, then the 1..7 leftover columns as one straight-line block (all
// loads first) instead of a rolled remainder loop that exposes one load
// latency per column.
// (NEG: the coefficients negated, cgs_project's fma(-s, q, .) chain.)
// K2 per C2 cycle 30.6 -> 29.7 ms (p <= 8: 0.71-0.93x the time), and 48
// instead of 64 registers.
template <bool NEG = false>
__device__ __forceinline__ void fma_chain2_tail(double2& acc, const double* __restrict__ X,
                                                int64_t ld, int64_t r, const double* c,
                                                int kend) {
  const int k8 = kend & ~7;
  for (int k0 = 0; k0 < k8; k0 += 8) {
    double2 q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) q[j] = ld2(X + (int64_t)(k0 + j) * ld + r);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double cc = NEG ? -c[k0 + j] : c[k0 + j];
      acc.x = fma(cc, q[j].x, acc.x);
      acc.y = fma(cc, q[j].y, acc.y);
    }
  }
  switch (kend - k8) {
#define LSB_TAIL(R)                                                          \
    case R: {                                                                \
      double2 q[R];                                                          \
      _Pragma("unroll") for (int j = 0; j < R; ++j)                          \
        q[j] = ld2(X + (int64_t)(k8 + j) * ld + r);                          \
      _Pragma("unroll") for (int j = 0; j < R; ++j) {                        \
        const double cc = NEG ? -c[k8 + j] : c[k8 + j];                      \
        acc.x = fma(cc, q[j].x, acc.x);                                      \
        acc.y = fma(cc, q[j].y, acc.y);                                      \
      }                                                                      \
    } break;
    LSB_TAIL(1) LSB_TAIL(2) LSB_TAIL(3) LSB_TAIL(4) LSB_TAIL(5) LSB_TAIL(6) LSB_TAIL(7)
#undef LSB_TAIL
    default: break;
  }
}
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// Dynamic shared memory for a k-entry coefficient vector, padded: the
// unrolled coefficient loops are vectorised into 128-bit LDS that may touch
// sc[k] (unused) -- keep that inside the allocation (compute-sanitizer).
static inline size_t coef_smem(int k) { return sizeof(double) * ((k > 0 ? k : 1) + 16); }

static int row_grid(int64_t n, int per_sm = 8) {
  const int64_t pairs = (n + 1) / 2;
  int64_t g = (pairs + kThreads - 1) / kThreads;
  const int knob = tuning(LSB_TUNE_ROW_CTAS_PER_SM);
  if (knob > 0) per_sm = knob;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// ------------------------------------------------------------------ maxpy
// out = y + sign * X alpha   (kernels.py:350-362; cgs_iterated uses sign -1)
__global__ void __launch_bounds__(kThreads)
maxpy_kernel(const double* __restrict__ y, const double* __restrict__ X, int64_t ld, int64_t n,
             int p, const double* __restrict__ alpha, double sign, double* out,
             const lsb_flags* gate, int it) {
  if (gated_off(gate, it)) return;
  extern __shared__ double sa[];
  for (int k = threadIdx.x; k < p; k += blockDim.x) sa[k] = sign * alpha[k];
  __syncthreads();
  const int64_t npair = n / 2;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npair;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = 2 * j;
    double2 acc = make_double2(0.0, 0.0);
    fma_chain2_tail(acc, X, ld, r, sa, p);
    const double2 yy = ld2(y + r);
    st2(out + r, make_double2(yy.x + acc.x, yy.y + acc.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t r = n - 1;
    double acc = 0.0;
    for (int k = 0; k < p; ++k) acc = fma(sa[k], X[(int64_t)k * ld + r], acc);
    out[r] = y[r] + acc;
  }
}

int launch_maxpy(const double* y, const double* X, int64_t ld, int64_t n, int p,
                 const double* alpha, int sign, double* out, const lsb_flags* gate, int it,
                 cudaStream_t st) {
  if (n <= 0) return LSB_OK;
  static const int occ_ = wave(maxpy_kernel, 2048);
  maxpy_kernel<<<row_grid(n, occ_), kThreads, coef_smem(p), st>>>(
      y, X, ld, n, p, alpha, sign < 0 ? -1.0 : 1.0, out, gate, it);
  return check_launch("maxpy");
}

// ------------------------------------------------------------------ lagged update (K2)
// gram_schmidt.py:230-242:  u /= beta;  (krylov) w /= beta;  w -= Q c
// with Q's last column already the normalised u.  One pass: reads Q and w,
// writes u and w.
__global__ void __launch_bounds__(kThreads)
lagged_update_kernel(lsb_arnoldi S, int it, int p, int ks, lsb_halo_push hp) {
  pdl_enter();
  const bool push = hp.epoch != nullptr;
  // a gated-off or broken-down iteration does no row work; with the fused
  // halo push it still advances this rank's halo epoch and signals the
  // neighbours, so every rank issues the same epochs whatever moment its own
  // flags were set (pipeline2 settles on a side stream, so the gate can
  // close at different points of the kernel sequence on different ranks)
  __shared__ int s_skip;   // one decision per CTA (the flags may change under a side-stream settle)
  if (threadIdx.x == 0)
    s_skip = gated_off(S.flags, it) || (S.flags && S.flags->broke_iter == it);
  __syncthreads();
  const bool skip = s_skip != 0;
  if (skip && !push) return;
  if (!skip) {
  extern __shared__ double sc[];
  for (int k = threadIdx.x; k < p; k += blockDim.x) sc[k] = S.coef[k];
  __syncthreads();
  const double beta = S.scal[LSB_S_BETA];
  const int64_t ld = S.ld, n = S.n;
  double* __restrict__ u = S.V + (int64_t)(p - 1) * ld;
  double* __restrict__ w = S.V + (int64_t)p * ld;
  const double cu = sc[p - 1];
  const int64_t npair = n / 2;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npair;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = 2 * j;
    double2 acc = make_double2(0.0, 0.0);
    fma_chain2_tail(acc, S.V, ld, r, sc, p - 1);
    double2 uu = ld2(u + r);
    uu.x = __ddiv_rn(uu.x, beta);
    uu.y = __ddiv_rn(uu.y, beta);
    st2(u + r, uu);
    acc.x = fma(cu, uu.x, acc.x);
    acc.y = fma(cu, uu.y, acc.y);
    double2 ww = ld2(w + r);
    if (ks) { ww.x = __ddiv_rn(ww.x, beta); ww.y = __ddiv_rn(ww.y, beta); }
    const double2 out = make_double2(ww.x - acc.x, ww.y - acc.y);
    st2(w + r, out);
    if (hp.lo_dst || hp.hi_dst) {   // boundary rows of the new column into the neighbours' ghost rows
      if (hp.lo_dst && r < hp.plane) st2(hp.lo_dst + r, out);
      if (hp.hi_dst && r >= n - hp.plane) st2(hp.hi_dst + (r - (n - hp.plane)), out);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t r = n - 1;
    double acc = 0.0;
    for (int k = 0; k < p - 1; ++k) acc = fma(sc[k], S.V[(int64_t)k * ld + r], acc);
    const double uu = __ddiv_rn(u[r], beta);
    u[r] = uu;
    acc = fma(cu, uu, acc);
    double ww = w[r];
    if (ks) ww = __ddiv_rn(ww, beta);
    w[r] = ww - acc;
  }
  }   // !skip
  if (push) {
    // every CTA's remote stores are visible system-wide before the last CTA
    // releases the neighbours' signals with this rank's next halo epoch
    __threadfence_system();
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) s_last = atomicAdd(hp.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      __threadfence_system();
      const int64_t e = *hp.epoch + 1;
      if (hp.sig_lo) st_release_sys64(hp.sig_lo, e);
      if (hp.sig_hi) st_release_sys64(hp.sig_hi, e);
      *hp.epoch = e;
      *hp.counter = 0u;
    }
  }
}

int launch_lagged_update(const lsb_arnoldi& S, int it, int p, int ks, cudaStream_t st,
                         const lsb_halo_push* hp) {
  if (p < 1) return LSB_OK;
  lsb_halo_push h = {};
  if (hp) {
    if (!hp->epoch || !hp->counter || hp->plane < 0 || (hp->plane & 1) || hp->plane > S.n ||
        (hp->lo_dst && !hp->sig_lo) || (hp->hi_dst && !hp->sig_hi))
      return LSB_EINVAL;
    h = *hp;
  }
  static const int occ_ = wave(lagged_update_kernel, 2048);
  const cudaError_t le = launch_chain(use_pdl(S.n), lagged_update_kernel, dim3((unsigned)row_grid(S.n, occ_)), dim3(kThreads),
               coef_smem(p), st, S, it, p, ks, h);
  return check_launch("lagged_update", le);
}

// w -= Q coef2   (cgs2_lvl2 second projection, gram_schmidt.py:277)
__global__ void __launch_bounds__(kThreads)
lagged_correct_kernel(lsb_arnoldi S, int it, int p) {
  pdl_enter();
  if (gated_off(S.flags, it)) return;
  if (S.flags && S.flags->broke_iter == it) return;
  extern __shared__ double sc[];
  for (int k = threadIdx.x; k < p; k += blockDim.x) sc[k] = S.coef2[k];
  __syncthreads();
  const int64_t ld = S.ld, n = S.n;
  double* __restrict__ w = S.V + (int64_t)p * ld;
  const int64_t npair = n / 2;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npair;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = 2 * j;
    double2 acc = make_double2(0.0, 0.0);
    fma_chain2_tail(acc, S.V, ld, r, sc, p);
    const double2 ww = ld2(w + r);
    st2(w + r, make_double2(ww.x - acc.x, ww.y - acc.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t r = n - 1;
    double acc = 0.0;
    for (int k = 0; k < p; ++k) acc = fma(sc[k], S.V[(int64_t)k * ld + r], acc);
    w[r] = w[r] - acc;
  }
}

int launch_lagged_correct(const lsb_arnoldi& S, int it, int p, cudaStream_t st) {
  if (p < 1) return LSB_OK;
  static const int occ_ = wave(lagged_correct_kernel, 2048);
  const cudaError_t le = launch_chain(use_pdl(S.n) && p <= 32, lagged_correct_kernel, dim3((unsigned)row_grid(S.n, occ_)),
               dim3(kThreads), coef_smem(p), st, S, it, p);
  return check_launch("lagged_correct", le);
}

// ------------------------------------------------------------------ level-1 MGS pass (K8)
// gram_schmidt.py:154-158: pass k applies the (k-1)-th rank-1 update
// `work -= h * Q[:, k-1]` (numpy: product then difference, two roundings)
// and produces the k-th dot `Q[:, k] . work` -- or, after the last update,
// the (max|z|, sum z^2) pair of the norm.  z is read and written once.
__device__ __forceinline__ double sum_parts(const lsb_arnoldi& S, int e) {
  double v = S.G[e];
  for (int q = 1; q < S.g_parts; ++q) v += S.G[(int64_t)q * S.g_stride + e];
  return v;
}

// The rows of pass k: z -= h q_{k-1} (k > 0), then a0 = q_k . z (k < p) or
// (a0, a1) = (max|z|, sum z^2) (k == p).  Shared by the per-pass kernel and
// the cooperative all-passes kernel, so both produce the same partials.
__device__ __forceinline__ void mgs1_rows(const lsb_arnoldi& S, int col, int k, int p, double h,
                                          double& a0, double& a1) {
  const int64_t ld = S.ld, n = S.n;
  double* __restrict__ z = S.V + (int64_t)col * ld;
  const double* qm = k > 0 ? S.V + (int64_t)(k - 1) * ld : nullptr;
  const double* qk = k < p ? S.V + (int64_t)k * ld : nullptr;
  auto row = [&](double zz, double qmv, double qkv) -> double {
    if (qm) zz = __dsub_rn(zz, __dmul_rn(h, qmv));
    if (qk) a0 = fma(qkv, zz, a0);
    else { a0 = fmax(a0, fabs(zz)); a1 = fma(zz, zz, a1); }
    return zz;
  };
  // row pairs, two pairs per thread per step: six independent 128-bit loads
  // in flight (a scalar row loop leaves the pass latency-bound)
  const int64_t npair = n / 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double2 zero2 = make_double2(0.0, 0.0);
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npair; j += 2 * stride) {
    const int64_t j2 = j + stride;
    const bool two = j2 < npair;
    const double2 z0 = ld2(z + 2 * j);
    const double2 z1 = two ? ld2(z + 2 * j2) : zero2;
    const double2 m0 = qm ? ld2(qm + 2 * j) : zero2;
    const double2 m1 = qm && two ? ld2(qm + 2 * j2) : zero2;
    const double2 k0 = qk ? ld2(qk + 2 * j) : zero2;
    const double2 k1 = qk && two ? ld2(qk + 2 * j2) : zero2;
    double2 o0;
    o0.x = row(z0.x, m0.x, k0.x);
    o0.y = row(z0.y, m0.y, k0.y);
    if (qm) st2(z + 2 * j, o0);
    if (two) {
      double2 o1;
      o1.x = row(z1.x, m1.x, k1.x);
      o1.y = row(z1.y, m1.y, k1.y);
      if (qm) st2(z + 2 * j2, o1);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t r = n - 1;
    const double zz = row(z[r], qm ? qm[r] : 0.0, qk ? qk[r] : 0.0);
    if (qm) z[r] = zz;
  }
}

__global__ void __launch_bounds__(kThreads)
mgs1_pass_kernel(lsb_arnoldi S, int it, int col, int k, int p) {
  pdl_enter();
  if (gated_off(S.flags, it)) return;
  double h = 0.0;
  if (k > 0) {
    h = sum_parts(S, 0);
    if (blockIdx.x == 0 && threadIdx.x == 0) S.coef[k - 1] = h;
  }
  double a0 = 0.0, a1 = 0.0;  // dot  or  (amax, ssq)
  mgs1_rows(S, col, k, p, h, a0, a1);
  if (k < p) {
    const double v[1] = {a0};
    const int op[1] = {0};
    grid_reduce<1>(v, op, S.ws.partial, S.ws.counter, S.Gloc);
  } else {
    const double v[2] = {a0, a1};
    const int op[2] = {1, 0};
    grid_reduce<2>(v, op, S.ws.partial, S.ws.counter, S.Gloc);
  }
}

// All p + 1 passes of one column in ONE cooperative launch (single rank:
// the reduction of pass k feeds pass k + 1 without a host all-gather).  Each
// pass ends with a grid barrier instead of a kernel boundary; the pass-k dot
// is then summed redundantly by every CTA in exactly grid_reduce's order
// over the same per-CTA partials (same grid, same rows per CTA as the
// per-pass kernel), so h, coef and z are bitwise the per-pass results.
// Partials alternate between two halves of the workspace (a fast CTA writes
// pass k+1's partial while a slow one still reads pass k's); the final
// (max, ssq) reduction uses the next 2G entries (lsb_partial_len >= 4 *
// 8 * SMs >= 4G).
__global__ void __launch_bounds__(kThreads)
mgs1_grid_kernel(lsb_arnoldi S, int it, int col, int p) {
  if (gated_off(S.flags, it)) return;      // grid-uniform: no CTA reaches a barrier
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  __shared__ double red[kWarps];
  __shared__ double s_h;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  double h = 0.0;
  for (int k = 0; k <= p; ++k) {
    if (k > 0 && blockIdx.x == 0 && threadIdx.x == 0) S.coef[k - 1] = h;
    double a0 = 0.0, a1 = 0.0;
    mgs1_rows(S, col, k, p, h, a0, a1);
    if (k == p) {   // (max, ssq) past both halves: slow CTAs may still read pass p-1's
      const double v[2] = {a0, a1};
      const int op[2] = {1, 0};
      grid_reduce<2>(v, op, S.ws.partial + 2 * (size_t)G, S.ws.counter, S.Gloc);
      break;
    }
    double* part = S.ws.partial + (size_t)(k & 1) * G;
    const double x = warp_sum(a0);
    if (lane == 0) red[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      double y = red[0];
      for (int w = 1; w < kWarps; ++w) y = y + red[w];
      part[blockIdx.x] = y;
    }
    grid.sync();
    if (warp == 0) {
      double y = 0.0;
      bool first = true;
      for (int c = lane; c < G; c += 32) {
        const double t = __ldcg(part + c);
        if (first) { y = t; first = false; } else { y = y + t; }
      }
      if (first) y = 0.0;
      y = warp_sum(y);
      if (lane == 0) s_h = y;
    }
    __syncthreads();
    h = s_h;
    if (blockIdx.x == 0 && threadIdx.x == 0) S.Gloc[0] = h;
    __syncthreads();                       // s_h is rewritten after the next barrier only
  }
}

int launch_mgs1_pass(const lsb_arnoldi& S, int it, int col, int k, int p, cudaStream_t st) {
  static const int occ_ = wave(mgs1_pass_kernel, 0);
  // consecutive passes chain through programmatic dependent launch at every
  // n: pass k+1's CTAs become resident during pass k's reduction tail
  // (LSB_TUNE_PDL = 2 turns it off)
  const cudaError_t le = launch_chain(tuning(LSB_TUNE_PDL) != 2, mgs1_pass_kernel,
                                      dim3((unsigned)row_grid(S.n / 2 + 1, occ_)), dim3(kThreads),
                                      0, st, S, it, col, k, p);
  return check_launch("mgs1_pass", le);
}

// lsb_mgs1_passes: passes 0..p of column col.  Cooperative single launch
// when the rank is alone (g_parts == 1, G aliases Gloc) and the per-pass
// grid is co-resident for the cooperative kernel; else p + 1 chained
// per-pass launches (identical results either way).
int launch_mgs1_passes(const lsb_arnoldi& S, int it, int col, int p, cudaStream_t st) {
  if (S.g_parts != 1 || S.G != S.Gloc) return LSB_EINVAL;
  static const int occ_pass = wave(mgs1_pass_kernel, 0);
  static const int occ_grid = wave(mgs1_grid_kernel, 0);
  const int G = row_grid(S.n / 2 + 1, occ_pass);
  if (tuning(LSB_TUNE_MGS1_GRID) != 2 && (int64_t)G <= (int64_t)sm_count() * occ_grid) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return check_launch("mgs1_grid", cudaLaunchKernelEx(&cfg, mgs1_grid_kernel, S, it, col, p));
  }
  for (int k = 0; k <= p; ++k) {
    const int rc = launch_mgs1_pass(S, it, col, k, p, st);
    if (rc) return rc;
  }
  return LSB_OK;
}

// z <- z - Q coef2 (cgs_iterated pass, gram_schmidt.py:136-138), optional
// (max|z|, sum z^2) of the result for the following norm.
template <bool DIV>
__global__ void __launch_bounds__(kThreads)
cgs_project_kernel(lsb_arnoldi S, int it, int col, int p, int want_norm) {
  if (gated_off(S.flags, it)) return;
  extern __shared__ double sc[];
  for (int k = threadIdx.x; k < p; k += blockDim.x) sc[k] = S.coef2[k];
  __syncthreads();
  const int64_t ld = S.ld, n = S.n;
  double* __restrict__ z = S.V + (int64_t)col * ld;
  // want_norm == 2: then q = z / r_diag unless the column broke down
  // (lsb_direct_normalize fused: the same rounded difference, then the same
  // division -- bitwise the two-kernel result)
  // (a separate instantiation: the extra live registers would lower the
  // occupancy of the plain projection, 40 -> 48 registers, ~5% of a cgs2 cycle)
  const bool divide = DIV && !(S.flags && S.flags->broke_iter == it);
  const double d = DIV ? S.scal[LSB_S_BETA] : 1.0;
  double amax = 0.0, ssq = 0.0;
  const int64_t npair = n / 2;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npair;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = 2 * j;
    double2 acc = make_double2(0.0, 0.0);
    fma_chain2_tail<true>(acc, S.V, ld, r, sc, p);
    double2 zz = ld2(z + r);
    zz.x = zz.x + acc.x;
    zz.y = zz.y + acc.y;
    if (DIV && divide) {
      zz.x = __ddiv_rn(zz.x, d);
      zz.y = __ddiv_rn(zz.y, d);
    }
    st2(z + r, zz);
    amax = fmax(amax, fmax(fabs(zz.x), fabs(zz.y)));
    ssq = fma(zz.x, zz.x, ssq);
    ssq = fma(zz.y, zz.y, ssq);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t r = n - 1;
    double acc = 0.0;
    for (int k = 0; k < p; ++k) acc = fma(-sc[k], S.V[(int64_t)k * ld + r], acc);
    double zz = z[r] + acc;
    if (DIV && divide) zz = __ddiv_rn(zz, d);
    z[r] = zz;
    amax = fmax(amax, fabs(zz));
    ssq = fma(zz, zz, ssq);
  }
  if (!DIV && want_norm == 1) {
    const double v[2] = {amax, ssq};
    const int op[2] = {1, 0};
    grid_reduce<2>(v, op, S.ws.partial, S.ws.counter, S.Gloc);
  }
}

int launch_cgs_project(const lsb_arnoldi& S, int it, int col, int p, int want_norm,
                       cudaStream_t st) {
  if (want_norm == 2) {
    static const int occd = wave(cgs_project_kernel<true>, 2048);
    cgs_project_kernel<true><<<row_grid(S.n, occd), kThreads, coef_smem(p), st>>>(
        S, it, col, p, want_norm);
    return check_launch("cgs_project_div");
  }
  static const int occ_ = wave(cgs_project_kernel<false>, 2048);
  cgs_project_kernel<false><<<row_grid(S.n, occ_), kThreads, coef_smem(p), st>>>(
      S, it, col, p, want_norm);
  return check_launch("cgs_project");
}

// ------------------------------------------------------------------ norms
__global__ void __launch_bounds__(kThreads)
norm_partial_kernel(const double* __restrict__ x, int64_t n, double* out2, double* partial,
                    unsigned* counter, const lsb_flags* gate, int it) {
  if (gated_off(gate, it)) return;
  double amax = 0.0, ssq = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[r];
    amax = fmax(amax, fabs(v));
    if (isnan(v)) amax = v;
    ssq = fma(v, v, ssq);
  }
  const double v[2] = {amax, ssq};
  const int op[2] = {1, 0};
  grid_reduce<2>(v, op, partial, counter, out2);
}

int launch_norm_partial(const double* x, int64_t n, double* out2, const lsb_workspace* ws,
                        const lsb_flags* gate, int it, cudaStream_t st) {
  norm_partial_kernel<<<row_grid(2 * n, 4), kThreads, 0, st>>>(x, n, out2, ws->partial,
                                                               ws->counter, gate, it);
  return check_launch("norm_partial");
}

// ||x|| from stacked (amax, ssq) partials.  In-range magnitudes use
// sqrt(sum x^2) directly; outside [2^-450, 2^450] every CTA re-reads x with
// an exact power-of-two scale (no rounding from the scaling itself), the
// overflow/underflow-safe path of the reference's amax-scaled norm.
__global__ void __launch_bounds__(kThreads)
norm_finish_kernel(const double* parts, int nparts, int stride, const double* __restrict__ x,
                   int64_t n, double* out, double* partial, unsigned* counter,
                   const lsb_flags* gate, int it) {
  if (gated_off(gate, it)) return;
  double amax = parts[0], ssq = parts[1];
  for (int q = 1; q < nparts; ++q) {
    amax = fmax(amax, parts[(int64_t)q * stride]);
    ssq += parts[(int64_t)q * stride + 1];
  }
  const double lo = 0x1p-450, hi = 0x1p450;
  if (amax == 0.0 || isnan(amax) || (amax >= lo && amax <= hi) || nparts > 1) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
      *out = amax == 0.0 ? 0.0 : (isnan(amax) ? amax : sqrt(ssq));
    return;
  }
  int e;
  frexp(amax, &e);
  const double s = ldexp(1.0, -e);
  double acc = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[r] * s;
    acc = fma(v, v, acc);
  }
  const double v[1] = {acc};
  const int op[1] = {0};
  __shared__ double res;
  if (grid_reduce<1>(v, op, partial, counter, &res)) {
    __syncthreads();
    if (threadIdx.x == 0) *out = sqrt(res) / s;
  }
}

int launch_norm_finish(const double* parts, int nparts, int stride, const double* x, int64_t n,
                       double* out, const lsb_workspace* ws, const lsb_flags* gate, int it,
                       cudaStream_t st) {
  norm_finish_kernel<<<row_grid(2 * n, 4), kThreads, 0, st>>>(parts, nparts, stride, x, n, out,
                                                              ws->partial, ws->counter, gate, it);
  return check_launch("norm_finish");
}

// Row-partitioned restart norm, second round (ranks > 1): from the gathered
// (amax, ssq) parts, when max|x| leaves [2^-450, 2^450] each rank forms its
// sum of (x * 2^-e)^2 with the exponent e of the GLOBAL amax (the same exact
// power-of-two scale on every rank), else 0.  The caller all-gathers that
// and finishes with lsb_norm_finish_scaled.
__device__ __forceinline__ bool norm_needs_rescale(const double* parts, int nparts, int stride,
                                                   double& amax, double& ssq) {
  amax = parts[0];
  ssq = parts[1];
  for (int q = 1; q < nparts; ++q) {
    amax = fmax(amax, parts[(int64_t)q * stride]);
    ssq += parts[(int64_t)q * stride + 1];
  }
  return !(amax == 0.0 || isnan(amax) || (amax >= 0x1p-450 && amax <= 0x1p450));
}

__global__ void __launch_bounds__(kThreads)
norm_scaled_partial_kernel(const double* parts, int nparts, int stride,
                           const double* __restrict__ x, int64_t n, double* out2,
                           double* partial, unsigned* counter) {
  double amax, ssq;
  const bool resc = norm_needs_rescale(parts, nparts, stride, amax, ssq);
  double acc = 0.0;
  if (resc) {
    int e;
    frexp(amax, &e);
    const double s = ldexp(1.0, -e);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
      const double v = x[r] * s;
      acc = fma(v, v, acc);
    }
  }
  const double v[2] = {acc, 0.0};
  const int op[2] = {0, 0};
  grid_reduce<2>(v, op, partial, counter, out2);
}

__global__ void norm_finish_scaled_kernel(const double* parts, const double* parts2, int nparts,
                                          int stride, int stride2, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double amax, ssq;
  if (!norm_needs_rescale(parts, nparts, stride, amax, ssq)) {
    *out = amax == 0.0 ? 0.0 : (isnan(amax) ? amax : sqrt(ssq));
    return;
  }
  int e;
  frexp(amax, &e);
  double q = parts2[0];
  for (int k = 1; k < nparts; ++k) q += parts2[(int64_t)k * stride2];
  *out = sqrt(q) / ldexp(1.0, -e);
}

int launch_norm_scaled_partial(const double* parts, int nparts, int stride, const double* x,
                               int64_t n, double* out2, const lsb_workspace* ws, cudaStream_t st) {
  norm_scaled_partial_kernel<<<row_grid(2 * n, 4), kThreads, 0, st>>>(
      parts, nparts, stride, x, n, out2, ws->partial, ws->counter);
  return check_launch("norm_scaled_partial");
}

int launch_norm_finish_scaled(const double* parts, const double* parts2, int nparts, int stride,
                              int stride2, double* out, cudaStream_t st) {
  norm_finish_scaled_kernel<<<1, 32, 0, st>>>(parts, parts2, nparts, stride, stride2, out);
  return check_launch("norm_finish_scaled");
}

// ------------------------------------------------------------------ scalings
__global__ void __launch_bounds__(kThreads)
scale_div_kernel(const double* __restrict__ x, int64_t n, const double* s, double* out,
                 const lsb_flags* gate, int it, int skip_if_broke) {
  if (gated_off(gate, it)) return;
  if (skip_if_broke && gate && gate->broke_iter == it) return;
  const double d = *s;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    out[r] = __ddiv_rn(x[r], d);
}

// 16-byte aligned x/out: row pairs, two pairs per thread per step (four
// 128-bit loads in flight; the scalar loop ran at ~0.69 of HBM)
__global__ void __launch_bounds__(kThreads)
scale_div2_kernel(const double* __restrict__ x, int64_t n, const double* s, double* out,
                  const lsb_flags* gate, int it, int skip_if_broke) {
  if (gated_off(gate, it)) return;
  if (skip_if_broke && gate && gate->broke_iter == it) return;
  const double d = *s;
  const int64_t npair = n / 2, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npair; j += 2 * stride) {
    const int64_t j2 = j + stride;
    const double2 a = ld2(x + 2 * j);
    const double2 b = j2 < npair ? ld2(x + 2 * j2) : make_double2(0.0, 0.0);
    st2(out + 2 * j, make_double2(__ddiv_rn(a.x, d), __ddiv_rn(a.y, d)));
    if (j2 < npair) st2(out + 2 * j2, make_double2(__ddiv_rn(b.x, d), __ddiv_rn(b.y, d)));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) out[n - 1] = __ddiv_rn(x[n - 1], d);
}

// out[e] = sum over ranks q (in rank order) of parts[q*stride + e]: the
// multi-rank completion of a reduction whose partials were all-gathered
// (the same fixed order as the small-state kernels' sums, small_body.cuh).
__global__ void sum_parts_kernel(const double* __restrict__ parts, int nparts, int stride,
                                 int count, double* __restrict__ out, const lsb_flags* gate,
                                 int it) {
  if (gated_off(gate, it)) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) {
    double v = parts[e];
    for (int q = 1; q < nparts; ++q) v += parts[(int64_t)q * stride + e];
    out[e] = v;
  }
}

int launch_sum_parts(const double* parts, int nparts, int stride, int count, double* out,
                     const lsb_flags* gate, int it, cudaStream_t st) {
  if (count <= 0) return LSB_OK;
  sum_parts_kernel<<<(count + 255) / 256, 256, 0, st>>>(parts, nparts, stride, count, out, gate,
                                                        it);
  return check_launch("sum_parts");
}

int launch_scale_div(const double* x, int64_t n, const double* s, double* out,
                     const lsb_flags* gate, int it, int skip_if_broke, cudaStream_t st) {
  if (n <= 0) return LSB_OK;
  if ((uintptr_t)x % 16 == 0 && (uintptr_t)out % 16 == 0) {
    static const int occ2 = wave(scale_div2_kernel, 0);
    scale_div2_kernel<<<row_grid(n / 2 + 1, occ2), kThreads, 0, st>>>(x, n, s, out, gate, it,
                                                                       skip_if_broke);
    return check_launch("scale_div2");
  }
  static const int occ_ = wave(scale_div_kernel, 2048);
  scale_div_kernel<<<row_grid(2 * n, occ_), kThreads, 0, st>>>(x, n, s, out, gate, it, skip_if_broke);
  return check_launch("scale_div");
}

// ------------------------------------------------------------------ extract (K10)
// x <- x + Mi (V_k y), k and y (coef2) produced on device by cycle_lsq
// (_extract, gmres.py:294-297).
__global__ void __launch_bounds__(kThreads)
extract_kernel(lsb_arnoldi S, double* __restrict__ x, const double* __restrict__ d) {
  const int k = S.flags->k;
  if (k < 1 || S.flags->status == LSB_SINGULAR) return;
  extern __shared__ double sy[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) sy[j] = S.coef2[j];
  __syncthreads();
  const int64_t ld = S.ld;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < S.n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
#pragma unroll 8
    for (int j = 0; j < k; ++j) acc = fma(sy[j], S.V[(int64_t)j * ld + r], acc);
    if (d) acc = __dmul_rn(acc, d[r]);
    x[r] = x[r] + acc;
  }
}

int launch_extract(const lsb_arnoldi& S, double* x, const double* d, cudaStream_t st) {
  static const int occ_ = wave(extract_kernel, 2048);
  extract_kernel<<<row_grid(2 * S.n, occ_), kThreads, coef_smem(S.cap), st>>>(S, x, d);
  return check_launch("extract");
}

// xt = x + Mi (V_k y) with k = it: the trial iterate of the true-residual
// probe (gmres.py:273-278).  y[0] NaN (singular trial) propagates.
__global__ void __launch_bounds__(kThreads)
trial_combine_kernel(lsb_arnoldi S, int it, const double* __restrict__ x,
                     const double* __restrict__ y, double* __restrict__ xt,
                     const double* __restrict__ d) {
  if (gated_off(S.flags, it)) return;
  extern __shared__ double sy[];
  const int k = it;
  for (int j = threadIdx.x; j < k; j += blockDim.x) sy[j] = y[j];
  __syncthreads();
  const int64_t ld = S.ld;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < S.n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
#pragma unroll 8
    for (int j = 0; j < k; ++j) acc = fma(sy[j], S.V[(int64_t)j * ld + r], acc);
    if (d) acc = __dmul_rn(acc, d[r]);
    xt[r] = x[r] + acc;
  }
}

int launch_trial_combine(const lsb_arnoldi& S, int it, const double* x, const double* y,
                         double* xt, const double* d, cudaStream_t st) {
  if (it < 1 || it >= S.cap) return LSB_ERANGE;
  static const int occ_ = wave(trial_combine_kernel, 2048);
  trial_combine_kernel<<<row_grid(2 * S.n, occ_), kThreads, coef_smem(S.cap), st>>>(S, it, x, y,
                                                                                  xt, d);
  return check_launch("trial_combine");
}

// lsb_preload: one kernel of this translation unit (its module)
const void* tu_anchor_update() { return (const void*)maxpy_kernel; }

}  // namespace lsb
