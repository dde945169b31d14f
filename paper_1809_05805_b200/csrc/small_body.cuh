// K5 small-state device code shared by the per-iteration kernels (small.cu)
// and the persistent cluster cycle (persist.cu).  Reference: see small.cu.
#pragma once
#include "reduce.cuh"

namespace lsb {

constexpr int kSmall = 256;  // threads; cap <= kSmall

__device__ __forceinline__ double gsum(const lsb_arnoldi& S, int e) {
  double v = S.G[e];
  for (int q = 1; q < S.g_parts; ++q) v += S.G[(int64_t)q * S.g_stride + e];
  return v;
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Copy an r x c block of a row-major global matrix (row stride src_ld)
// into shared memory (row stride dst_ld) with every thread keeping U loads
// in flight: a load-then-store loop leaves each thread one L2 round trip
// per element (ncu: the K5 kernel at p = 100 spent most of its 30 us on the
// T block copy).  All threads call it; no trailing barrier.
template <int U = 8>
__device__ __forceinline__ void stage_block(double* dst, int dst_ld, const double* src,
                                            int64_t src_ld, int r, int c) {
  const int tot = r * c;
  for (int base = threadIdx.x; base < tot; base += U * blockDim.x) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * blockDim.x;
      if (e < tot) {
        const int j = e / c, l = e - j * c;
        v[u] = src[(int64_t)j * src_ld + l];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * blockDim.x;
      if (e < tot) {
        const int j = e / c, l = e - j * c;
        dst[j * dst_ld + l] = v[u];
      }
    }
  }
}

// The cycle's small state laid out in one CTA's shared memory (the
// persistent cycles keep it resident there across iterations): offsets of
// the lsb_arnoldi arrays the K5 code touches.
struct StateLayout {
  int R, T, tri, rot, g, res, coef, G, scal, flags, total;   // offsets (doubles)
  __host__ __device__ static StateLayout make(int cap, int m) {
    StateLayout L{};
    int o = 0;
    L.R = o; o += cap * cap;
    L.T = o; o += cap * cap;
    L.tri = o; o += (m + 1) * m;
    L.rot = o; o += 2 * m;
    L.g = o; o += m + 1;
    L.res = o; o += m + 1;
    L.coef = o; o += cap;
    L.G = o; o += 2 * cap;
    L.scal = o; o += LSB_S_COUNT;
    L.flags = o; o += (int)(sizeof(lsb_flags) / sizeof(double));
    L.total = o;
    return L;
  }
};

__device__ __forceinline__ void copy_d(double* dst, const double* src, int n) {
  for (int e = threadIdx.x; e < n; e += blockDim.x) dst[e] = src[e];
}

struct SmallShared {
  double a[kSmall];     // G[:,0] / scaled
  double y[kSmall];     // G[:,1] / y
  double col[kSmall + 2];  // R column (r_col, then the Hessenberg column)
  double rot[2 * kSmall];
  double beta, tol;
  int broke;
};

// tol = btf * eps * sqrt(n) * hypot(r_diag, ||r_col||)   (gram_schmidt.py:96-100)
// ss_pre >= 0: ||r_col||^2 already reduced by the caller (persist.cu).
__device__ inline double breakdown_tol(const lsb_arnoldi& S, double r_diag, const double* rcol,
                                       int len, double ss_pre = -1.0) {
  double pre = r_diag;
  if (len > 0) {
    double ss = ss_pre;
    if (ss < 0.0) {
      ss = 0.0;
      for (int j = 0; j < len; ++j) ss = fma(rcol[j], rcol[j], ss);
    }
    pre = py_hypot(r_diag, sqrt(ss));
  }
  const double btf = S.scal[LSB_S_BTF];
  return __dmul_rn(__dmul_rn(__dmul_rn(btf, kEps), sqrt((double)S.n_global)), pre);
}

// Block-cooperative settle (gmres.py:427-435): Hessenberg column gc-1 is
// sh.col[0..gc] (= R[0..gc, gc], with R[gc,gc] = 0 after a breakdown);
// fold it into the Givens state, record |g[gc]|, stop on convergence or
// breakdown.  All threads must call it.
// resident: sh.rot already holds rotations 0..gc-2 (a persistent caller
// that ran every earlier fold of the cycle in this CTA).
__device__ inline void settle_block(const lsb_arnoldi& S, SmallShared& sh, int it, int gc,
                                    bool broke, bool resident = false) {
  const int t = threadIdx.x;
  if (!resident)
    for (int e = t; e < 2 * (gc - 1); e += blockDim.x) sh.rot[e] = S.rot[e];
  __syncthreads();
  if (t == 0) {
    const double res = givens_fold(sh.col, sh.rot, S.g, gc);
    S.rot[2 * (gc - 1)] = sh.rot[2 * (gc - 1)];
    S.rot[2 * (gc - 1) + 1] = sh.rot[2 * (gc - 1) + 1];
    S.res[gc] = res;
    const double target = S.scal[LSB_S_TARGET];
    if (res <= target || broke) {
      S.flags->stop_iter = it;
      S.flags->status = res <= target ? LSB_CONVERGED : LSB_BREAKDOWN;
    }
  }
  __syncthreads();
  for (int j = t; j <= gc; j += blockDim.x) S.tri[(int64_t)j * S.m + (gc - 1)] = sh.col[j];
}

// Shared front of both lagged kernels: gathered G, deferred norm beta,
// breakdown test against R[:p-1, p-1] (gram_schmidt.py:227-229 / 261-263).
__device__ inline bool lagged_front(const lsb_arnoldi& S, SmallShared& sh, int it, int p, int gc) {
  const int t = threadIdx.x, cap = S.cap;
  for (int e = t; e < p; e += blockDim.x) {
    sh.a[e] = gsum(S, 2 * e);
    sh.y[e] = gsum(S, 2 * e + 1);
    if (e < p - 1) sh.col[e] = S.R[(int64_t)e * cap + (p - 1)];
  }
  __syncthreads();
  if (t == 0) {
    const double bsq = sh.a[p - 1];
    const double beta = bsq > 0.0 ? sqrt(bsq) : 0.0;
    const double tol = breakdown_tol(S, beta, sh.col, p - 1);
    sh.beta = beta;
    sh.tol = tol;
    sh.broke = beta <= tol;
    S.scal[LSB_S_BETA] = beta;
    S.scal[LSB_S_TOL] = tol;
    if (sh.broke) {
      S.flags->broke_iter = it;
      if (gc == 0) { S.flags->stop_iter = it; S.flags->status = LSB_STARTUP_BREAKDOWN; }
      sh.col[p - 1] = 0.0;   // H[i, i-1] = 0 (gmres.py:416)
    } else {
      sh.col[p - 1] = beta;  // H[i, i-1] = R[i, i] = beta (gmres.py:418)
      S.R[(int64_t)(p - 1) * cap + (p - 1)] = beta;
    }
  }
  __syncthreads();
  return sh.broke;
}

// mgs_lvl2 small state (gram_schmidt.py:226-245 + gmres.py:418-435): one
// CTA, every thread calls it.  sT: p*p doubles of shared memory when
// use_smem (the T block), else unused.
__device__ inline void mgs_small_body(const lsb_arnoldi& S, SmallShared& sh, double* sT, int it,
                                      int p, int ks, int gc, bool use_smem,
                                      bool resident = false) {
  const int t = threadIdx.x, cap = S.cap;
  // The kernel is a chain of dependent L2 round trips, not work (ncu: ~2K
  // warp instructions in ~20K cycles): issue every independent load up
  // front -- the T block (not touched by lagged_front) and L1 prefetches of
  // the scalars, rotations and g that the breakdown test and the Givens
  // fold read later.
  const bool st = use_smem;
  if (st) stage_block(sT, p, S.T, cap, p - 1, p - 1);
  if (!resident) {   // (resident: the state is in shared memory already)
    if (t == 0) {
      prefetch_l1(S.scal);
      if (gc > 0) prefetch_l1(S.g + gc - 1);
    }
    if (gc > 1 && 16 * t < 2 * (gc - 1)) prefetch_l1(S.rot + 16 * t);
  }
  const bool broke = lagged_front(S, sh, it, p, gc);
  if (broke) {
    if (gc > 0) settle_block(S, sh, it, gc, true);
    return;
  }
  const double beta = sh.beta;
  // T block in shared memory when it fits (p x p, row stride p): the two
  // triangular mat-vecs then run at smem latency (launch sets the size)
  // T[:p-1, p-1] = -(T[:p-1, :p-1] @ (G[:p-1, 0] / beta));  T[p-1, p-1] = 1
  for (int e = t; e < p - 1; e += blockDim.x) sh.a[e] = __ddiv_rn(sh.a[e], beta);
  if (t == 0) sh.y[p - 1] = __ddiv_rn(sh.y[p - 1], beta);
  __syncthreads();
  for (int j = t; j < p - 1; j += blockDim.x) {
    double acc = 0.0;
    if (st) {
      for (int l = j; l < p - 1; ++l) acc = fma(sT[j * p + l], sh.a[l], acc);
      sT[j * p + (p - 1)] = -acc;
    } else {
      for (int l = j; l < p - 1; ++l) acc = fma(S.T[(int64_t)j * cap + l], sh.a[l], acc);
    }
    S.T[(int64_t)j * cap + (p - 1)] = -acc;
  }
  if (t == 0) {
    S.T[(int64_t)(p - 1) * cap + (p - 1)] = 1.0;
    if (st) {
      sT[(p - 1) * p + (p - 1)] = 1.0;
      for (int l = 0; l < p - 1; ++l) sT[(p - 1) * p + l] = 0.0;
    }
  }
  __syncthreads();
  // c = T[:p,:p]^T y  (/beta);  R[:p, p] = c
  for (int j = t; j < p; j += blockDim.x) {
    double acc = 0.0;
    if (st) {
      for (int l = 0; l <= j; ++l) acc = fma(sT[l * p + j], sh.y[l], acc);
    } else {
      for (int l = 0; l <= j; ++l) acc = fma(S.T[(int64_t)l * cap + j], sh.y[l], acc);
    }
    if (ks) acc = __ddiv_rn(acc, beta);
    S.coef[j] = acc;
    S.R[(int64_t)j * cap + p] = acc;
  }
  if (gc > 0) settle_block(S, sh, it, gc, false);
}

}  // namespace lsb
