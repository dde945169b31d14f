// Shared device helpers for liblsb200 (sm_100a).
//
// Bit-fidelity helpers: the reference (pure numpy + CPython floats) never
// contracts a*b+c into an FMA, so every expression that must reproduce the
// reference bit for bit is written with __dmul_rn/__dadd_rn/__dsub_rn/
// __ddiv_rn, which nvcc never fuses.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/lsb200.h"

namespace lsb {

constexpr double kEps = 2.220446049250313e-16;  // np.finfo(np.float64).eps
constexpr int kNoStop = 0x7fffffff;

// ---------------------------------------------------------------- gate
// Cycle kernels receive the device flag block and their iteration number;
// once the solver has stopped (converged / breakdown) at iteration d, every
// kernel of an iteration > d returns immediately.  That keeps a whole
// restart cycle launchable as one CUDA graph with zero host syncs.
__device__ __forceinline__ bool gated_off(const lsb_flags* f, int it) {
  if (f == nullptr || it < 0) return false;
  const int stop = *((volatile const int*)&f->stop_iter);
  const int broke = *((volatile const int*)&f->broke_iter);
  // an earlier breakdown also stops later iterations (with a deferred
  // Givens fold the stop flag itself may land one iteration late)
  return stop < it || (broke >= 0 && broke < it);
}

// ---------------------------------------------------------------- warp sums
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------- numpy pairwise
// numpy's add.reduceat sums a row segment a[0..cnt) as
//   a[0] + pairwise(a[1..cnt))
// with pairwise() from numpy/_core/src/umath/loops_utils.h.src:
//   n < 8      : res = -0.0; res += a[i] sequentially
//   n <= 128   : 8 strided accumulators, tree ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//                then the n%8 tail sequentially
//   n > 128    : split at n2 = n/2 - (n/2)%8 and recurse.
// Acc is any functor returning the j-th product (already rounded).
template <class Acc>
__device__ double np_pairwise_block(const Acc& a, int64_t s, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a(s + i));
    return res;
  }
  double r0 = a(s + 0), r1 = a(s + 1), r2 = a(s + 2), r3 = a(s + 3);
  double r4 = a(s + 4), r5 = a(s + 5), r6 = a(s + 6), r7 = a(s + 7);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = __dadd_rn(r0, a(s + i + 0)); r1 = __dadd_rn(r1, a(s + i + 1));
    r2 = __dadd_rn(r2, a(s + i + 2)); r3 = __dadd_rn(r3, a(s + i + 3));
    r4 = __dadd_rn(r4, a(s + i + 4)); r5 = __dadd_rn(r5, a(s + i + 5));
    r6 = __dadd_rn(r6, a(s + i + 6)); r7 = __dadd_rn(r7, a(s + i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < n; ++i) res = __dadd_rn(res, a(s + i));
  return res;
}

template <class Acc>
__device__ double np_pairwise(const Acc& a, int64_t s, int64_t n) {
  if (n <= 128) return np_pairwise_block(a, s, n);
  // explicit stack instead of recursion: leaves are visited left to right and
  // combined exactly as the recursive definition does (post-order).
  struct Frame { int64_t s, n; int state; double left; };
  Frame st[48];
  int top = 0;
  st[0] = {s, n, 0, 0.0};
  double ret = 0.0;
  while (top >= 0) {
    Frame& f = st[top];
    if (f.n <= 128) { ret = np_pairwise_block(a, f.s, f.n); --top; continue; }
    int64_t n2 = f.n / 2; n2 -= n2 % 8;
    if (f.state == 0) { f.state = 1; st[top + 1] = {f.s, n2, 0, 0.0}; ++top; continue; }
    if (f.state == 1) { f.left = ret; f.state = 2; st[top + 1] = {f.s + n2, f.n - n2, 0, 0.0}; ++top; continue; }
    ret = __dadd_rn(f.left, ret);
    --top;
  }
  return ret;
}

// Row sum exactly as np.add.reduceat: first element + pairwise(rest).
template <class Acc>
__device__ __forceinline__ double np_row_sum(const Acc& a, int64_t cnt) {
  if (cnt <= 0) return 0.0;
  double first = a(0);
  if (cnt == 1) return first;
  return __dadd_rn(first, np_pairwise(a, 1, cnt - 1));
}

// ---------------------------------------------------------------- CPython hypot
// math.hypot(a, b) of CPython 3.12 (Modules/mathmodule.c vector_norm):
// lossless scaling to [0.5, 1), double-length squares and sums, one
// differential correction.  Reproduced operation by operation so the Givens
// rotations and breakdown tolerances match the reference bit for bit.
__device__ __forceinline__ void dl_mul(double x, double y, double& hi, double& lo) {
  hi = __dmul_rn(x, y);
  lo = fma(x, y, -hi);
}
__device__ __forceinline__ void dl_fast_sum(double a, double b, double& hi, double& lo) {
  hi = __dadd_rn(a, b);
  lo = __dadd_rn(__dsub_rn(a, hi), b);
}
__device__ inline double py_vector_norm2(double x0, double x1, double mx) {
  if (isinf(mx)) return mx;
  if (isnan(x0) || isnan(x1)) return nan("");
  if (mx == 0.0) return mx;
  int e;
  frexp(mx, &e);
  double pre = 1.0;
  if (e < -1023) {  // subnormal max: rescale by DBL_MIN first
    const double dmin = 2.2250738585072014e-308;
    x0 = x0 / dmin; x1 = x1 / dmin; mx = mx / dmin; pre = dmin;
    frexp(mx, &e);
  }
  double scale = ldexp(1.0, -e);
  double csum = 1.0, frac1 = 0.0, frac2 = 0.0, hi, lo, shi, slo;
  double xs[2] = {x0, x1};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    double x = __dmul_rn(xs[i], scale);
    dl_mul(x, x, hi, lo);
    dl_fast_sum(csum, hi, shi, slo);
    csum = shi;
    frac1 = __dadd_rn(frac1, lo);
    frac2 = __dadd_rn(frac2, slo);
  }
  double h = sqrt(__dadd_rn(__dsub_rn(csum, 1.0), __dadd_rn(frac1, frac2)));
  dl_mul(-h, h, hi, lo);
  dl_fast_sum(csum, hi, shi, slo);
  csum = shi;
  frac1 = __dadd_rn(frac1, lo);
  frac2 = __dadd_rn(frac2, slo);
  double x = __dadd_rn(__dsub_rn(csum, 1.0), __dadd_rn(frac1, frac2));
  h = __dadd_rn(h, __ddiv_rn(x, __dmul_rn(2.0, h)));
  return __dmul_rn(pre, __ddiv_rn(h, scale));
}
__device__ inline double py_hypot(double a, double b) {
  a = fabs(a); b = fabs(b);
  double mx = a > b ? a : b;
  if (isnan(a)) mx = a;
  return py_vector_norm2(a, b, mx);
}

// ---------------------------------------------------------------- Givens
// gmres.py:143-177: rotation() + givens_update() on column h[0..i] (i>=1),
// every product and sum rounded separately as CPython/numpy scalars do.
__device__ inline double givens_fold(double* h, double* rot, double* g, int i) {
  for (int k = 0; k < i - 1; ++k) {
    const double c = rot[2 * k], s = rot[2 * k + 1];
    const double hk = h[k], hk1 = h[k + 1];
    const double t = __dadd_rn(__dmul_rn(c, hk), __dmul_rn(s, hk1));
    h[k + 1] = __dadd_rn(__dmul_rn(-s, hk), __dmul_rn(c, hk1));
    h[k] = t;
  }
  const double a = h[i - 1], b = h[i];
  double c, s;
  if (b == 0.0) { c = 1.0; s = 0.0; }
  else if (a == 0.0) { c = 0.0; s = 1.0; }
  else { const double r = py_hypot(a, b); c = __ddiv_rn(a, r); s = __ddiv_rn(b, r); }
  h[i - 1] = __dadd_rn(__dmul_rn(c, a), __dmul_rn(s, b));
  h[i] = 0.0;
  rot[2 * (i - 1)] = c;
  rot[2 * (i - 1) + 1] = s;
  const double gi = g[i - 1];
  g[i - 1] = __dmul_rn(c, gi);
  g[i] = __dmul_rn(-s, gi);
  return fabs(g[i]);
}

// ---------------------------------------------------------------- launch helpers
int sm_count();
int check_launch(const char* what);

}  // namespace lsb
