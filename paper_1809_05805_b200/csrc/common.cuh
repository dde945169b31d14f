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

// Same order for a row whose length C is a compile-time constant and whose
// products sit in a register array: every index is folded after unrolling,
// so nothing spills to local memory (the runtime-length np_row_sum on a
// register array forces the array into local memory).
template <int S, int N, int M>
__device__ __forceinline__ double np_pw_fixed(const double (&a)[M]) {
  if constexpr (N < 8) {
    double res = -0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) res = __dadd_rn(res, a[S + i]);
    return res;
  } else if constexpr (N <= 128) {
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = a[S + k];
#pragma unroll
    for (int i = 8; i < N - (N % 8); i += 8)
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[S + i + k]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
    for (int i = N - (N % 8); i < N; ++i) res = __dadd_rn(res, a[S + i]);
    return res;
  } else {
    constexpr int n2 = N / 2 - (N / 2) % 8;
    return __dadd_rn(np_pw_fixed<S, n2>(a), np_pw_fixed<S + n2, N - n2>(a));
  }
}

template <int C, int M>
__device__ __forceinline__ double np_row_sum_fixed(const double (&a)[M]) {
  if constexpr (C <= 0) return 0.0;
  else if constexpr (C == 1) return a[0];
  else return __dadd_rn(a[0], np_pw_fixed<1, C - 1>(a));
}

// ---------------------------------------------------------------- 27-point box rows
// The 27-point box stencil (offsets (dx,dy,dz) in {-1,0,1}^3, CSR column
// order o = (dz+1)*9 + (dy+1)*3 + (dx+1)).  With Dirichlet boundaries the
// present neighbours of a row are a sub-box fixed by one state per axis:
// bit 0 = the -1 neighbour exists, bit 1 = the +1 neighbour exists.  For
// each of the 4^3 state triples the compacted product list (and hence
// numpy's pairwise order over it) is a compile-time fact: box27_row<SX,SY,SZ>
// sums it fully unrolled in registers.
struct Box27Plan {
  int cnt;
  int idx[27];
};
__host__ __device__ constexpr Box27Plan box27_plan(int sx, int sy, int sz) {
  Box27Plan P{0, {}};
  for (int o = 0; o < 27; ++o) {
    const int d[3] = {o % 3 - 1, (o / 3) % 3 - 1, o / 9 - 1};
    const int s[3] = {sx, sy, sz};
    bool ok = true;
    for (int a = 0; a < 3; ++a) {
      if (d[a] < 0 && !(s[a] & 1)) ok = false;
      if (d[a] > 0 && !(s[a] & 2)) ok = false;
    }
    if (ok) P.idx[P.cnt++] = o;
  }
  return P;
}

// g(o): (already scaled) x at the neighbour of offset o; c(o): its
// coefficient (offsets in column order).
template <int SX, int SY, int SZ, class Gx, class Cf>
__device__ __forceinline__ double box27_row(const Gx& g, const Cf& c) {
  constexpr Box27Plan P = box27_plan(SX, SY, SZ);
  double q[P.cnt > 0 ? P.cnt : 1];
#pragma unroll
  for (int j = 0; j < P.cnt; ++j) q[j] = __dmul_rn(c(P.idx[j]), g(P.idx[j]));
  return np_row_sum_fixed<P.cnt>(q);
}

// state = sx + 4*sy + 16*sz -> box27_row<sx, sy, sz>
template <class Gx, class Cf>
__device__ __forceinline__ double box27_dispatch(int state, const Gx& g, const Cf& c) {
  if (state == 63) return box27_row<3, 3, 3>(g, c);   // interior: the hot case
  switch (state) {
#define LSB_B27(k) case k: return box27_row<((k) & 3), (((k) >> 2) & 3), ((k) >> 4)>(g, c);
#define LSB_B27x4(k) LSB_B27(k) LSB_B27(k + 1) LSB_B27(k + 2) LSB_B27(k + 3)
#define LSB_B27x16(k) LSB_B27x4(k) LSB_B27x4(k + 4) LSB_B27x4(k + 8) LSB_B27x4(k + 12)
    LSB_B27x16(0) LSB_B27x16(16) LSB_B27x16(32)
    LSB_B27x4(48) LSB_B27x4(52) LSB_B27x4(56) LSB_B27(60) LSB_B27(61) LSB_B27(62)
    default: return 0.0;
#undef LSB_B27x16
#undef LSB_B27x4
#undef LSB_B27
  }
}

// Two x-consecutive rows (ix even) of the 27-point box from the 9 (dz, dy)
// lines around them, v[l][0..3] = x[ix-1 .. ix+2] of line l = (dz+1)*3 +
// (dy+1).  Rows with both x neighbours share one plan (switch on the y/z
// state); x-edge pairs take the per-row dispatch.
template <int SY, int SZ, class Cf>
__device__ __forceinline__ void box27_pair_row(const double (&v)[9][4], const Cf& cf, double& y0,
                                               double& y1) {
  y0 = box27_row<3, SY, SZ>([&](int o) { return v[o / 3][o % 3]; }, cf);
  y1 = box27_row<3, SY, SZ>([&](int o) { return v[o / 3][o % 3 + 1]; }, cf);
}

template <class Cf>
__device__ __forceinline__ void box27_pair(const double (&v)[9][4], int sy, int sz, bool xm,
                                           bool xp, const Cf& cf, double& y0, double& y1) {
  if (xm && xp) {
    switch (sy | (sz << 2)) {
#define LSB_P27(k) case k: box27_pair_row<((k) & 3), ((k) >> 2)>(v, cf, y0, y1); break;
      LSB_P27(0) LSB_P27(1) LSB_P27(2) LSB_P27(3) LSB_P27(4) LSB_P27(5) LSB_P27(6)
      LSB_P27(7) LSB_P27(8) LSB_P27(9) LSB_P27(10) LSB_P27(11) LSB_P27(12) LSB_P27(13)
      LSB_P27(14)
#undef LSB_P27
      default: box27_pair_row<3, 3>(v, cf, y0, y1); break;
    }
  } else {
    const int s0 = (xm ? 1 : 0) | 2 | (sy << 2) | (sz << 4);
    const int s1 = 1 | (xp ? 2 : 0) | (sy << 2) | (sz << 4);
    y0 = box27_dispatch(s0, [&](int o) { return v[o / 3][o % 3]; }, cf);
    y1 = box27_dispatch(s1, [&](int o) { return v[o / 3][o % 3 + 1]; }, cf);
  }
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

// ---------------------------------------------------------------- peer signals
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int64_t ld_acquire_sys64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys64(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// spin until *sig >= e (acquire); false after timeout_ns (<= 0: 60 s)
__device__ inline bool spin_signal(const int64_t* sig, int64_t e, int64_t timeout_ns) {
  if (ld_acquire_sys64(sig) >= e) return true;
  const long long lim = timeout_ns > 0 ? timeout_ns : 60000000000LL;
  const unsigned long long t0 = gtimer_ns();
  unsigned k = 0;
  while (ld_acquire_sys64(sig) < e) {
    if ((++k & 255u) == 0 && (long long)(gtimer_ns() - t0) > lim) return false;
    __nanosleep(32);
  }
  return true;
}

// ---------------------------------------------------------------- launch helpers
int sm_count();
int check_launch(const char* what);
// launch status of an explicit launch (cudaLaunchKernelEx), else the last error
int check_launch(const char* what, cudaError_t launch_status);
int tuning(int key);

// Programmatic dependent launch (LSB_TUNE_PDL = 1): the per-iteration chain
// K1 -> K5 -> K2 -> K1 ... launches each kernel while its predecessor is
// still running; every such kernel starts with pdl_enter() -- wait for the
// predecessor's completion (and memory) before touching global memory, then
// let the successor launch.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Measured (tools/pdl_ab.py, C3 one-sync, L2 flushed): +4..6% at n = 2^20,
// +1..3% at 2^21..2^22, -1.3% at 2^24 and on the C2 cycle (fused K1 and K2
// fill the machine; early-resident waiting CTAs only get in the way) -- so
// auto = on below 2^23 rows.
inline bool use_pdl(int64_t n) {
  const int k = tuning(LSB_TUNE_PDL);
  return k == 1 || (k == 0 && n < ((int64_t)1 << 23));
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_chain(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                cudaStream_t st, Args... args) {
  if (!pdl) {
    k<<<grid, block, smem, st>>>(args...);
    return cudaSuccess;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace lsb
