// Grid-persistent cycle: iterations 0..m of a one-sync lagged GMRES(m)
// restart cycle (gmres.py:389-466 with mgs_lvl2, gram_schmidt.py:206-245)
// in ONE cooperative launch over every SM, for the sizes between the
// one-cluster persistent cycle (persist.cu: the basis must fit one cluster's
// shared memory) and the sizes where the per-iteration kernels stream HBM
// long enough to hide their launch and grid-reduction latencies.
//
// At those sizes (3D 32^3: n = 32,768, the basis 13.6 MB and resident in
// L2) an iteration of the per-iteration path is ~40 us of latency -- three
// launches, three grid-wide last-CTA reductions and the small-state
// kernel's chain of L2 round trips -- for ~15 MB of L2 traffic.  Here one
// grid of co-resident CTAs (cooperative launch) runs every iteration with
// five grid barriers per iteration:
//   (1) w = A u on every row (CSR, numpy's row order: bitwise the K7 bits)
//   (2) per-CTA partial [Q^T u, Q^T w] over the CTA's contiguous row block
//       (warp per column, lanes over rows, warp tree), written per CTA;
//       then G = the CTA partials summed by one warp per entry (lanes over
//       CTAs, butterfly: a fixed order, deterministic)
//   (3) CTA 0: the K5 small state -- mgs_small_body: beta,
//       breakdown test, T column, c = T^T y / beta, Hessenberg column and
//       the Givens fold, convergence flags (the same code as the
//       per-iteration kernel)
//   (4) K2 on every row: u /= beta, w = w / beta - Q c (lagged_update_kernel's
//       row expression)
// then the next iteration, unless the flags (read by every CTA after the
// barrier, so the decision is uniform) say the cycle stopped.  Only the
// mdot summation order differs from the per-iteration kernels (a per-CTA
// warp tree, then a CTA-ordered sum), so histories agree to rounding.
//
// V is read with plain (coherent) loads: it is written inside the same
// launch.  The cycle epilogue (least squares, extract, restart residual)
// stays with the per-cycle kernels, as for the cluster cycle.
#include <cooperative_groups.h>

#include "small_body.cuh"
#include "tile.cuh"

namespace lsb {

namespace cgg = cooperative_groups;

constexpr int kGT = 256;   // threads per CTA (= kSmall, the K5 body's block)
static_assert(kGT == kSmall, "the control CTA runs the K5 body with its own threads");

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// phase anatomy (LSB_TUNE_GRID_TRACE = 1; CTA 0's view: [3] = its sums and
// the wait for every CTA's, [4] = K5): CTA 0 thread 0 accumulates the
// globaltimer ns spent in each phase of every iteration; lsb_grid_trace
__device__ long long g_gtrace[8];

struct CsrRowAccG {          // the K7 product, x read coherently (written in-launch)
  const int32_t* col;
  const double* val;
  const double* x;
  const double* d;
  __device__ double operator()(int64_t j) const {
    const int64_t c = (int64_t)__ldg(col + j);
    double xv = ld_cg(x + c);
    if (d) xv = __dmul_rn(xv, __ldg(d + c));
    return __dmul_rn(__ldg(val + j), xv);
  }
};

__global__ void __launch_bounds__(kGT)
grid_cycle_kernel(lsb_arnoldi S, lsb_csr A, int ks, double* __restrict__ part, int64_t part_len,
                  int stage_uw, int trace) {
  cgg::grid_group grid = cgg::this_grid();
  extern __shared__ __align__(16) double dyn[];
  __shared__ SmallShared sh;
  __shared__ double cs[kSmall + 2];            // coefficients c (K2)
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  constexpr int kW = kGT / 32;
  const int cap = S.cap, m = S.m;
  const int64_t n = S.n, ld = S.ld;
  // CTA 0 is the control CTA (K5 and the Givens fold, no rows, so the fold
  // overlaps the others' K2); row CTAs 1..G-1 own contiguous row blocks
  const int GR = G - 1, br = b - 1;
  const int64_t per = (n + GR - 1) / GR;
  const int64_t r0 = b == 0 ? n : (int64_t)br * per, r1 = b == 0 ? n : min(n, r0 + per);
  const int nr = r1 > r0 ? (int)(r1 - r0) : 0;
  const int64_t gtid = b == 0 ? n : (int64_t)br * kGT + tid, gstride = (int64_t)GR * kGT;
  // shared memory: [u rows | w rows] of the block (stage_uw), then CTA 0's
  // resident small state -- R, T, the rotations, g, the triangle stay in
  // shared memory for the whole cycle, so K5 makes no global round trips
  // but the gathered G in and c, beta and the flags out
  double* su = dyn;
  double* sw = su + (stage_uw ? per : 0);
  double* st = dyn + (stage_uw ? ((2 * per + 1) & ~(int64_t)1) : 0);
  const StateLayout SL = StateLayout::make(cap, m);
  lsb_arnoldi L = S;
  L.R = st + SL.R; L.T = st + SL.T; L.tri = st + SL.tri; L.rot = st + SL.rot; L.g = st + SL.g;
  L.res = st + SL.res; L.coef = st + SL.coef; L.G = st + SL.G; L.scal = st + SL.scal;
  L.flags = reinterpret_cast<lsb_flags*>(st + SL.flags);
  L.g_parts = 1;
  if (b == 0) {
    copy_d(L.R, S.R, cap * cap);
    copy_d(L.T, S.T, cap * cap);
    copy_d(L.tri, S.tri, (m + 1) * m);
    copy_d(L.rot, S.rot, 2 * m);
    copy_d(L.g, S.g, m + 1);
    copy_d(L.res, S.res, m + 1);
    copy_d(L.coef, S.coef, cap);
    copy_d(L.scal, S.scal, LSB_S_COUNT);
    if (tid < (int)(sizeof(lsb_flags) / sizeof(int)))
      reinterpret_cast<int*>(L.flags)[tid] = reinterpret_cast<const int*>(S.flags)[tid];
    __syncthreads();
  }
  // arrival counter of phase (2b) (monotone: G per iteration), zeroed by
  // CTA 0 before the first grid barrier
  unsigned* arrive = reinterpret_cast<unsigned*>(part + part_len - 2);
  if (b == 0 && tid == 0) *arrive = 0u;
  bool bad = false;
  const bool tr = trace && b == 0 && tid == 0;
  long long tt[8] = {0};
  unsigned long long tm = tr ? gtimer_ns() : 0ull;
  auto mark = [&](int k) {
    if (tr) { const unsigned long long t = gtimer_ns(); tt[k] += (long long)(t - tm); tm = t; }
  };
  for (int i = 0; i <= m; ++i) {
    const int p = i + 1;
    if (gated_off(S.flags, i)) break;          // uniform: read after a grid barrier
    const double* u = S.V + (int64_t)(p - 1) * ld;
    double* w = S.V + (int64_t)p * ld;
    // (1) w = A u  (V.push(A v_i), gmres.py:411)
    for (int64_t r = gtid; r < n; r += gstride) {
      const int lo = __ldg(A.row_ptr + r), hi = __ldg(A.row_ptr + r + 1);
      const double s = np_row_sum(CsrRowAccG{A.col_idx + lo, A.values + lo, u, A.col_scale},
                                  hi - lo);
      if (!isfinite(s)) bad = true;
      w[r] = s;
    }
    mark(0);
    grid.sync();
    mark(1);
    // (2) this CTA's partial [Q^T u, Q^T w] (_lagged_reduce, gram_schmidt.py:195-203):
    // u and w rows of the block staged once, every column read once
    const double* pu = u + r0;
    const double* pw = w + r0;
    if (stage_uw && b > 0) {
      for (int j = tid; j < nr; j += kGT) {
        su[j] = ld_cg(u + r0 + j);
        sw[j] = ld_cg(w + r0 + j);
      }
      __syncthreads();
    }
    if (stage_uw) {
      pu = su;
      pw = sw;
    }
    for (int k = wid; k < p && b > 0; k += 2 * kW) {    // two columns per warp in flight
      const int k2 = k + kW;
      const double* q = S.V + (int64_t)k * ld + r0;
      const double* q2 = S.V + (int64_t)k2 * ld + r0;
      double a = 0.0, c = 0.0, a2 = 0.0, c2 = 0.0;
#pragma unroll 8
      for (int j = lane; j < nr; j += 32) {
        const double qv = ld_cg(q + j);
        const double qv2 = k2 < p ? ld_cg(q2 + j) : 0.0;
        const double uv = stage_uw ? pu[j] : ld_cg(pu + j);
        const double wv = stage_uw ? pw[j] : ld_cg(pw + j);
        a = fma(qv, uv, a);
        c = fma(qv, wv, c);
        a2 = fma(qv2, uv, a2);
        c2 = fma(qv2, wv, c2);
      }
      a = warp_sum(a);
      c = warp_sum(c);
      a2 = warp_sum(a2);
      c2 = warp_sum(c2);
      if (lane == 0 && b > 0) {
        part[(int64_t)(2 * k) * GR + br] = a;
        part[(int64_t)(2 * k + 1) * GR + br] = c;
        if (k2 < p) {
          part[(int64_t)(2 * k2) * GR + br] = a2;
          part[(int64_t)(2 * k2 + 1) * GR + br] = c2;
        }
      }
    }
    mark(2);
    grid.sync();
    // (2b) G[e] = the CTA partials of entry e summed by one warp (lanes over
    // CTAs, then the fixed butterfly): every warp of the grid takes entries,
    // so the 2p sums cost one L2 round trip instead of a serial CTA-0 loop
    for (int e = b * kW + wid; e < 2 * p; e += G * kW) {
      double v = 0.0;
      for (int c = lane; c < GR; c += 32) v += __ldcg(part + (int64_t)e * GR + c);
      v = warp_sum(v);
      if (lane == 0) S.G[e] = v;
    }
    // one-sided: every CTA signals its sums done; only CTA 0 (which needs
    // all of G) waits -- the others go straight on to barrier (4)
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(arrive, 1u);
    }
    mark(3);
    // (3) CTA 0: the K5 small state of iteration i on the resident state
    // (the Givens fold deferred to phase (4), where it overlaps K2), then
    // c, beta and the flags out for the other CTAs
    if (b == 0) {
      if (tid == 0) {
        const unsigned target = (unsigned)G * (unsigned)(i + 1);
        while (*((volatile unsigned*)arrive) < target) __nanosleep(20);
        __threadfence();
      }
      __syncthreads();
      for (int e = tid; e < 2 * p; e += kGT) L.G[e] = __ldcg(S.G + e);
      __syncthreads();
      mgs_small_body(L, sh, nullptr, i, p, ks, -i, false, /*resident=*/true);
      __syncthreads();
      for (int e = tid; e < p; e += kGT) S.coef[e] = L.coef[e];
      if (tid == 0) S.scal[LSB_S_BETA] = L.scal[LSB_S_BETA];
      if (tid < (int)(sizeof(lsb_flags) / sizeof(int)) && tid != 4)   // (nonfinite: OR-ed)
        reinterpret_cast<int*>(S.flags)[tid] = reinterpret_cast<const int*>(L.flags)[tid];
    }
    mark(4);
    grid.sync();
    mark(5);
    // (4) K2 rows unless iteration i broke down (lagged_update_kernel);
    // CTA 0 first folds Hessenberg column i-1 into the Givens state (the
    // pipeline2 deferral of gmres.py:444-462: a convergence it finds is in
    // the flags before barrier (5), so iteration i+1 never starts)
    const int broke = *((volatile const int*)&S.flags->broke_iter) == i;
    if (b == 0 && i >= 1) {
      for (int j = tid; j <= i; j += kGT) sh.col[j] = L.R[(int64_t)j * cap + i];
      __syncthreads();
      if (broke && tid == 0) sh.col[i] = 0.0;
      settle_block(L, sh, i, i, broke != 0);
      __syncthreads();
      if (tid < (int)(sizeof(lsb_flags) / sizeof(int)) && tid != 4)
        reinterpret_cast<int*>(S.flags)[tid] = reinterpret_cast<const int*>(L.flags)[tid];
    }
    if (!broke && b > 0) {
      for (int e = tid; e < p; e += kGT) cs[e] = __ldcg(S.coef + e);
      __syncthreads();
      const double beta = __ldcg(S.scal + LSB_S_BETA);
      const double cu = cs[p - 1];
      for (int64_t r = gtid; r < n; r += gstride) {
        double acc = 0.0;
        for (int k = 0; k < p - 1; ++k) acc = fma(cs[k], ld_cg(S.V + (int64_t)k * ld + r), acc);
        const double uu = __ddiv_rn(ld_cg(u + r), beta);
        const_cast<double*>(u)[r] = uu;
        acc = fma(cu, uu, acc);
        double ww = w[r];
        if (ks) ww = __ddiv_rn(ww, beta);
        w[r] = ww - acc;
      }
    }
    mark(6);
    grid.sync();
    mark(7);
    if (broke) break;
  }
  if (bad) atomicOr(&S.flags->nonfinite, 1);
  if (b == 0) {      // the resident small state back for the cycle epilogue kernels
    copy_d(S.R, L.R, cap * cap);
    copy_d(S.T, L.T, cap * cap);
    copy_d(S.tri, L.tri, (m + 1) * m);
    copy_d(S.rot, L.rot, 2 * m);
    copy_d(S.g, L.g, m + 1);
    copy_d(S.res, L.res, m + 1);
    copy_d(S.coef, L.coef, cap);
    copy_d(S.scal, L.scal, LSB_S_COUNT);
    if (tid < (int)(sizeof(lsb_flags) / sizeof(int)) && tid != 4)
      reinterpret_cast<int*>(S.flags)[tid] = reinterpret_cast<const int*>(L.flags)[tid];
    if (tid == 0 && L.flags->nonfinite) atomicOr(&S.flags->nonfinite, 1);
  }
  if (tr)
    for (int k = 0; k < 8; ++k) g_gtrace[k] += tt[k];
}

// n * cap doubles up to which the grid cycle is chosen over the
// per-iteration kernels (the engine asks lsb_cycle_grid_fits): the basis is
// then small enough that an iteration's HBM/L2 passes take a few us and the
// per-iteration path is dominated by launch and reduction latency.
constexpr int64_t kGridMaxElems = (int64_t)1 << 23;   // 8M doubles = 64 MB (in L2)

int grid_fits(int64_t n, int cap) {
  if (n < 1 || cap < 3 || cap > kSmall || n * (int64_t)cap > kGridMaxElems) return 0;
  // the control CTA's resident small state (lagged: m = cap - 2) must fit
  // its shared memory next to the staged u/w rows
  const StateLayout SL = StateLayout::make(cap, cap - 2);
  return sizeof(double) * (size_t)SL.total <= 136 * 1024;
}

int launch_cycle_grid(const lsb_arnoldi& S, const lsb_csr* A, int ks, double* part,
                      int64_t part_len, cudaStream_t st) {
  if (!A || S.g_parts != 1 || S.m + 2 > S.cap || A->n_rows != S.n || A->n_cols != S.n ||
      A->x_lo != 0 || A->row0 != 0 || !part)
    return LSB_ERANGE;
  if (!grid_fits(S.n, S.cap)) return LSB_ERANGE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(grid_cycle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr = true;
  }
  const StateLayout SL = StateLayout::make(S.cap, S.m);
  const size_t state_b = sizeof(double) * (size_t)SL.total;
  // CTAs per SM: LSB_TUNE_GRID_OCC (0: 1 -- fewer CTAs make every grid
  // barrier and the CTA-partial sums cheaper; the row work is small here)
  int occ = tuning(LSB_TUNE_GRID_OCC) > 0 ? tuning(LSB_TUNE_GRID_OCC) : 1;
  int G = 0, stage_uw = 0;
  size_t smem = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    G = sm_count() * occ;
    const int64_t rows_per = (S.n + kGT - 1) / kGT;   // no more row CTAs than row blocks of kGT
    if (G > rows_per + 1) G = (int)(rows_per + 1);
    if ((int64_t)2 * S.cap * G + 4 > part_len) G = (int)((part_len - 4) / (2 * S.cap));
    if (G < 2) return LSB_ERANGE;
    const int64_t per = (S.n + G - 2) / (G - 1);
    // u/w rows of a CTA's block staged in shared memory when they fit
    stage_uw = per * 2 * 8 <= 64 * 1024 ? 1 : 0;
    smem = state_b + (stage_uw ? sizeof(double) * (size_t)((2 * per + 1) & ~1LL) : 0);
    if (smem > 200 * 1024) return LSB_ERANGE;
    int fit = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, grid_cycle_kernel, kGT, smem);
    if (fit < 1) return LSB_ERANGE;
    if (fit >= occ) break;
    occ = fit;                   // fewer CTAs: larger blocks, recompute
  }
  // cooperative launch through cudaLaunchKernelEx: co-residency is
  // guaranteed (grid.sync) and the launch is capturable in the cycle graph
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)G);
  cfg.blockDim = dim3(kGT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int trace = tuning(LSB_TUNE_GRID_TRACE) == 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, grid_cycle_kernel, S, *A, ks, part, part_len,
                                           stage_uw, trace);
  return check_launch("cycle_grid", e);
}

int grid_trace(long long* out, int count) {
  if (count > 8) count = 8;
  if (cudaMemcpyFromSymbol(out, g_gtrace, sizeof(long long) * count) != cudaSuccess)
    return check_launch("grid_trace");
  static const long long zero[8] = {0};
  cudaMemcpyToSymbol(g_gtrace, zero, sizeof zero);
  return LSB_OK;
}

// lsb_preload: one kernel of this translation unit (its module)
const void* tu_anchor_gridcycle() { return (const void*)grid_cycle_kernel; }

}  // namespace lsb
