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
grid_cycle_kernel(lsb_arnoldi S, lsb_csr A, int ks, double* __restrict__ part, int use_smem) {
  cgg::grid_group grid = cgg::this_grid();
  extern __shared__ double sT[];               // CTA 0: the T block for K5
  __shared__ SmallShared sh;
  __shared__ double cs[kSmall + 2];            // coefficients c (K2)
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, wid = tid >> 5;
  constexpr int kW = kGT / 32;
  const int64_t n = S.n, ld = S.ld;
  // this CTA's contiguous row block for the reductions
  const int64_t per = (n + G - 1) / G;
  const int64_t r0 = (int64_t)b * per, r1 = min(n, r0 + per);
  const int64_t gtid = (int64_t)b * kGT + tid, gstride = (int64_t)G * kGT;
  bool bad = false;
  for (int i = 0; i <= S.m; ++i) {
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
    grid.sync();
    // (2) this CTA's partial [Q^T u, Q^T w] (_lagged_reduce, gram_schmidt.py:195-203)
    for (int k = wid; k < p; k += kW) {
      const double* q = S.V + (int64_t)k * ld;
      double a = 0.0, c = 0.0;
      for (int64_t r = r0 + lane; r < r1; r += 32) {
        const double qv = ld_cg(q + r);
        a = fma(qv, ld_cg(u + r), a);
        c = fma(qv, ld_cg(w + r), c);
      }
      a = warp_sum(a);
      c = warp_sum(c);
      if (lane == 0) {
        part[(int64_t)(2 * k) * G + b] = a;
        part[(int64_t)(2 * k + 1) * G + b] = c;
      }
    }
    grid.sync();
    // (2b) G[e] = the CTA partials of entry e summed by one warp (lanes over
    // CTAs, then the fixed butterfly): every warp of the grid takes entries,
    // so the 2p sums cost one L2 round trip instead of a serial CTA-0 loop
    for (int e = b * kW + wid; e < 2 * p; e += G * kW) {
      double v = 0.0;
      for (int c = lane; c < G; c += 32) v += __ldcg(part + (int64_t)e * G + c);
      v = warp_sum(v);
      if (lane == 0) S.G[e] = v;
    }
    grid.sync();
    // (3) CTA 0: the K5 small state of iteration i
    if (b == 0) mgs_small_body(S, sh, sT, i, p, ks, i, use_smem != 0);
    grid.sync();
    // (4) K2 rows unless iteration i broke down (lagged_update_kernel)
    const int broke = *((volatile const int*)&S.flags->broke_iter) == i;
    if (!broke) {
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
    grid.sync();
    if (broke) break;
  }
  if (bad) S.flags->nonfinite = 1;
}

// n * cap doubles up to which the grid cycle is chosen over the
// per-iteration kernels (the engine asks lsb_cycle_grid_fits): the basis is
// then small enough that an iteration's HBM/L2 passes take a few us and the
// per-iteration path is dominated by launch and reduction latency.
constexpr int64_t kGridMaxElems = (int64_t)1 << 23;   // 8M doubles = 64 MB (in L2)

int grid_fits(int64_t n, int cap) {
  return n >= 1 && cap >= 2 && cap <= kSmall && n * (int64_t)cap <= kGridMaxElems;
}

int launch_cycle_grid(const lsb_arnoldi& S, const lsb_csr* A, int ks, double* part,
                      int64_t part_len, cudaStream_t st) {
  if (!A || S.g_parts != 1 || S.m + 2 > S.cap || A->n_rows != S.n || A->n_cols != S.n ||
      A->x_lo != 0 || A->row0 != 0 || !part)
    return LSB_ERANGE;
  if (!grid_fits(S.n, S.cap)) return LSB_ERANGE;
  constexpr size_t kMaxT = 160 * 1024;
  const size_t need = sizeof(double) * (size_t)S.cap * S.cap;
  const int use = need <= kMaxT;
  const size_t smem = use ? need : 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(grid_cycle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMaxT);
    attr = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_cycle_kernel, kGT, smem);
  if (occ < 1) return LSB_ERANGE;
  if (occ > 2) occ = 2;
  int G = sm_count() * occ;
  const int64_t rows_per = (S.n + kGT - 1) / kGT;   // no more CTAs than row blocks of kGT
  if (G > rows_per) G = (int)(rows_per > 0 ? rows_per : 1);
  if ((int64_t)2 * S.cap * G > part_len) G = (int)(part_len / (2 * S.cap));
  if (G < 1) return LSB_ERANGE;
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
  const cudaError_t e = cudaLaunchKernelEx(&cfg, grid_cycle_kernel, S, *A, ks, part, use);
  return check_launch("cycle_grid", e);
}

// lsb_preload: one kernel of this translation unit (its module)
const void* tu_anchor_gridcycle() { return (const void*)grid_cycle_kernel; }

}  // namespace lsb
