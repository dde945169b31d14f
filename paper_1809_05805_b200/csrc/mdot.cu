// K1: fused tall-skinny mass inner product  out = X^T [u, w]  (FP64).
//
// Replaces mdot_pair / mass_inner_product / fused_mdot_norm / dot
// (reference kernels.py:275-347), whose numpy form reads X twice (two
// dgemv-T calls, kernels.py:345-346).  Here X is streamed from HBM exactly
// once:
//   * persistent CTAs walk row tiles of kTile rows;
//   * the tile of u (and w) is staged once in shared memory;
//   * warp `wp` owns columns k = wp, wp+8, ... and keeps one register
//     accumulator per (owned column, vector) across all its tiles, so the
//     per-tile work is 16 independent 128-bit loads per lane per column with
//     no shuffles at all;
//   * the CTA totals are butterfly-reduced once at the end and the last CTA
//     sums the per-CTA partials in a fixed order (deterministic).
#include "reduce.cuh"

namespace lsb {

constexpr int kTile = 1024;                  // rows per tile
constexpr int kLoads = kTile / 64;           // double2 loads per lane per column

__device__ __forceinline__ double2 ld_stream(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

template <int NV, int SLOTS>
__global__ void __launch_bounds__(kThreads, 2)
mdot_kernel(const double* __restrict__ X, int64_t ld, int64_t n, int p,
            const double* __restrict__ y0, const double* __restrict__ y1,
            double* __restrict__ out, double* __restrict__ partial, unsigned* counter,
            const lsb_flags* gate, int it) {
  if (gated_off(gate, it)) return;
  __shared__ __align__(16) double2 sy[NV][kTile / 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[SLOTS][NV];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s)
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[s][v] = 0.0;

  const int64_t ntiles = (n + kTile - 1) / kTile;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t r0 = t * kTile;
    const bool full = r0 + kTile <= n;
    // stage the u/w tile (coalesced, once per tile)
    for (int j = threadIdx.x; j < kTile / 2; j += kThreads) {
      const int64_t r = r0 + 2 * j;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double* y = v == 0 ? y0 : y1;
        double2 val;
        if (full) {
          val = *reinterpret_cast<const double2*>(y + r);
        } else {
          val.x = r < n ? y[r] : 0.0;
          val.y = r + 1 < n ? y[r + 1] : 0.0;
        }
        sy[v][j] = val;
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int k = warp + kWarps * s;
      if (k < p) {
        const double* col = X + (int64_t)k * ld + r0;
        double a[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) a[v] = 0.0;
        if (full) {
          double2 xv[kLoads];
#pragma unroll
          for (int q = 0; q < kLoads; ++q) xv[q] = ld_stream(col + 2 * (lane + 32 * q));
#pragma unroll
          for (int q = 0; q < kLoads; ++q) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const double2 yy = sy[v][lane + 32 * q];
              a[v] = fma(xv[q].x, yy.x, a[v]);
              a[v] = fma(xv[q].y, yy.y, a[v]);
            }
          }
        } else {
          for (int q = 0; q < kLoads; ++q) {
            const int j = lane + 32 * q;
            const int64_t r = r0 + 2 * j;
            const double xa = r < n ? col[2 * j] : 0.0;
            const double xb = r + 1 < n ? col[2 * j + 1] : 0.0;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const double2 yy = sy[v][j];
              a[v] = fma(xa, yy.x, a[v]);
              a[v] = fma(xb, yy.y, a[v]);
            }
          }
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[s][v] += a[v];
      }
    }
    __syncthreads();
  }

  // CTA partials: one butterfly per owned (column, vector)
  const int G = gridDim.x;
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const int k = warp + kWarps * s;
    if (k < p) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double x = warp_sum(acc[s][v]);
        if (lane == 0) partial[(size_t)(k * NV + v) * G + blockIdx.x] = x;
      }
    }
  }
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == (unsigned)G - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int E = p * NV;
  for (int e = warp; e < E; e += kWarps) {
    double x = 0.0;
    for (int c = lane; c < G; c += 32) x += __ldcg(partial + (size_t)e * G + c);
    x = warp_sum(x);
    if (lane == 0) out[e] = x;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

template <int NV, int SLOTS>
static int launch_mdot_t(const double* X, int64_t ld, int64_t n, int p, const double* u,
                         const double* w, double* out, const lsb_workspace* ws,
                         const lsb_flags* gate, int it, cudaStream_t st) {
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mdot_kernel<NV, SLOTS>, kThreads, 0);
    if (occ < 1) occ = 1;
  }
  const int64_t ntiles = (n + kTile - 1) / kTile;
  int64_t grid = (int64_t)sm_count() * occ;
  if (ws->grid > 0 && ws->grid < grid) grid = ws->grid;
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  mdot_kernel<NV, SLOTS><<<(unsigned)grid, kThreads, 0, st>>>(X, ld, n, p, u, w, out, ws->partial,
                                                             ws->counter, gate, it);
  return check_launch("mdot");
}

template <int NV>
static int launch_mdot_nv(const double* X, int64_t ld, int64_t n, int p, const double* u,
                          const double* w, double* out, const lsb_workspace* ws,
                          const lsb_flags* gate, int it, cudaStream_t st) {
  if (p <= 8) return launch_mdot_t<NV, 1>(X, ld, n, p, u, w, out, ws, gate, it, st);
  if (p <= 16) return launch_mdot_t<NV, 2>(X, ld, n, p, u, w, out, ws, gate, it, st);
  if (p <= 32) return launch_mdot_t<NV, 4>(X, ld, n, p, u, w, out, ws, gate, it, st);
  if (p <= 64) return launch_mdot_t<NV, 8>(X, ld, n, p, u, w, out, ws, gate, it, st);
  return launch_mdot_t<NV, 16>(X, ld, n, p, u, w, out, ws, gate, it, st);
}

constexpr int kMaxCols = 128;

int launch_mdot(const double* X, int64_t ld, int64_t n, int p, const double* u, const double* w,
                double* out, const lsb_workspace* ws, const lsb_flags* gate, int it,
                cudaStream_t st) {
  if (p <= 0) return LSB_OK;
  if (n <= 0) {  // empty vectors: all products are zero
    cudaMemsetAsync(out, 0, sizeof(double) * p * (w ? 2 : 1), st);
    return check_launch("mdot-empty");
  }
  // column chunks of kMaxCols (one launch each, sequential on the stream)
  const int nv = w ? 2 : 1;
  for (int k0 = 0; k0 < p; k0 += kMaxCols) {
    const int pc = p - k0 < kMaxCols ? p - k0 : kMaxCols;
    const double* Xc = X + (int64_t)k0 * ld;
    double* oc = out + (int64_t)k0 * nv;
    int rc = w ? launch_mdot_nv<2>(Xc, ld, n, pc, u, w, oc, ws, gate, it, st)
               : launch_mdot_nv<1>(Xc, ld, n, pc, u, w, oc, ws, gate, it, st);
    if (rc) return rc;
  }
  return LSB_OK;
}

}  // namespace lsb
