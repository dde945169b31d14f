// K6 / K7: SpMV feeding the Arnoldi loop, bitwise equal to the reference.
//
// The reference (kernels.py:256-272) forms the products values*x[col]
// unfused and sums each row with np.add.reduceat, i.e. first product plus
// numpy's pairwise sum of the rest (common.cuh np_row_sum).  Both kernels
// reproduce that order with non-contracting intrinsics, so y matches the
// reference bit for bit (tests/test_gpu_parity.py).
//
// K6 is matrix-free: a constant-coefficient box stencil (5-point 2D,
// 7-point and 27-point 3D) whose offsets are given in CSR column order; it
// moves 16 B/row of compulsory HBM traffic instead of CSR's ~12*nnz/n + 20.
// The 7-point and 27-point operators work on row pairs with 128-bit loads;
// the 27-point rows pick their present-neighbour sub-box at compile time
// (common.cuh box27_row) so products and pairwise sums stay in registers.
// Other layouts take the generic per-row path.  K7 is a general CSR kernel
// with 32-bit indices: a warp stages the products of 32 consecutive rows in
// shared memory from coalesced col/value streams, then every lane sums its
// own row in numpy's order.
#include <cuda.h>

#include <algorithm>

#include "tile.cuh"

namespace lsb {

struct StencilK {
  int nx, ny, nz, noff, halo_lo, halo_hi;
  int dx[LSB_MAX_OFF], dy[LSB_MAX_OFF], dz[LSB_MAX_OFF];
  int lin[LSB_MAX_OFF];
  double val[LSB_MAX_OFF];
  const double* d;
  FastDiv fx, fy;
  int zlo, zhi;    // valid neighbour z range: [zlo, zhi] (halo planes included)
  int rx, ry, rz;  // stencil reach per axis
};

struct ArrAcc {
  const double* a;
  __device__ double operator()(int64_t j) const { return a[j]; }
};

__device__ __forceinline__ double ldx(const StencilK& K, const double* __restrict__ x, int64_t c) {
  double v = __ldg(x + c);
  if (K.d) v = __dmul_rn(v, __ldg(K.d + c));
  return v;
}

// Any subset of neighbours present (boundary rows): packed local array.
template <int NOFF>
__device__ __noinline__ double stencil_row_generic(const StencilK& K, const double* __restrict__ x,
                                                   int ix, int iy, int iz, int64_t r) {
  double packed[LSB_MAX_OFF];
  int cnt = 0;
  const int noff = NOFF > 0 ? NOFF : K.noff;
  for (int o = 0; o < noff; ++o) {
    const int jx = ix + K.dx[o], jy = iy + K.dy[o], jz = iz + K.dz[o];
    if (jx >= 0 && jx < K.nx && jy >= 0 && jy < K.ny && jz >= K.zlo && jz <= K.zhi)
      packed[cnt++] = __dmul_rn(K.val[o], ldx(K, x, r + K.lin[o]));
  }
  return np_row_sum(ArrAcc{packed}, cnt);
}

// All NOFF neighbours present: products stay in registers.
template <int NOFF>
__device__ __forceinline__ double stencil_row_interior(const StencilK& K,
                                                       const double* __restrict__ x, int64_t r) {
  double prod[NOFF];
#pragma unroll
  for (int o = 0; o < NOFF; ++o) prod[o] = __dmul_rn(K.val[o], ldx(K, x, r + K.lin[o]));
  return np_row_sum(ArrAcc{prod}, NOFF);
}

template <int NOFF>
__global__ void __launch_bounds__(256)
stencil_kernel(const StencilK K, const double* __restrict__ x, const double* __restrict__ b,
               double* __restrict__ y, lsb_flags* flags, int it) {
  if (gated_off(flags, it)) return;
  const uint32_t n = (uint32_t)K.nx * K.ny * K.nz;
  // reach of the stencil along each axis (1 for all shipped operators)
  bool bad = false;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const uint32_t line = K.fx.div(r);
    const int ix = (int)(r - line * (uint32_t)K.nx);
    const uint32_t iz = K.fy.div(line);
    const int iy = (int)(line - iz * (uint32_t)K.ny);
    const bool interior = NOFF > 0 && ix - K.rx >= 0 && ix + K.rx < K.nx && iy - K.ry >= 0 &&
                          iy + K.ry < K.ny && (int)iz - K.rz >= K.zlo && (int)iz + K.rz <= K.zhi;
    double s;
    if (interior && NOFF > 0)
      s = stencil_row_interior<(NOFF > 0 ? NOFF : 1)>(K, x, r);
    else
      s = stencil_row_generic<NOFF>(K, x, ix, iy, (int)iz, r);
    if (!isfinite(s)) bad = true;
    y[r] = b ? __dsub_rn(b[r], s) : s;
  }
  if (bad && flags) flags->nonfinite = 1;
}

// 27-point box operator (offsets {-1,0,1}^3 in column order): one row per
// thread, the row's present-neighbour sub-box picked by box27_dispatch so the
// 27 products and numpy's pairwise sum stay in registers (the generic
// stencil_kernel<27> kept them in local memory: 204 GB/s at 256^3).
__global__ void __launch_bounds__(256)
stencil27_kernel(const StencilK K, const double* __restrict__ x, const double* __restrict__ b,
                 double* __restrict__ y, lsb_flags* flags, int it) {
  if (gated_off(flags, it)) return;
  const uint32_t n = (uint32_t)K.nx * K.ny * K.nz;
  bool bad = false;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const uint32_t line = K.fx.div(r);
    const int ix = (int)(r - line * (uint32_t)K.nx);
    const uint32_t iz = K.fy.div(line);
    const int iy = (int)(line - iz * (uint32_t)K.ny);
    const int state = (ix >= 1) | ((ix + 1 < K.nx) << 1) | ((iy >= 1) << 2) |
                      ((iy + 1 < K.ny) << 3) | (((int)iz - 1 >= K.zlo) << 4) |
                      (((int)iz + 1 <= K.zhi) << 5);
    const double s = box27_dispatch(
        state, [&](int o) { return ldx(K, x, (int64_t)r + K.lin[o]); },
        [&](int o) { return K.val[o]; });
    if (!isfinite(s)) bad = true;
    y[r] = b ? __dsub_rn(b[r], s) : s;
  }
  if (bad && flags) flags->nonfinite = 1;
}

// Same operator on row pairs (nx even, x 16-byte aligned, no column scale):
// each of the 9 (dz, dy) lines is loaded once for both rows as one LDG.128
// plus two LDG.64 from a line base pointer (immediate offsets), 27 loads per
// two rows instead of 54 loads with a 64-bit address each.  Absent lines
// (Dirichlet planes / edges) are not loaded; the row's plan never reads them.
// Work items are split so warps do not diverge on the x edges: first the
// interior pairs of every x-line (ix = 2 .. nx-4, both rows have both x
// neighbours: one shared plan), then the two edge pairs of every line.
__device__ __forceinline__ void load27_pair(const double* __restrict__ x, int64_t r,
                                            int64_t nx, int64_t plane, int sy, int sz,
                                            bool xm, bool xp, double (&v)[9][4]) {
#pragma unroll
  for (int l = 0; l < 9; ++l) {
    const int dz = l / 3 - 1, dy = l % 3 - 1;
    const bool pres = (dy < 0 ? (sy & 1) : dy > 0 ? (sy & 2) : 1) &&
                      (dz < 0 ? (sz & 1) : dz > 0 ? (sz & 2) : 1);
    const double* base = x + r + dz * plane + dy * nx;
    double2 c2 = make_double2(0.0, 0.0);
    v[l][0] = v[l][3] = 0.0;
    if (pres) {
      c2 = __ldg(reinterpret_cast<const double2*>(base));
      if (xm) v[l][0] = __ldg(base - 1);
      if (xp) v[l][3] = __ldg(base + 2);
    }
    v[l][1] = c2.x;
    v[l][2] = c2.y;
  }
}

// 128-thread CTAs: at ~94 registers a 256-thread CTA fits twice per SM
// (16 warps); 128-thread CTAs fit five times (20 warps) -- more warps to
// hide the FP64 and load latency of the unfused products.
constexpr int kS27Threads = 128;

__global__ void __launch_bounds__(kS27Threads)
stencil27_pair_kernel(const StencilK K, FastDiv fint, const double* __restrict__ x,
                      const double* __restrict__ b, double* __restrict__ y, lsb_flags* flags,
                      int it) {
  if (gated_off(flags, it)) return;
  const uint32_t lines = (uint32_t)K.ny * K.nz;
  const uint32_t nint = K.nx >= 6 ? (uint32_t)(K.nx / 2 - 2) : 0u;  // interior pairs per line
  const uint32_t items_int = lines * nint, items = items_int + 2u * lines;
  const int64_t nx = K.nx, plane = (int64_t)K.nx * K.ny;
  auto cf = [&](int o) { return K.val[o]; };
  bool bad = false;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < items; i += gridDim.x * blockDim.x) {
    uint32_t line;
    int ix;
    if (i < items_int) {
      line = fint.div(i);
      ix = 2 + 2 * (int)(i - line * nint);
    } else {
      const uint32_t e = i - items_int;
      line = e >> 1;
      ix = (e & 1) ? K.nx - 2 : 0;
    }
    const uint32_t iz = K.fy.div(line);
    const int iy = (int)(line - iz * (uint32_t)K.ny);
    const int64_t r = (int64_t)line * nx + ix;
    const int sy = (iy >= 1) | ((iy + 1 < K.ny) << 1);
    const int sz = ((int)iz - 1 >= K.zlo) | (((int)iz + 1 <= K.zhi) << 1);
    const bool xm = ix >= 1, xp = ix + 2 < K.nx;
    double v[9][4];
    load27_pair(x, r, nx, plane, sy, sz, xm, xp, v);
    double y0, y1;
    box27_pair(v, sy, sz, xm, xp, cf, y0, y1);
    if (!isfinite(y0) || !isfinite(y1)) bad = true;
    double2 out;
    if (b) {
      const double2 bb = *reinterpret_cast<const double2*>(b + r);
      out = make_double2(__dsub_rn(bb.x, y0), __dsub_rn(bb.y, y1));
    } else {
      out = make_double2(y0, y1);
    }
    *reinterpret_cast<double2*>(y + r) = out;
  }
  if (bad && flags) flags->nonfinite = 1;
}

// z-marching variant (2.5D blocking in registers): a thread owns one row
// pair position (ix, iy) and walks a chunk of consecutive planes.  The nine
// (dz, dy) lines of a pair overlap those of the next plane's pair in six
// lines, which stay in registers (v[l] for dz = 0, +1 become dz = -1, 0);
// each step loads only the three dz = +1 lines -- 9 loads per row pair
// instead of 27.  Products, plans and summation order are the pair
// kernel's (box27_pair), so y is bitwise the same.
constexpr int kS27MarchZ = 16;   // planes per work item

__device__ __forceinline__ void load27_lines(const double* __restrict__ x, int64_t r, int64_t nx,
                                             int sy, bool pres_z, bool xm, bool xp,
                                             double (&v)[9][4], int l0) {
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy) {
    const int l = l0 + dy + 1;
    const bool pres = pres_z && (dy < 0 ? (sy & 1) : dy > 0 ? (sy & 2) : 1);
    const double* base = x + r + dy * nx;
    double2 c2 = make_double2(0.0, 0.0);
    v[l][0] = v[l][3] = 0.0;
    if (pres) {
      c2 = __ldg(reinterpret_cast<const double2*>(base));
      if (xm) v[l][0] = __ldg(base - 1);
      if (xp) v[l][3] = __ldg(base + 2);
    }
    v[l][1] = c2.x;
    v[l][2] = c2.y;
  }
}

// Interior march (both x and y neighbours present, every plane of the chunk
// has its z-1 and z+1 planes): the same products and order as box27_pair's
// interior case, with no per-plane dispatch or presence predicates, and the
// three plane buffers rotated by unrolling the plane loop by three instead of
// copying six lines of registers per plane (those moves were a fifth of the
// generic march's instructions).
template <class Cf>
__device__ __forceinline__ void march27_interior(const double* __restrict__ x,
                                                 const double* __restrict__ b,
                                                 double* __restrict__ y, int64_t r00, int64_t nx,
                                                 int64_t plane, int z0, int z1, const Cf& cf,
                                                 bool& bad) {
  double A[3][4], B[3][4], Q[3][4];
  auto load = [&](double (&d)[3][4], int64_t r) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const double* base = x + r + dy * nx;
      const double2 c2 = __ldg(reinterpret_cast<const double2*>(base));
      d[dy + 1][0] = __ldg(base - 1);
      d[dy + 1][1] = c2.x;
      d[dy + 1][2] = c2.y;
      d[dy + 1][3] = __ldg(base + 2);
    }
  };
  auto step = [&](const double (&m)[3][4], const double (&c)[3][4], double (&p)[3][4], int iz) {
    const int64_t r = r00 + (int64_t)iz * plane;
    load(p, r + plane);
    auto g0 = [&](int o) {
      const int l = o / 3, k = o % 3;
      return l < 3 ? m[l][k] : (l < 6 ? c[l - 3][k] : p[l - 6][k]);
    };
    auto g1 = [&](int o) {
      const int l = o / 3, k = o % 3 + 1;
      return l < 3 ? m[l][k] : (l < 6 ? c[l - 3][k] : p[l - 6][k]);
    };
    const double y0 = box27_row<3, 3, 3>(g0, cf);
    const double y1 = box27_row<3, 3, 3>(g1, cf);
    if (!isfinite(y0) || !isfinite(y1)) bad = true;
    double2 out;
    if (b) {
      const double2 bb = *reinterpret_cast<const double2*>(b + r);
      out = make_double2(__dsub_rn(bb.x, y0), __dsub_rn(bb.y, y1));
    } else {
      out = make_double2(y0, y1);
    }
    *reinterpret_cast<double2*>(y + r) = out;
  };
  load(A, r00 + (int64_t)(z0 - 1) * plane);
  load(B, r00 + (int64_t)z0 * plane);
  for (int iz = z0; iz < z1; iz += 3) {
    step(A, B, Q, iz);
    if (iz + 1 >= z1) break;
    step(B, Q, A, iz + 1);
    if (iz + 2 >= z1) break;
    step(Q, A, B, iz + 2);
  }
}

__global__ void __launch_bounds__(kS27Threads, 4)
stencil27_march_kernel(const StencilK K, FastDiv fint, const double* __restrict__ x,
                       const double* __restrict__ b, double* __restrict__ y, lsb_flags* flags,
                       int it, int nzc, int tuning_fast27) {
  if (gated_off(flags, it)) return;
  // work items: (z chunk, line in plane, pair slot); interior pairs of the
  // line first (one shared plan), then the two x-edge pairs -- as the pair
  // kernel, so warps do not diverge on the x edges
  const uint32_t nint = K.nx >= 6 ? (uint32_t)(K.nx / 2 - 2) : 0u;
  const uint32_t per_line = nint + 2u;
  const uint32_t lines = (uint32_t)K.ny;                 // lines of one plane
  const uint32_t items_int = (uint32_t)nzc * lines * nint;
  const uint32_t items = items_int + 2u * (uint32_t)nzc * lines;
  const int64_t nx = K.nx, plane = (int64_t)K.nx * K.ny;
  auto cf = [&](int o) { return K.val[o]; };
  bool bad = false;
  (void)per_line;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < items; i += gridDim.x * blockDim.x) {
    uint32_t zc, iy;
    int ix;
    if (i < items_int) {
      const uint32_t q = fint.div(i);               // (zc, iy) index
      ix = 2 + 2 * (int)(i - q * nint);
      zc = q / lines;
      iy = q - zc * lines;
    } else {
      const uint32_t e = i - items_int;
      const uint32_t q = e >> 1;
      ix = (e & 1) ? K.nx - 2 : 0;
      zc = q / lines;
      iy = q - zc * lines;
    }
    const int z0 = (int)zc * kS27MarchZ;
    const int z1 = min(K.nz, z0 + kS27MarchZ);
    const int sy = ((int)iy >= 1) | (((int)iy + 1 < K.ny) << 1);
    const bool xm = ix >= 1, xp = ix + 2 < K.nx;
    const int64_t r00 = (int64_t)iy * nx + ix;       // row of (ix, iy) in plane 0
    if (xm && xp && sy == 3 && z0 - 1 >= K.zlo && z1 <= K.zhi && tuning_fast27) {
      march27_interior(x, b, y, r00, nx, plane, z0, z1, cf, bad);
      continue;
    }
    double v[9][4];
    // lines of planes z0-1 (dz = -1) and z0 (dz = 0)
    load27_lines(x, r00 + (int64_t)(z0 - 1) * plane, nx, sy, z0 - 1 >= K.zlo, xm, xp, v, 0);
    load27_lines(x, r00 + (int64_t)z0 * plane, nx, sy, true, xm, xp, v, 3);
    for (int iz = z0; iz < z1; ++iz) {
      const int64_t r = r00 + (int64_t)iz * plane;
      load27_lines(x, r + plane, nx, sy, iz + 1 <= K.zhi, xm, xp, v, 6);
      const int sz = (iz - 1 >= K.zlo) | ((iz + 1 <= K.zhi) << 1);
      double y0, y1;
      box27_pair(v, sy, sz, xm, xp, cf, y0, y1);
      if (!isfinite(y0) || !isfinite(y1)) bad = true;
      double2 out;
      if (b) {
        const double2 bb = *reinterpret_cast<const double2*>(b + r);
        out = make_double2(__dsub_rn(bb.x, y0), __dsub_rn(bb.y, y1));
      } else {
        out = make_double2(y0, y1);
      }
      *reinterpret_cast<double2*>(y + r) = out;
#pragma unroll
      for (int l = 0; l < 6; ++l)
#pragma unroll
        for (int c = 0; c < 4; ++c) v[l][c] = v[l + 3][c];
    }
  }
  if (bad && flags) flags->nonfinite = 1;
}

// ---------------------------------------------------------------- 27-point plane tiles (TMA)
// A CTA owns a 32 x 16 (x, y) tile of rows and marches a chunk of planes.
// Each plane's tile plus its one-row halo (36 x 18 doubles) lands in shared
// memory by ONE 3-D tensor copy (cp.async.bulk.tensor, OOB zero-filled --
// absent neighbours are never read by the row plans, so the fill value does
// not matter), issued `kT27Stages` planes ahead into a ring: the plane loads
// never sit on a thread's critical path (the z-march kernel above stalls on
// them: ncu long-scoreboard 4.4 of 8.6 cycles per instruction).  A thread
// owns one row pair (ix, ix+1) of the tile and keeps the (dz, dy) lines of
// the previous two planes in registers, so each step reads only the new
// plane's three lines from shared memory (8 + 16 + 8 bytes per line).
// Products, plans and summation order are box27_pair's: y is bitwise the
// same as every other 27-point kernel.  NEG: the 20 edge/corner
// coefficients are exactly -1.0, so their products are exact negations
// folded into the DADDs (the same bits as __dmul_rn(-1.0, x)): 7 DMUL + 26
// DADD per interior row instead of 27 + 26.
#ifndef LSB_T27_STAGES
#define LSB_T27_STAGES 6
#endif
constexpr int kT27X = 32, kT27Y = 8;
constexpr int kT27Threads = (kT27X / 2) * kT27Y;                  // 256: one row pair each
// a tensor copy's inner start must be 16-byte aligned (an odd x start traps
// with an illegal instruction -- tools/micro/tma3d.cu), so a smem row holds
// x0-2 .. x0+33 and a pair reads its four x values as 8 + 16 + 8 bytes
constexpr int kT27RowD = kT27X + 4;
constexpr int kT27PlaneB = kT27RowD * (kT27Y + 2) * 8;            // 5184 B per staged plane
constexpr int kT27PlaneD = (kT27PlaneB + 127) / 128 * 128 / 8;    // 128-byte aligned slots
constexpr int kT27Stages = LSB_T27_STAGES;
constexpr size_t kT27Smem = (size_t)kT27Stages * kT27PlaneD * 8 + 128 + 2 * kT27Stages * 8;

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__host__ __device__ constexpr bool box27_face_or_centre(int o) {
  return o == 4 || o == 10 || o == 12 || o == 13 || o == 14 || o == 16 || o == 22;
}

// The rows of the 27-point box with at least one neighbour missing, as row
// pairs (ix even): the two x-edge pairs of every line, the y-edge lines'
// x-interior pairs, and the x/y-interior pairs of a z-edge plane (one with
// no neighbour plane below / above, i.e. no ghost plane there).  A
// grid-stride loop of the calling CTAs, row-pair kernel style (global
// loads, box27_pair): ~3% of the rows at 256^3.
__device__ __forceinline__ void stencil27_boundary_rows(const StencilK& K, const double* __restrict__ x,
                                                     const double* __restrict__ b,
                                                     double* __restrict__ y, lsb_flags* flags,
                                                     unsigned cta, unsigned ctas) {
  const int64_t nx = K.nx, plane = (int64_t)K.nx * K.ny;
  const uint32_t nxi = (uint32_t)(K.nx / 2 - 2);               // x-interior pairs per line
  const uint32_t nX = 2u * (uint32_t)K.ny * (uint32_t)K.nz;
  const uint32_t nyl = K.ny >= 2 ? 2u : 1u;                     // y-edge lines per plane
  const uint32_t nY = nyl * (uint32_t)K.nz * nxi;
  const int zb0 = K.zlo == 0 ? 0 : -1;                          // z-edge planes (-1: none)
  const int zb1 = (K.zhi == K.nz - 1 && K.nz - 1 != zb0) ? K.nz - 1 : -1;
  const uint32_t nzp = (zb0 >= 0) + (zb1 >= 0);
  const uint32_t lyi = K.ny >= 2 ? (uint32_t)(K.ny - 2) : 0u;   // y-interior lines
  const uint32_t nZ = nzp * lyi * nxi;
  auto cf = [&](int o) { return K.val[o]; };
  bool bad = false;
  for (uint32_t i = cta * blockDim.x + threadIdx.x; i < nX + nY + nZ; i += ctas * blockDim.x) {
    int ix, iy, iz;
    if (i < nX) {
      const uint32_t line = i >> 1;
      ix = (i & 1) ? K.nx - 2 : 0;
      iz = (int)(line / (uint32_t)K.ny);
      iy = (int)(line - (uint32_t)iz * K.ny);
    } else if (i < nX + nY) {
      const uint32_t e = i - nX, q = e / nxi;
      ix = 2 + 2 * (int)(e - q * nxi);
      iz = (int)(q / nyl);
      iy = (q - (uint32_t)iz * nyl) ? K.ny - 1 : 0;
    } else {
      const uint32_t e = i - nX - nY, q = e / nxi;
      ix = 2 + 2 * (int)(e - q * nxi);
      const uint32_t pz = q / lyi;
      iy = 1 + (int)(q - pz * lyi);
      iz = (pz == 0 && zb0 >= 0) ? zb0 : zb1;
    }
    const int64_t r = (int64_t)iz * plane + (int64_t)iy * nx + ix;
    const int sy = (iy >= 1) | ((iy + 1 < K.ny) << 1);
    const int sz = (iz - 1 >= K.zlo) | ((iz + 1 <= K.zhi) << 1);
    const bool xm = ix >= 1, xp = ix + 2 < K.nx;
    double v[9][4];
    load27_pair(x, r, nx, plane, sy, sz, xm, xp, v);
    double y0, y1;
    box27_pair(v, sy, sz, xm, xp, cf, y0, y1);
    if (!isfinite(y0) || !isfinite(y1)) bad = true;
    double2 out;
    if (b) {
      const double2 bb = __ldg(reinterpret_cast<const double2*>(b + r));
      out = make_double2(__dsub_rn(bb.x, y0), __dsub_rn(bb.y, y1));
    } else {
      out = make_double2(y0, y1);
    }
    *reinterpret_cast<double2*>(y + r) = out;
  }
  if (bad && flags) flags->nonfinite = 1;
}

template <bool NEG, bool HASB>
__global__ void __launch_bounds__(kT27Threads, 4)
stencil27_tile_kernel(const __grid_constant__ CUtensorMap tm, const StencilK K,
                      const double* __restrict__ x, const double* __restrict__ b,
                      double* __restrict__ y, lsb_flags* flags, int it, int zc, int tiles_x,
                      int nbnd) {
  if (gated_off(flags, it)) return;
  if (blockIdx.y == 0) {                 // the boundary rows (first, so they are not a tail)
    if ((int)blockIdx.x < nbnd) stencil27_boundary_rows(K, x, b, y, flags, blockIdx.x, nbnd);
    return;
  }
  // all shared memory dynamic, the plane slots 128-byte aligned by hand (the
  // tensor copy's destination alignment); offsetting the shared array itself
  // (not a cast integer) keeps the reads LDS rather than generic loads
  extern __shared__ __align__(128) double t27_raw[];
  double* const t27_smem = t27_raw + ((128u - (smem_u32(t27_raw) & 127u)) & 127u) / 8u;
  uint64_t* const full = reinterpret_cast<uint64_t*>(t27_smem + kT27Stages * kT27PlaneD);
  uint64_t* const empty = full + kT27Stages;   // slot read by all 8 warps
  const int tx = (int)blockIdx.x % tiles_x, ty = (int)blockIdx.x / tiles_x;
  const int z0 = ((int)blockIdx.y - 1) * zc, z1 = min(K.nz, z0 + zc);
  const int x0 = tx * kT27X, y0 = ty * kT27Y;
  const int lx = 2 * ((int)threadIdx.x & 15), ly = (int)threadIdx.x >> 4;
  const int ix = x0 + lx, iy = y0 + ly;
  const int nload = z1 - z0 + 2;                           // planes z0-1 .. z1
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kT27Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kT27Threads / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int k) {                                 // load k = plane z0-1+k
    uint64_t* bar = &full[k % kT27Stages];
    mbar_arrive_tx(bar, (unsigned)kT27PlaneB);
    tma_load_3d(t27_smem + (k % kT27Stages) * kT27PlaneD, &tm, x0 - 2, y0 - 1,
                z0 - 1 + k - K.zlo, bar);
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < kT27Stages && k < nload; ++k) issue(k);
  auto read = [&](double (&d)[3][4], int k) {
    mbar_wait(&full[k % kT27Stages], (unsigned)(k / kT27Stages) & 1u);
    const double* row = t27_smem + (k % kT27Stages) * kT27PlaneD + ly * kT27RowD + lx + 1;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const double2 c = *reinterpret_cast<const double2*>(row + l * kT27RowD + 1);
      d[l][0] = row[l * kT27RowD];
      d[l][1] = c.x; d[l][2] = c.y;
      d[l][3] = row[l * kT27RowD + 3];
    }
    // a slot is read exactly once (the z-window then lives in registers):
    // each warp releases it right away (arrive = release semantics)
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[k % kT27Stages]);
  };
  // no CTA barrier per plane: thread 0 refills the slot of load t-1 (read by
  // every warp at its step t-3) with load t-1+S before reading its own plane
  auto refill = [&](int t) {
    const int j = t - 1;
    if (threadIdx.x == 0 && j >= 0 && j + kT27Stages < nload) {
      mbar_wait(&empty[j % kT27Stages], (unsigned)(j / kT27Stages) & 1u);
      issue(j + kT27Stages);
    }
  };
  const int64_t nx = K.nx, plane = (int64_t)K.nx * K.ny;
  bool bad = false;
  unsigned emax = 0;
  double* const yrow = y + (int64_t)iy * nx + ix;
  const double* const brow = HASB ? b + (int64_t)iy * nx + ix : nullptr;
  auto emit = [&](int iz, double y0v, double y1v) {
    // non-finite test on the exponent bits (integer pipe; a DSETP would
    // take FP64 issue slots from the row sums): the largest exponent field
    // seen, compared once at the end (all ones = Inf/NaN)
    emax = max(emax, max((unsigned)__double2hiint(y0v) & 0x7ff00000u,
                         (unsigned)__double2hiint(y1v) & 0x7ff00000u));
    const int64_t r = (int64_t)iz * plane;
    double2 out;
    if (HASB) {      // residual form b - A x: a compile-time branch
      const double2 bb = __ldg(reinterpret_cast<const double2*>(brow + r));
      out = make_double2(__dsub_rn(bb.x, y0v), __dsub_rn(bb.y, y1v));
    } else {
      out = make_double2(y0v, y1v);
    }
    *reinterpret_cast<double2*>(yrow + r) = out;
  };
  auto mul = [&](int o, double v) {
    if (NEG && !box27_face_or_centre(o)) return -v;
    return __dmul_rn(K.val[o], v);
  };
  // interior rows only (all 26 neighbours present: the fixed interior plan,
  // plane buffers rotated by a 3-way unrolled loop -- no register moves);
  // the boundary rows are the blockIdx.y == 0 CTAs' work
  const bool xy_int = ix >= 1 && ix + 2 < K.nx && iy >= 1 && iy + 1 < K.ny;
  double A[3][4], B[3][4], Q[3][4];
  auto step = [&](const double (&m)[3][4], const double (&c)[3][4], double (&p)[3][4], int t) {
    refill(t);
    read(p, t + 2);
    const int iz = z0 + t;
    if (xy_int && iz - 1 >= K.zlo && iz + 1 <= K.zhi) {
      constexpr Box27Plan P = box27_plan(3, 3, 3);
      double q0[27], q1[27];
#pragma unroll
      for (int j = 0; j < 27; ++j) {
        const int o = P.idx[j], l = o / 3, k = o % 3;
        const double v0 = l < 3 ? m[l][k] : (l < 6 ? c[l - 3][k] : p[l - 6][k]);
        const double v1 = l < 3 ? m[l][k + 1] : (l < 6 ? c[l - 3][k + 1] : p[l - 6][k + 1]);
        q0[j] = mul(o, v0);
        q1[j] = mul(o, v1);
      }
      emit(iz, np_row_sum_fixed<27>(q0), np_row_sum_fixed<27>(q1));
    }
  };
  read(A, 0);
  read(B, 1);
  const int nt = z1 - z0;
  for (int t = 0; t < nt; t += 3) {
    step(A, B, Q, t);
    if (t + 1 >= nt) break;
    step(B, Q, A, t + 1);
    if (t + 2 >= nt) break;
    step(Q, A, B, t + 2);
  }
  if ((bad || emax == 0x7ff00000u) && flags) flags->nonfinite = 1;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the
// library links no libcuda).
typedef CUresult (*t27_encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static t27_encode_fn t27_encoder() {
  static t27_encode_fn f = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      return (t27_encode_fn) nullptr;
    return reinterpret_cast<t27_encode_fn>(p);
  }();
  return f;
}

// Launch the tile kernel; returns false (nothing launched) when the tensor
// map cannot be encoded, so the caller falls back to the z-march.
static bool launch_stencil27_tile(const StencilK& K, const double* x, const double* b, double* y,
                                  lsb_flags* flags, int it, cudaStream_t st) {
  t27_encode_fn enc = t27_encoder();
  if (!enc) return false;
  const int64_t plane = (int64_t)K.nx * K.ny;
  const int nplanes = K.zhi - K.zlo + 1;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)K.nx, (cuuint64_t)K.ny, (cuuint64_t)nplanes};
  const cuuint64_t strides[2] = {(cuuint64_t)K.nx * 8, (cuuint64_t)plane * 8};
  const cuuint32_t box[3] = {(cuuint32_t)kT27RowD, (cuuint32_t)(kT27Y + 2), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)(x + (int64_t)K.zlo * plane), dims,
          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  bool neg = true;
  for (int o = 0; o < 27; ++o)
    if (!box27_face_or_centre(o) && K.val[o] != -1.0) neg = false;
  const int tiles_x = (K.nx + kT27X - 1) / kT27X, tiles_y = (K.ny + kT27Y - 1) / kT27Y;
  // plane chunk: the longest of 64/32/16 planes that still fills one wave
  // of tile CTAs (4 per SM; at 256^3: 64 planes 0.0745 ms, 32 0.0757, 16 0.0784)
  const int64_t txy = (int64_t)tiles_x * tiles_y, slots = 4LL * sm_count();
  int zc = tuning(LSB_TUNE_S27_TILE_Z);
  if (zc <= 0) {
    zc = 16;
    for (int c : {64, 32})
      if (txy * ((K.nz + c - 1) / c) >= slots) { zc = c; break; }
  }
  const int nch = (K.nz + zc - 1) / zc;
  // boundary-row CTAs (grid row 0, dispatched first): as few as keep them
  // off the critical path -- each holds a tile slot for the whole run, so
  // 256 of them at 256^3 cost 5% (0.0784 vs 0.0743 ms with 64); their
  // latency-bound gathers get ~32 row pairs per thread at 256^3, scaled
  // with n (the tile phase's length), at least 4
  const int64_t nxi = K.nx / 2 - 2, lyi = K.ny >= 2 ? K.ny - 2 : 0;
  const int zb0 = K.zlo == 0 ? 0 : -1;
  const int nzp = (zb0 >= 0) + ((K.zhi == K.nz - 1 && K.nz - 1 != zb0) ? 1 : 0);
  const int64_t nbp = 2LL * K.ny * K.nz + (K.ny >= 2 ? 2 : 1) * (int64_t)K.nz * nxi +
                      (int64_t)nzp * lyi * nxi;
  const int64_t n = (int64_t)K.nx * K.ny * K.nz;
  const int64_t ipt = std::max<int64_t>(4, (32 * n) >> 24);
  const int64_t nb = std::min<int64_t>(txy, std::max<int64_t>(1, (nbp + kT27Threads * ipt - 1) /
                                                                     (kT27Threads * ipt)));
  const dim3 grid((unsigned)txy, (unsigned)nch + 1);   // y = 0: boundary rows
  auto go = [&](auto kern) {
    kern<<<grid, kT27Threads, kT27Smem, st>>>(tm, K, x, b, y, flags, it, zc, tiles_x, (int)nb);
  };
  if (neg)
    b ? go(stencil27_tile_kernel<true, true>) : go(stencil27_tile_kernel<true, false>);
  else
    b ? go(stencil27_tile_kernel<false, true>) : go(stencil27_tile_kernel<false, false>);
  return true;
}

static bool canonical27(const lsb_stencil* S) {
  if (S->noff != 27) return false;
  for (int o = 0; o < 27; ++o)
    if (S->dx[o] != o % 3 - 1 || S->dy[o] != (o / 3) % 3 - 1 || S->dz[o] != o / 9 - 1) return false;
  return true;
}

// 7-point operator on row pairs (nx even): 5 x LDG.128 + 2 x LDG.64 per
// two rows instead of 14 scalar loads.  Offsets in column order:
// -plane, -nx, -1, 0, +1, +nx, +plane.
__global__ void __launch_bounds__(256)
stencil7_pair_kernel(const StencilK K, const double* __restrict__ x, const double* __restrict__ b,
                     double* __restrict__ y, lsb_flags* flags, int it) {
  if (gated_off(flags, it)) return;
  const uint32_t n = (uint32_t)K.nx * K.ny * K.nz;
  const uint32_t npair = n >> 1;
  const int nx = K.nx, plane = K.nx * K.ny;
  const double c0 = K.val[0], c1 = K.val[1], c2 = K.val[2], c3 = K.val[3], c4 = K.val[4],
               c5 = K.val[5], c6 = K.val[6];
  bool bad = false;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < npair; j += gridDim.x * blockDim.x) {
    const uint32_t r = 2 * j;
    const uint32_t line = K.fx.div(r);
    const int ix = (int)(r - line * (uint32_t)nx);
    const uint32_t iz = K.fy.div(line);
    const int iy = (int)(line - iz * (uint32_t)K.ny);
    // presence of each neighbour (Dirichlet: absent terms are dropped, so
    // the row sum is first present product + sequential sum of the rest,
    // numpy's n < 8 pairwise order).  Branch-free, registers only.
    const bool pzm = (int)iz - 1 >= K.zlo, pzp = (int)iz + 1 <= K.zhi;
    const bool pym = iy >= 1, pyp = iy + 1 < K.ny;
    const bool pxm = ix >= 1, pxp = ix + 2 < nx;
    const double2 z2 = make_double2(0.0, 0.0);
    const double2 zm = pzm ? __ldg(reinterpret_cast<const double2*>(x + r - plane)) : z2;
    const double2 ym = pym ? __ldg(reinterpret_cast<const double2*>(x + r - nx)) : z2;
    const double xm = pxm ? __ldg(x + r - 1) : 0.0;
    const double2 cc = __ldg(reinterpret_cast<const double2*>(x + r));
    const double xp = pxp ? __ldg(x + r + 2) : 0.0;
    const double2 yp = pyp ? __ldg(reinterpret_cast<const double2*>(x + r + nx)) : z2;
    const double2 zp = pzp ? __ldg(reinterpret_cast<const double2*>(x + r + plane)) : z2;
    double f0 = 0.0, a0 = -0.0, f1 = 0.0, a1 = -0.0;
    bool h0 = false, h1 = false;
#define LSB_T(pres, c, v, f, a, h)                 \
    if (pres) {                                     \
      const double pv = __dmul_rn(c, v);            \
      if (h) a = __dadd_rn(a, pv); else f = pv;     \
      h = true;                                     \
    }
    LSB_T(pzm, c0, zm.x, f0, a0, h0) LSB_T(pzm, c0, zm.y, f1, a1, h1)
    LSB_T(pym, c1, ym.x, f0, a0, h0) LSB_T(pym, c1, ym.y, f1, a1, h1)
    LSB_T(pxm, c2, xm, f0, a0, h0)   LSB_T(true, c2, cc.x, f1, a1, h1)
    LSB_T(true, c3, cc.x, f0, a0, h0) LSB_T(true, c3, cc.y, f1, a1, h1)
    LSB_T(true, c4, cc.y, f0, a0, h0) LSB_T(pxp, c4, xp, f1, a1, h1)
    LSB_T(pyp, c5, yp.x, f0, a0, h0) LSB_T(pyp, c5, yp.y, f1, a1, h1)
    LSB_T(pzp, c6, zp.x, f0, a0, h0) LSB_T(pzp, c6, zp.y, f1, a1, h1)
#undef LSB_T
    const double s0 = __dadd_rn(f0, a0), s1 = __dadd_rn(f1, a1);
    if (!isfinite(s0) || !isfinite(s1)) bad = true;
    double2 out;
    if (b) {
      const double2 bb = *reinterpret_cast<const double2*>(b + r);
      out = make_double2(__dsub_rn(bb.x, s0), __dsub_rn(bb.y, s1));
    } else {
      out = make_double2(s0, s1);
    }
    *reinterpret_cast<double2*>(y + r) = out;
  }
  if (bad && flags) flags->nonfinite = 1;
}

int launch_stencil(const lsb_stencil* S, const double* x, const double* b, double* y,
                   lsb_flags* flags, int it, cudaStream_t st) {
  if (S->noff < 1 || S->noff > LSB_MAX_OFF || S->nx < 1 || S->ny < 1 || S->nz < 1)
    return LSB_EINVAL;
  const int64_t n64 = (int64_t)S->nx * S->ny * S->nz;
  if (n64 >= (1LL << 31)) return LSB_ERANGE;
  StencilK K;
  K.nx = S->nx; K.ny = S->ny; K.nz = S->nz; K.noff = S->noff;
  K.halo_lo = S->halo_lo; K.halo_hi = S->halo_hi; K.d = S->col_scale;
  K.zlo = S->halo_lo ? -1 : 0;
  K.zhi = S->halo_hi ? S->nz : S->nz - 1;
  K.fx = FastDiv::make((uint32_t)S->nx);
  K.fy = FastDiv::make((uint32_t)S->ny);
  long long prev = -(1LL << 62);
  bool unit = true;
  K.rx = K.ry = K.rz = 0;
  for (int o = 0; o < S->noff; ++o) {
    K.dx[o] = S->dx[o]; K.dy[o] = S->dy[o]; K.dz[o] = S->dz[o]; K.val[o] = S->val[o];
    const long long lin = ((long long)S->dz[o] * S->ny + S->dy[o]) * S->nx + S->dx[o];
    if (lin <= prev) return LSB_EINVAL;  // must be CSR column order
    prev = lin;
    K.lin[o] = (int)lin;
    K.rx = max(K.rx, abs(S->dx[o])); K.ry = max(K.ry, abs(S->dy[o])); K.rz = max(K.rz, abs(S->dz[o]));
    if (S->dx[o] < -1 || S->dx[o] > 1 || S->dy[o] < -1 || S->dy[o] > 1 || S->dz[o] < -1 ||
        S->dz[o] > 1)
      unit = false;
  }
  for (int o = S->noff; o < LSB_MAX_OFF; ++o) {
    K.dx[o] = K.dy[o] = K.dz[o] = 0; K.val[o] = 0.0; K.lin[o] = 0;
  }
  const int64_t cap = (int64_t)sm_count() * 8;
  // canonical 7-point layout (the one laplace3d emits) gets the pair kernel
  const bool seven = S->noff == 7 && S->dz[0] == -1 && S->dy[1] == -1 && S->dx[2] == -1 &&
                     S->dx[3] == 0 && S->dy[3] == 0 && S->dz[3] == 0 && S->dx[4] == 1 &&
                     S->dy[5] == 1 && S->dz[6] == 1 && (S->nx % 2 == 0) && S->nx >= 4 && !S->col_scale &&
                     ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) &&
                     (!b || (uintptr_t)b % 16 == 0);
  if (seven) {
    static const int occ7 = wave(stencil7_pair_kernel, 0);
    int64_t g = (n64 / 2 + 255) / 256;
    if (g > (int64_t)sm_count() * occ7) g = (int64_t)sm_count() * occ7;
    if (g < 1) g = 1;
    stencil7_pair_kernel<<<(unsigned)g, 256, 0, st>>>(K, x, b, y, flags, it);
    return check_launch("stencil7");
  }
  int64_t g = (n64 + 255) / 256;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  if (canonical27(S) && S->nx % 2 == 0 && S->nx >= 4 && !S->col_scale &&
      (uintptr_t)x % 16 == 0 && (uintptr_t)y % 16 == 0 && (!b || (uintptr_t)b % 16 == 0)) {
    static const int occ27p = [] {
      int o = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, stencil27_pair_kernel, kS27Threads, 0);
      return o > 0 ? o : 1;
    }();
    int64_t gp = (n64 / 2 + kS27Threads - 1) / kS27Threads;
    if (gp > (int64_t)sm_count() * occ27p) gp = (int64_t)sm_count() * occ27p;
    if (gp < 1) gp = 1;
    const FastDiv fint = FastDiv::make(S->nx >= 6 ? (uint32_t)(S->nx / 2 - 2) : 1u);
    // auto: the TMA plane-tile kernel from 2^21 rows (128^3: 0.018 vs 0.023
    // ms for the row pairs), the row-pair kernel below (64^3: 0.0093 vs
    // 0.0133 tile, 0.0230 z-march); knob 4 forces the z-march, 2 row pairs
    const int mode = tuning(LSB_TUNE_S27_MARCH);
    if (mode == 0 && n64 >= (1LL << 21) && launch_stencil27_tile(K, x, b, y, flags, it, st))
      return check_launch("stencil27_tile");
    if (mode == 5 && launch_stencil27_tile(K, x, b, y, flags, it, st))
      return check_launch("stencil27_tile");
    if (S->nz >= 2 * kS27MarchZ && (mode == 3 || mode == 4)) {
      static const int occm = [] {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, stencil27_march_kernel, kS27Threads, 0);
        return o > 0 ? o : 1;
      }();
      const int nzc = (S->nz + kS27MarchZ - 1) / kS27MarchZ;
      const int64_t items = (int64_t)nzc * S->ny * (S->nx / 2);
      int64_t gm = (items + kS27Threads - 1) / kS27Threads;
      if (gm > (int64_t)sm_count() * occm) gm = (int64_t)sm_count() * occm;
      if (gm < 1) gm = 1;
      stencil27_march_kernel<<<(unsigned)gm, kS27Threads, 0, st>>>(
          K, fint, x, b, y, flags, it, nzc, tuning(LSB_TUNE_S27_MARCH) != 3);
      return check_launch("stencil27_march");
    }
    stencil27_pair_kernel<<<(unsigned)gp, kS27Threads, 0, st>>>(K, fint, x, b, y, flags, it);
    return check_launch("stencil27_pair");
  }
  if (canonical27(S)) {
    static const int occ27 = wave(stencil27_kernel, 0);
    if (g > (int64_t)sm_count() * occ27) g = (int64_t)sm_count() * occ27;
    stencil27_kernel<<<(unsigned)g, 256, 0, st>>>(K, x, b, y, flags, it);
    return check_launch("stencil27");
  }
  if (!unit) {
    stencil_kernel<0><<<(unsigned)g, 256, 0, st>>>(K, x, b, y, flags, it);
    return check_launch("stencil");
  }
  switch (S->noff) {
    case 5: stencil_kernel<5><<<(unsigned)g, 256, 0, st>>>(K, x, b, y, flags, it); break;
    case 7: stencil_kernel<7><<<(unsigned)g, 256, 0, st>>>(K, x, b, y, flags, it); break;
    case 27: stencil_kernel<27><<<(unsigned)g, 256, 0, st>>>(K, x, b, y, flags, it); break;
    default: stencil_kernel<0><<<(unsigned)g, 256, 0, st>>>(K, x, b, y, flags, it); break;
  }
  return check_launch("stencil");
}

// ------------------------------------------------------------------ CSR
struct CsrRowAcc {
  const int32_t* col;
  const double* val;
  const double* x;
  const double* d;
  int64_t x_lo;
  __device__ double operator()(int64_t j) const {
    const int64_t c = (int64_t)__ldg(col + j) - x_lo;
    double xv = __ldg(x + c);
    if (d) xv = __dmul_rn(xv, __ldg(d + c));
    return __dmul_rn(__ldg(val + j), xv);
  }
};

__global__ void __launch_bounds__(256)
csr_kernel(const lsb_csr A, const double* __restrict__ x, const double* __restrict__ b,
           double* __restrict__ y, lsb_flags* flags, int it) {
  if (gated_off(flags, it)) return;
  bool bad = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < A.n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = A.row_ptr[r], hi = A.row_ptr[r + 1];
    CsrRowAcc acc{A.col_idx + lo, A.values + lo, x, A.col_scale, A.x_lo};
    const double s = np_row_sum(acc, hi - lo);
    if (!isfinite(s)) bad = true;
    y[r] = b ? __dsub_rn(b[r], s) : s;
  }
  if (bad && flags) flags->nonfinite = 1;
}

// Dictionary-coded CSR (value-indexed + offset-indexed, "CSR-VI/DU"): when
// a matrix has at most 256 distinct values and at most 256 distinct column
// offsets col - row (constant-coefficient PDE discretisations), each entry
// is two u8 indices into per-matrix tables held in shared memory: 2 bytes
// per nonzero streamed instead of 12.  Thread per row: lane l of a warp owns
// row r0 + l, so entry k of 32 interior rows reads x at 32 consecutive
// addresses (one coalesced gather).  Products and numpy's reduceat order are
// csr_kernel's, so y is bitwise lsb_spmv_csr's.
struct CsrDictAcc {
  const uint8_t* vi;
  const uint8_t* oi;
  const double* vtab;
  const int32_t* otab;
  const double* x;
  const double* d;
  int64_t base;   // global row - x_lo
  __device__ double operator()(int64_t j) const {
    const int64_t c = base + otab[__ldg(oi + j)];
    double xv = __ldg(x + c);
    if (d) xv = __dmul_rn(xv, __ldg(d + c));
    return __dmul_rn(vtab[__ldg(vi + j)], xv);
  }
};

__global__ void __launch_bounds__(256)
csr_dict_kernel(const lsb_csr_dict A, const double* __restrict__ x, const double* __restrict__ b,
                double* __restrict__ y, lsb_flags* flags, int it) {
  if (gated_off(flags, it)) return;
  __shared__ double vtab[256];
  __shared__ int32_t otab[256];
  for (int k = threadIdx.x; k < A.n_val; k += blockDim.x) vtab[k] = A.val_tab[k];
  for (int k = threadIdx.x; k < A.n_off; k += blockDim.x) otab[k] = A.off_tab[k];
  __syncthreads();
  bool bad = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < A.n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = __ldg(A.row_ptr + r), hi = __ldg(A.row_ptr + r + 1);
    CsrDictAcc acc{A.val_idx + lo, A.off_idx + lo, vtab, otab, x, A.col_scale,
                   A.row0 + r - A.x_lo};
    const double s = np_row_sum(acc, hi - lo);
    if (!isfinite(s)) bad = true;
    y[r] = b ? __dsub_rn(b[r], s) : s;
  }
  if (bad && flags) flags->nonfinite = 1;
}

// Warp-staged variant (LSB_TUNE_CSR_DICT = 1, measured and kept off): a
// warp owns 32 consecutive rows, copies the u8 index bytes of their
// contiguous segment into shared memory with coalesced 32-bit loads, then
// each lane sums its own row from there, taking the index load out of the x
// gather's dependency chain.  0.78 ms vs 0.56 ms for the thread-per-row
// kernel at C5: the x gathers, not the index loads, bound it.  The index
// arrays are padded to whole words by the host (CsrOperator).
struct CsrDictSmemAcc {
  const uint8_t* vi;
  const uint8_t* oi;
  const double* vtab;
  const int32_t* otab;
  const double* x;
  const double* d;
  int64_t base;
  __device__ double operator()(int64_t j) const {
    const int64_t c = base + otab[oi[j]];
    double xv = __ldg(x + c);
    if (d) xv = __dmul_rn(xv, __ldg(d + c));
    return __dmul_rn(vtab[vi[j]], xv);
  }
};

constexpr int kDictWarps = 8;
constexpr int kDictSlabWords = 320;   // 1280 index bytes per stream per warp

__global__ void __launch_bounds__(kDictWarps * 32)
csr_dict_warp_kernel(const lsb_csr_dict A, const double* __restrict__ x,
                     const double* __restrict__ b, double* __restrict__ y, lsb_flags* flags,
                     int it) {
  if (gated_off(flags, it)) return;
  __shared__ double vtab[256];
  __shared__ int32_t otab[256];
  __shared__ uint32_t s_vi[kDictWarps][kDictSlabWords], s_oi[kDictWarps][kDictSlabWords];
  for (int k = threadIdx.x; k < A.n_val; k += blockDim.x) vtab[k] = A.val_tab[k];
  for (int k = threadIdx.x; k < A.n_off; k += blockDim.x) otab[k] = A.off_tab[k];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t* __restrict__ gvi = reinterpret_cast<const uint32_t*>(A.val_idx);
  const uint32_t* __restrict__ goi = reinterpret_cast<const uint32_t*>(A.off_idx);
  const uint8_t* svi = reinterpret_cast<const uint8_t*>(s_vi[wid]);
  const uint8_t* soi = reinterpret_cast<const uint8_t*>(s_oi[wid]);
  const int64_t n = A.n_rows, ngroups = (n + 31) >> 5;
  const int64_t wstride = (int64_t)gridDim.x * kDictWarps;
  bool bad = false;
  for (int64_t g = (int64_t)blockIdx.x * kDictWarps + wid; g < ngroups; g += wstride) {
    const int64_t r0 = g << 5, r = r0 + lane;
    const int64_t lo = __ldg(A.row_ptr + r0), hi = __ldg(A.row_ptr + min(r0 + 32, n));
    int64_t rs = 0, re = 0;
    if (r < n) { rs = __ldg(A.row_ptr + r); re = __ldg(A.row_ptr + r + 1); }
    const int64_t w0 = lo >> 2, nw = ((hi + 3) >> 2) - w0;
    double s;
    if (nw <= kDictSlabWords) {
#pragma unroll 4
      for (int j = lane; j < nw; j += 32) {
        s_vi[wid][j] = __ldg(gvi + w0 + j);
        s_oi[wid][j] = __ldg(goi + w0 + j);
      }
      __syncwarp();
      const int64_t o = rs - 4 * w0;
      s = np_row_sum(CsrDictSmemAcc{svi + o, soi + o, vtab, otab, x, A.col_scale,
                                    A.row0 + r - A.x_lo},
                     re - rs);
      __syncwarp();
    } else {
      s = np_row_sum(CsrDictAcc{A.val_idx + rs, A.off_idx + rs, vtab, otab, x, A.col_scale,
                                A.row0 + r - A.x_lo},
                     re - rs);
    }
    if (r < n) {
      if (!isfinite(s)) bad = true;
      y[r] = b ? __dsub_rn(b[r], s) : s;
    }
  }
  if (bad && flags) flags->nonfinite = 1;
}

int launch_csr_dict(const lsb_csr_dict* A, const double* x, const double* b, double* y,
                    lsb_flags* flags, int it, cudaStream_t st) {
  if (A->n_rows <= 0) return LSB_OK;
  if (A->n_val < 1 || A->n_val > 256 || A->n_off < 1 || A->n_off > 256) return LSB_EINVAL;
  if (tuning(LSB_TUNE_CSR_DICT) == 1) {
    static const int occw = wave(csr_dict_warp_kernel, 0);
    int64_t g = ((A->n_rows + 31) / 32 + kDictWarps - 1) / kDictWarps;
    if (g > (int64_t)sm_count() * occw) g = (int64_t)sm_count() * occw;
    csr_dict_warp_kernel<<<(unsigned)g, kDictWarps * 32, 0, st>>>(*A, x, b, y, flags, it);
    return check_launch("csr_dict_warp");
  }
  static const int occ = wave(csr_dict_kernel, 0);
  int64_t g = (A->n_rows + 255) / 256;
  if (g > (int64_t)sm_count() * occ) g = (int64_t)sm_count() * occ;
  csr_dict_kernel<<<(unsigned)g, 256, 0, st>>>(*A, x, b, y, flags, it);
  return check_launch("csr_dict");
}

// Warp-staged CSR: a warp owns 32 consecutive rows.  Their nonzeros form one
// contiguous segment [row_ptr[r0], row_ptr[r0+32]); the warp streams it with
// coalesced col/value loads (kCsrUnroll independent loads in flight per lane),
// forms each product val*x[col] exactly once, and parks it in a per-warp
// shared-memory slab.  Each lane then sums its own row from shared memory in
// numpy's reduceat order (np_row_sum), so y is bitwise the thread-per-row
// result.  A thread-per-row CSR warp touches 32 rows 12*nnz/n bytes apart per
// load instruction and depends on L1 to catch the rest of each sector;
// staging makes every col/value sector a single full-line request.
// Segments longer than the slab fall back to thread-per-row for that group.
constexpr int kCsrSlab = 1024;   // products per warp (8 KB)
constexpr int kCsrWarps = 8;

// col/value streams are read exactly once: keep them out of L1 so it holds x
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p) {
  int32_t r;
  asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double r;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

struct SmemAcc {
  const double* a;
  __device__ double operator()(int64_t j) const { return a[j]; }
};

template <int kCsrUnroll, int MINB = 1>
__global__ void __launch_bounds__(kCsrWarps * 32, MINB)
csr_warp_kernel(const lsb_csr A, const double* __restrict__ x, const double* __restrict__ b,
                double* __restrict__ y, lsb_flags* flags, int it) {
  if (gated_off(flags, it)) return;
  extern __shared__ double csr_slab[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* slab = csr_slab + wid * kCsrSlab;
  const int32_t* __restrict__ colv = A.col_idx;
  const double* __restrict__ valv = A.values;
  const double* __restrict__ d = A.col_scale;
  const int64_t n = A.n_rows, ngroups = (n + 31) >> 5;
  const int64_t wstride = (int64_t)gridDim.x * kCsrWarps;
  bool bad = false;
  for (int64_t g = (int64_t)blockIdx.x * kCsrWarps + wid; g < ngroups; g += wstride) {
    const int64_t r0 = g << 5, r = r0 + lane;
    const int64_t rlast = min(r0 + 32, n);
    const int64_t lo = __ldg(A.row_ptr + r0), hi = __ldg(A.row_ptr + rlast);
    int64_t rs = 0, re = 0;
    if (r < n) { rs = __ldg(A.row_ptr + r); re = __ldg(A.row_ptr + r + 1); }
    const int64_t seg = hi - lo;
    double s;
    if (seg <= kCsrSlab) {
      // three explicit phases per batch so every load of a phase is in flight
      // at once: col/value stream, then the x gathers, then products -> slab
      const int32_t* __restrict__ cg = colv + lo;
      const double* __restrict__ vg = valv + lo;
      const int segi = (int)seg;
      const int32_t c_pad = (int32_t)A.x_lo;
      for (int j0 = 0; j0 < segi; j0 += 32 * kCsrUnroll) {
        int32_t c[kCsrUnroll];
        double v[kCsrUnroll], xv[kCsrUnroll];
#pragma unroll
        for (int u = 0; u < kCsrUnroll; ++u) {
          const int j = j0 + u * 32 + lane;
          c[u] = j < segi ? ld_stream_i32(cg + j) : c_pad;
          v[u] = j < segi ? ld_stream_f64(vg + j) : 0.0;
        }
        if (d) {
          double dv[kCsrUnroll];
#pragma unroll
          for (int u = 0; u < kCsrUnroll; ++u) {
            const int64_t cc = (int64_t)c[u] - A.x_lo;
            xv[u] = __ldg(x + cc);
            dv[u] = __ldg(d + cc);
          }
#pragma unroll
          for (int u = 0; u < kCsrUnroll; ++u) xv[u] = __dmul_rn(xv[u], dv[u]);
        } else {
#pragma unroll
          for (int u = 0; u < kCsrUnroll; ++u) xv[u] = __ldg(x + ((int64_t)c[u] - A.x_lo));
        }
#pragma unroll
        for (int u = 0; u < kCsrUnroll; ++u) {
          const int j = j0 + u * 32 + lane;
          if (j < segi) slab[j] = __dmul_rn(v[u], xv[u]);
        }
      }
      __syncwarp();
      s = np_row_sum(SmemAcc{slab + (rs - lo)}, re - rs);
      __syncwarp();
    } else {
      s = np_row_sum(CsrRowAcc{colv + rs, valv + rs, x, d, A.x_lo}, re - rs);
    }
    if (r < n) {
      if (!isfinite(s)) bad = true;
      y[r] = b ? __dsub_rn(b[r], s) : s;
    }
  }
  if (bad && flags) flags->nonfinite = 1;
}

template <int U, int MINB = 1>
static int launch_csr_warp(const lsb_csr* A, const double* x, const double* b, double* y,
                           lsb_flags* flags, int it, cudaStream_t st) {
  constexpr size_t smem = sizeof(double) * kCsrSlab * kCsrWarps;
  static const int occ = [] {
    cudaFuncSetAttribute(csr_warp_kernel<U, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, csr_warp_kernel<U, MINB>, kCsrWarps * 32,
                                                  smem);
    return o > 0 ? o : 1;
  }();
  const int64_t groups = (A->n_rows + 31) / 32;
  int64_t g = (groups + kCsrWarps - 1) / kCsrWarps;
  if (g > (int64_t)sm_count() * occ) g = (int64_t)sm_count() * occ;
  csr_warp_kernel<U, MINB><<<(unsigned)g, kCsrWarps * 32, smem, st>>>(*A, x, b, y, flags, it);
  return check_launch("csr_warp");
}

int launch_csr(const lsb_csr* A, const double* x, const double* b, double* y, lsb_flags* flags,
               int it, cudaStream_t st) {
  if (A->n_rows <= 0) return LSB_OK;
  const int knob = tuning(LSB_TUNE_CSR_THREAD_ROW);
  if (knob != 1) {
    // 16 independent col/value loads per lane at 2 CTAs/SM (116 registers)
    // measured best on the 27-point CSR at 256^3: 5.02 TB/s vs 4.81 for 8
    // loads at 3 CTAs/SM (knob 2), 4.72 for 12 at 3 and 3.79 thread-per-row
    if (knob == 2) return launch_csr_warp<8, 3>(A, x, b, y, flags, it, st);
    return launch_csr_warp<16, 2>(A, x, b, y, flags, it, st);
  }
  int64_t g = (A->n_rows + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (g > cap) g = cap;
  csr_kernel<<<(unsigned)g, 256, 0, st>>>(*A, x, b, y, flags, it);
  return check_launch("csr");
}

// lsb_preload: one kernel of this translation unit (its module)
const void* tu_anchor_spmv() { return (const void*)csr_kernel; }

}  // namespace lsb
