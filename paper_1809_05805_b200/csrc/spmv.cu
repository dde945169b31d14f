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
// Interior rows (all neighbours present) take a register-only path; the
// 7-point operator additionally works on row pairs with 128-bit loads.
// Boundary rows fall back to a packed generic path.  K7 is a general CSR
// kernel with 32-bit indices.
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

int launch_csr(const lsb_csr* A, const double* x, const double* b, double* y, lsb_flags* flags,
               int it, cudaStream_t st) {
  if (A->n_rows <= 0) return LSB_OK;
  int64_t g = (A->n_rows + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (g > cap) g = cap;
  csr_kernel<<<(unsigned)g, 256, 0, st>>>(*A, x, b, y, flags, it);
  return check_launch("csr");
}

}  // namespace lsb
