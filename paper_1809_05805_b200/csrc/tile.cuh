// Streaming / staging helpers shared by the reduction kernels.
#pragma once
#include "reduce.cuh"

namespace lsb {

constexpr int kTile = 1024;  // rows per K1 tile

// runtime tuning knobs (lsb_set_tuning); defaults are the measured best
int tuning(int key);

// Resident CTAs per SM of kernel k (256 threads): persistent grid-stride
// kernels launch exactly one full wave, SMs x this.  A partial second wave
// costs up to 25% on the streaming kernels (tools/krow.py: K2 6.75 TB/s at
// one wave vs 6.45 at a fixed 8 CTAs/SM and 5.47 at 6).
template <class Kern>
inline int wave(Kern k, size_t smem) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, smem);
  return occ > 0 ? occ : 1;
}

// 128-bit streaming load that does not allocate in L1 (basis columns are
// read exactly once per pass).
__device__ __forceinline__ double2 ld_stream(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Stage rows [t*kTile, (t+1)*kTile) of y0 (and y1) into buf: cp.async for a
// full tile, zero-padded synchronous loads for the ragged last tile.
template <int NV>
__device__ __forceinline__ void stage_tile(double2 (*buf)[kTile / 2], const double* y0,
                                           const double* y1, int64_t n, int64_t t) {
  const int64_t r0 = t * kTile;
  if (r0 + kTile <= n) {
    for (int j = threadIdx.x; j < kTile / 2; j += kThreads)
#pragma unroll
      for (int v = 0; v < NV; ++v) cp_async16(&buf[v][j], (v == 0 ? y0 : y1) + r0 + 2 * j);
  } else {
    for (int j = threadIdx.x; j < kTile / 2; j += kThreads) {
      const int64_t r = r0 + 2 * j;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double* y = v == 0 ? y0 : y1;
        buf[v][j] = make_double2(r < n ? y[r] : 0.0, r + 1 < n ? y[r + 1] : 0.0);
      }
    }
  }
}

// ---------------------------------------------------------------- TMA bulk copies
// 1-D cp.async.bulk (UBLKCP) global -> shared, completion counted in bytes on
// an mbarrier: one elected thread moves a whole tile, no per-thread copies.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Stage rows [a, a+len) of src into dst: the part inside [lo, hi) by one
// bulk copy (issued by the calling elected thread, bytes added to *tx), the
// rest zero-filled by all threads of the CTA (call with every thread; only
// `leader` issues the copy).  a, len, lo, hi even (16-byte granules).
__device__ __forceinline__ void stage_bulk(double* dst, const double* src, int64_t a, int len,
                                          int64_t lo, int64_t hi, uint64_t* bar, bool leader,
                                          unsigned* tx) {
  const int64_t v0 = a > lo ? a : lo;
  const int64_t v1 = (a + len) < hi ? (a + len) : hi;
  if (v1 > v0) {
    if (leader) {
      bulk_g2s(dst + (v0 - a), src + v0, (unsigned)(8 * (v1 - v0)), bar);
      *tx += (unsigned)(8 * (v1 - v0));
    }
  }
  const int z0 = v1 > v0 ? (int)(v0 - a) : len;   // zero-fill [0, z0) and [z1, len)
  const int z1 = v1 > v0 ? (int)(v1 - a) : len;
  if (z0 > 0 || z1 < len) {
    for (int j = threadIdx.x; j < z0; j += blockDim.x) dst[j] = 0.0;
    for (int j = z1 + threadIdx.x; j < len; j += blockDim.x) dst[j] = 0.0;
    fence_proxy_async();
  }
}

// Unsigned 32-bit division by an invariant d (valid for n < 2^31).
struct FastDiv {
  uint32_t d, m, s;
  static FastDiv make(uint32_t d) {
    FastDiv f;
    f.d = d;
    f.s = 0;
    while ((1u << f.s) < d) ++f.s;
    const uint64_t one = 1;
    f.m = (uint32_t)(((one << 32) * ((one << f.s) - d)) / d + 1);
    return f;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    const uint32_t t = __umulhi(n, m);
    return (t + n) >> s;
  }
};

// The 7-point operator in the canonical column order laplace3d emits
// (-plane, -nx, -1, 0, +1, +nx, +plane), nx even, no column scaling: the
// layout the row-pair SpMV kernels (and the fused K1+SpMV) handle.
inline bool canonical7(const lsb_stencil* S) {
  return S->noff == 7 && S->dz[0] == -1 && S->dx[0] == 0 && S->dy[0] == 0 && S->dy[1] == -1 &&
         S->dx[1] == 0 && S->dz[1] == 0 && S->dx[2] == -1 && S->dy[2] == 0 && S->dz[2] == 0 &&
         S->dx[3] == 0 && S->dy[3] == 0 && S->dz[3] == 0 && S->dx[4] == 1 && S->dy[4] == 0 &&
         S->dz[4] == 0 && S->dy[5] == 1 && S->dx[5] == 0 && S->dz[5] == 0 && S->dz[6] == 1 &&
         S->dx[6] == 0 && S->dy[6] == 0 && (S->nx % 2 == 0) && S->nx >= 4 && !S->col_scale;
}

// Choose R in {1,2,4,8} row parts per tile column so the p*R (column,
// part) items deal evenly over 8 warps with at most 16 items per warp.
inline int slots_for(int p, int R) { return (p * R + kWarps - 1) / kWarps; }
inline int choose_parts(int p, int max_slots = 16) {
  const int forced = tuning(LSB_TUNE_FORCE_PARTS);   // experiments: 1, 2, 4 or 8
  if (forced == 1 || forced == 2 || forced == 4 || forced == 8)
    if (slots_for(p, forced) <= max_slots) return forced;
  // Measured (tools/kparts.py, tools/kfused.py at 256^3): whole-tile items
  // (R = 1, 16 independent 128-bit loads per lane) beat a perfectly even
  // deal of shorter items at every p >= 6 -- K1 reaches 7.0-7.1 TB/s with
  // R = 1 vs 5.9 with R = 4 at p = 26.  Below that, halves keep more warps busy.
  int R = p >= 6 ? 1 : 2;
  while (slots_for(p, R) > max_slots && R < 8) R *= 2;
  return R;
}

}  // namespace lsb
