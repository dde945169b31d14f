// K1+K6 fused: w = A u (7-point stencil, bitwise as the reference SpMV) and
// G = [Q^T u, Q^T w] in one pass over the basis.
//
// In the lagged loop the SpMV input u = V[:, p-1] is also the last column
// of Q, and its output w = V[:, p] is immediately reduced against Q
// (gmres.py:411-414 -> gram_schmidt.py:195-203).  Separately that costs the
// SpMV 16n bytes (read u, write w) plus K1 re-reading w: 8n(p+1) + 16n.
// Fused, each persistent CTA stages, with cp.async double-buffered one tile
// ahead, its u tile together with the stencil's halo -- nx rows either side
// and the two z-neighbour tiles (hot in L2: other CTAs of the same wave
// stream them) -- computes the tile's w rows entirely from shared memory,
// writes w once to HBM and keeps it in shared memory for the column sweep:
// 8n(p+1) bytes of compulsory HBM traffic, w never read back.
#include "tile.cuh"

namespace lsb {

struct Stencil7 {
  int nx, ny, zlo, zhi, plane;
  double c0, c1, c2, c3, c4, c5, c6;
  FastDiv fx, fy;
  int64_t lo_valid, hi_valid;  // u rows that exist in memory (ghost planes included)
  // ghost rows arriving by push (lsb_halo_wait): tiles are visited in the
  // order t -> (t + shift) mod ntiles, so the tiles reading ghost rows come
  // last; the staging of any tile >= wait_from waits for the signals first
  int64_t shift, wait_from;
  const int64_t* sig_lo;
  const int64_t* sig_hi;
  const int64_t* epoch;
  int64_t timeout_ns;
  lsb_flags* wflags;
  __device__ __forceinline__ int64_t row0(int64_t t, int64_t ntiles) const {
    int64_t v = t + shift;
    if (v >= ntiles) v -= ntiles;
    return v * kTile;
  }
  // leader thread, before staging tile t (t in visiting order)
  __device__ __forceinline__ void wait_ghosts(int64_t t, bool& waited) const {
    if (waited || t < wait_from || !(sig_lo || sig_hi)) return;
    waited = true;
    const int64_t e = *epoch;
    bool ok = true;
    if (sig_lo) ok = spin_signal(sig_lo, e, timeout_ns) && ok;
    if (sig_hi) ok = spin_signal(sig_hi, e, timeout_ns) && ok;
    if (!ok && wflags) wflags->comm_error = LSB_COMM_TIMEOUT;
    // the remote stores are read by the bulk-copy (async) proxy next
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
};

// One row pair (lr, lr+1) of w = A u from the staged tile (numpy order:
// first present product + sequential sum of the rest), written to the
// shared w tile and to HBM.
template <bool NORM = false>
__device__ __forceinline__ void s7_tile_pair(const Stencil7& K, const double* ut, const double* zt,
                                             const double* pt, int lr, int64_t r, int64_t n,
                                             double* sw, double* __restrict__ wout, bool& bad,
                                             double (&nrm)[2]) {
  if (r >= n) { sw[lr] = sw[lr + 1] = 0.0; return; }
  const uint32_t line = K.fx.div((uint32_t)r);
  const int ix = (int)((uint32_t)r - line * (uint32_t)K.nx);
  const uint32_t iz = K.fy.div(line);
  const int iy = (int)(line - iz * (uint32_t)K.ny);
  const bool pzm = (int)iz - 1 >= K.zlo, pzp = (int)iz + 1 <= K.zhi;
  const bool pym = iy >= 1, pyp = iy + 1 < K.ny;
  const bool pxm = ix >= 1, pxp = ix + 2 < K.nx;
  const double2 zm = *reinterpret_cast<const double2*>(zt + lr);
  const double2 zp = *reinterpret_cast<const double2*>(pt + lr);
  const double2 ym = *reinterpret_cast<const double2*>(ut + lr - K.nx);
  const double2 yp = *reinterpret_cast<const double2*>(ut + lr + K.nx);
  const double2 cc = *reinterpret_cast<const double2*>(ut + lr);
  const double xm = ut[lr - 1], xp = ut[lr + 2];
  double f0 = 0.0, a0 = -0.0, f1 = 0.0, a1 = -0.0;
  bool h0 = false, h1 = false;
#define LSB_T(pres, c, v, f, a, h)                 \
  if (pres) {                                       \
    const double pv = __dmul_rn(c, v);              \
    if (h) a = __dadd_rn(a, pv); else f = pv;       \
    h = true;                                       \
  }
  LSB_T(pzm, K.c0, zm.x, f0, a0, h0) LSB_T(pzm, K.c0, zm.y, f1, a1, h1)
  LSB_T(pym, K.c1, ym.x, f0, a0, h0) LSB_T(pym, K.c1, ym.y, f1, a1, h1)
  LSB_T(pxm, K.c2, xm, f0, a0, h0)   LSB_T(true, K.c2, cc.x, f1, a1, h1)
  LSB_T(true, K.c3, cc.x, f0, a0, h0) LSB_T(true, K.c3, cc.y, f1, a1, h1)
  LSB_T(true, K.c4, cc.y, f0, a0, h0) LSB_T(pxp, K.c4, xp, f1, a1, h1)
  LSB_T(pyp, K.c5, yp.x, f0, a0, h0) LSB_T(pyp, K.c5, yp.y, f1, a1, h1)
  LSB_T(pzp, K.c6, zp.x, f0, a0, h0) LSB_T(pzp, K.c6, zp.y, f1, a1, h1)
#undef LSB_T
  const double s0 = __dadd_rn(f0, a0), s1 = __dadd_rn(f1, a1);
  if (!isfinite(s0) || !isfinite(s1)) bad = true;
  if constexpr (NORM) {   // norm_partial's per-row update (a NaN row poisons max and ssq)
    nrm[0] = fmax(nrm[0], fabs(s0));
    if (isnan(s0)) nrm[0] = s0;
    nrm[1] = fma(s0, s0, nrm[1]);
    nrm[0] = fmax(nrm[0], fabs(s1));
    if (isnan(s1)) nrm[0] = s1;
    nrm[1] = fma(s1, s1, nrm[1]);
  }
  sw[lr] = s0;
  sw[lr + 1] = s1;
  *reinterpret_cast<double2*>(wout + r) = make_double2(s0, s1);
}

// NORM: also (max|w|, sum w^2) as entries 2p, 2p+1 (fused_mdot_norm)
template <int R, int SLOTS, int MINB, bool NORM = false>
__global__ void __launch_bounds__(kThreads, MINB)
mdot_spmv7_kernel(const double* __restrict__ X, int64_t ld, int64_t n, int p,
                  double* __restrict__ wout, const Stencil7 K, double* __restrict__ out,
                  double* __restrict__ partial, unsigned* counter, lsb_flags* flags, int it) {
  pdl_enter();
  if (gated_off(flags, it)) return;
  constexpr int kRows = kTile / R;
  constexpr int kLd = kRows / 64;
  extern __shared__ __align__(16) double smem[];
  const int H = K.nx;                          // row halo each side
  const int span = kTile + 2 * H;              // u tile with halo
  const int stage = span + 2 * kTile;          // + z-1 and z+1 tiles
  double* sw = smem + 2 * stage;               // w tile
  __shared__ double red[kWarps * SLOTS][2];
  const double* __restrict__ u = X + (int64_t)(p - 1) * ld;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int part = warp % R;
  double acc[SLOTS][2];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) acc[s][0] = acc[s][1] = 0.0;
  bool bad = false;
  double nrm[2] = {0.0, 0.0};

  // u tile + halo + z-neighbour tiles arrive by three TMA bulk copies issued
  // by one thread, completion on a per-buffer mbarrier (double-buffered)
  __shared__ __align__(8) uint64_t bars[2];
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t ntiles = (n + kTile - 1) / kTile;
  bool waited = false;
  auto stage_all = [&](int b, int64_t t) {
    double* base = smem + b * stage;
    const int64_t r0 = K.row0(t, ntiles);
    unsigned tx = 0;
    const bool leader = threadIdx.x == 0;
    if (leader) K.wait_ghosts(t, waited);
    stage_bulk(base, u, r0 - H, span, K.lo_valid, K.hi_valid, &bars[b], leader, &tx);
    stage_bulk(base + span, u, r0 - K.plane, kTile, K.lo_valid, K.hi_valid, &bars[b], leader, &tx);
    stage_bulk(base + span + kTile, u, r0 + K.plane, kTile, K.lo_valid, K.hi_valid, &bars[b],
               leader, &tx);
    if (leader) mbar_arrive_tx(&bars[b], tx);
  };

  int64_t t = blockIdx.x;
  int buf = 0;
  unsigned phase = 0;
  if (t < ntiles) stage_all(0, t);
  for (; t < ntiles; t += gridDim.x) {
    // two barriers per tile: (A) tile t landed and every warp done with
    // tile t-1 (so buf^1 and sw are free), (B) w of tile t complete
    mbar_wait(&bars[buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;
    __syncthreads();
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) stage_all(buf ^ 1, tn);
    const int64_t r0 = K.row0(t, ntiles);
    const double* ut = smem + buf * stage + H;   // ut[lr] = u[r0 + lr], lr in [-H, kTile+H)
    const double* zt = smem + buf * stage + span;
    const double* pt = zt + kTile;
    const bool full = r0 + kTile <= n;
    const int rbase = part * kRows;
    // the first item's basis loads do not depend on w: issue them now so
    // they are in flight while the stencil phase below runs (only when few
    // items per warp leave registers to spare: it spills at 8+ items)
    constexpr bool kPrefetch = SLOTS <= 4 && kLd <= 8 && MINB == 2;
    double2 pre[kLd];
    if (kPrefetch) {
      const int k0 = warp / R;
      if (full && k0 < p) {
        const double* col = X + (int64_t)k0 * ld + r0 + rbase;
#pragma unroll
        for (int q = 0; q < kLd; ++q) pre[q] = ld_stream(col + 2 * (lane + 32 * q));
      }
    }
    // ---- w = A u for the tile rows (row pairs; nx even keeps pairs in a line)
#pragma unroll 2
    for (int j = threadIdx.x; j < kTile / 2; j += kThreads)
      s7_tile_pair<NORM>(K, ut, zt, pt, 2 * j, r0 + 2 * j, n, sw, wout, bad, nrm);
    __syncthreads();
    // ---- column sweep: [Q^T u, Q^T w] partials (same item deal as mdot_kernel)
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int k = (warp + kWarps * s) / R;
      if (k < p) {
        const double* col = X + (int64_t)k * ld + r0 + rbase;
        double a0 = 0.0, a1 = 0.0;
        if (full) {
          double2 xv[kLd];
#pragma unroll
          for (int q = 0; q < kLd; ++q)
            xv[q] = (kPrefetch && s == 0) ? pre[q] : ld_stream(col + 2 * (lane + 32 * q));
#pragma unroll
          for (int q = 0; q < kLd; ++q) {
            const int lr = rbase + 2 * (lane + 32 * q);
            const double2 yu = *reinterpret_cast<const double2*>(ut + lr);
            const double2 yw = *reinterpret_cast<const double2*>(sw + lr);
            a0 = fma(xv[q].x, yu.x, a0);
            a0 = fma(xv[q].y, yu.y, a0);
            a1 = fma(xv[q].x, yw.x, a1);
            a1 = fma(xv[q].y, yw.y, a1);
          }
        } else {
          for (int q = 0; q < kLd; ++q) {
            const int lr = rbase + 2 * (lane + 32 * q);
            const int64_t r = r0 + lr;
            const double xa = r < n ? col[lr - rbase] : 0.0;
            const double xb = r + 1 < n ? col[lr - rbase + 1] : 0.0;
            const double ua = r < n ? ut[lr] : 0.0, ub = r + 1 < n ? ut[lr + 1] : 0.0;
            a0 = fma(xa, ua, a0);
            a0 = fma(xb, ub, a0);
            a1 = fma(xa, sw[lr], a1);
            a1 = fma(xb, sw[lr + 1], a1);
          }
        }
        acc[s][0] += a0;
        acc[s][1] += a1;
      }
    }
    buf ^= 1;
  }
  if (bad && flags) flags->nonfinite = 1;

#pragma unroll
  for (int s = 0; s < SLOTS; ++s)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const double x = warp_sum(acc[s][v]);
      if (lane == 0) red[warp + kWarps * s][v] = x;
    }
  __shared__ double nred[kWarps][2];
  if (NORM) {
    const double m = warp_max(nrm[0]), q = warp_sum(nrm[1]);
    if (lane == 0) { nred[warp][0] = m; nred[warp][1] = q; }
  }
  __syncthreads();
  const int G = gridDim.x;
  for (int e = threadIdx.x; e < p * 2; e += kThreads) {
    const int k = e / 2, v = e % 2;
    double x = red[k * R][v];
#pragma unroll
    for (int pr = 1; pr < R; ++pr) x += red[k * R + pr][v];
    partial[(size_t)e * G + blockIdx.x] = x;
  }
  if (NORM && threadIdx.x < 2) {
    const int v = threadIdx.x;
    double x = nred[0][v];
    for (int w = 1; w < kWarps; ++w) x = v == 0 ? fmax(x, nred[w][v]) : x + nred[w][v];
    partial[(size_t)(2 * p + v) * G + blockIdx.x] = x;
  }
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == (unsigned)G - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int E = 2 * p + (NORM ? 2 : 0);
  for (int e = warp; e < E; e += kWarps) {
    const bool mx = NORM && e == 2 * p;
    double x = 0.0;
    for (int c = lane; c < G; c += 32) {
      const double y = __ldcg(partial + (size_t)e * G + c);
      x = mx ? fmax(x, y) : x + y;
    }
    x = mx ? warp_max(x) : warp_sum(x);
    if (lane == 0) out[e] = x;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// Pipelined variant: one barrier per tile, and the stencil work of tile
// t+1 is done inside tile t's column sweep, between issuing an item's basis
// loads and consuming them, so it hides under the load latency instead of
// stalling all warps between two barriers.  Two w buffers: the sweep of t
// reads sw[t], the stencil of t+1 writes sw[t+1].  Tile t+1's u data is
// staged (TMA, issued at the top of tile t) into the other stage buffer.
// Same arithmetic and the same item deal / summation order as
// mdot_spmv7_kernel, so w and the partials are bitwise equal.
template <int R, int SLOTS, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
mdot_spmv7_pipe_kernel(const double* __restrict__ X, int64_t ld, int64_t n, int p,
                       double* __restrict__ wout, const Stencil7 K, double* __restrict__ out,
                       double* __restrict__ partial, unsigned* counter, lsb_flags* flags, int it) {
  pdl_enter();
  if (gated_off(flags, it)) return;
  constexpr int kRows = kTile / R;
  constexpr int kLd = kRows / 64;
  extern __shared__ __align__(16) double smem[];
  const int H = K.nx;
  const int span = kTile + 2 * H;
  const int stage = span + 2 * kTile;
  double* swb = smem + 2 * stage;              // two w tiles
  __shared__ double red[kWarps * SLOTS][2];
  const double* __restrict__ u = X + (int64_t)(p - 1) * ld;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int part = warp % R;
  double acc[SLOTS][2];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) acc[s][0] = acc[s][1] = 0.0;
  bool bad = false;
  double nrm[2];   // unused (no norm in the pipelined variant)
  __shared__ __align__(8) uint64_t bars[2];
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t ntiles = (n + kTile - 1) / kTile;
  bool waited = false;
  auto stage_all = [&](int b, int64_t t) {
    double* base = smem + b * stage;
    const int64_t r0 = K.row0(t, ntiles);
    unsigned tx = 0;
    const bool leader = threadIdx.x == 0;
    if (leader) K.wait_ghosts(t, waited);
    stage_bulk(base, u, r0 - H, span, K.lo_valid, K.hi_valid, &bars[b], leader, &tx);
    stage_bulk(base + span, u, r0 - K.plane, kTile, K.lo_valid, K.hi_valid, &bars[b], leader, &tx);
    stage_bulk(base + span + kTile, u, r0 + K.plane, kTile, K.lo_valid, K.hi_valid, &bars[b],
               leader, &tx);
    if (leader) mbar_arrive_tx(&bars[b], tx);
  };
  int64_t t = blockIdx.x;
  int buf = 0;
  unsigned phase = 0;
  if (t < ntiles) {            // prologue: w of the first tile, whole
    stage_all(0, t);
    mbar_wait(&bars[0], 0u);
    phase ^= 1u;
    const double* ut = smem + H;
    const double* zt = smem + span;
    const int64_t rp0 = K.row0(t, ntiles);
    for (int j = threadIdx.x; j < kTile / 2; j += kThreads)
      s7_tile_pair(K, ut, zt, zt + kTile, 2 * j, rp0 + 2 * j, n, swb, wout, bad, nrm);
  }
  for (; t < ntiles; t += gridDim.x) {
    __syncthreads();           // w of tile t complete; tile t-1 fully consumed
    const int64_t tn = t + gridDim.x;
    const bool nxt = tn < ntiles;
    if (nxt) stage_all(buf ^ 1, tn);
    const int64_t r0 = K.row0(t, ntiles);
    const double* ut = smem + buf * stage + H;
    const double* sw = swb + buf * kTile;
    const double* utn = smem + (buf ^ 1) * stage + H;
    const double* ztn = smem + (buf ^ 1) * stage + span;
    double* swn = swb + (buf ^ 1) * kTile;
    const int64_t rn0 = nxt ? K.row0(tn, ntiles) : 0;
    const bool full = r0 + kTile <= n;
    const int rbase = part * kRows;
    bool ready = false;
    auto chunk = [&](int c) {  // stencil pairs of tile tn owned by chunk c
      if (!nxt) return;
      if (!ready) {
        mbar_wait(&bars[buf ^ 1], (phase >> (buf ^ 1)) & 1u);
        phase ^= 1u << (buf ^ 1);
        ready = true;
      }
      const int j0 = SLOTS == 1 ? 0 : c, j1 = SLOTS == 1 ? 2 : c + 1;
      for (int jj = j0; jj < j1; ++jj) {
        const int j = threadIdx.x + jj * kThreads;
        s7_tile_pair(K, utn, ztn, ztn + kTile, 2 * j, rn0 + 2 * j, n, swn, wout, bad, nrm);
      }
    };
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int k = (warp + kWarps * s) / R;
      const bool live = k < p;
      const double* col = X + (int64_t)k * ld + r0 + rbase;
      double2 xv[kLd];
      if (live && full) {
#pragma unroll
        for (int q = 0; q < kLd; ++q) xv[q] = ld_stream(col + 2 * (lane + 32 * q));
      }
      if (s < 2) chunk(s);     // overlaps the loads just issued
      if (live) {
        double a0 = 0.0, a1 = 0.0;
        if (full) {
#pragma unroll
          for (int q = 0; q < kLd; ++q) {
            const int lr = rbase + 2 * (lane + 32 * q);
            const double2 yu = *reinterpret_cast<const double2*>(ut + lr);
            const double2 yw = *reinterpret_cast<const double2*>(sw + lr);
            a0 = fma(xv[q].x, yu.x, a0);
            a0 = fma(xv[q].y, yu.y, a0);
            a1 = fma(xv[q].x, yw.x, a1);
            a1 = fma(xv[q].y, yw.y, a1);
          }
        } else {
          for (int q = 0; q < kLd; ++q) {
            const int lr = rbase + 2 * (lane + 32 * q);
            const int64_t r = r0 + lr;
            const double xa = r < n ? col[lr - rbase] : 0.0;
            const double xb = r + 1 < n ? col[lr - rbase + 1] : 0.0;
            const double ua = r < n ? ut[lr] : 0.0, ub = r + 1 < n ? ut[lr + 1] : 0.0;
            a0 = fma(xa, ua, a0);
            a0 = fma(xb, ub, a0);
            a1 = fma(xa, sw[lr], a1);
            a1 = fma(xb, sw[lr + 1], a1);
          }
        }
        acc[s][0] += a0;
        acc[s][1] += a1;
      }
    }
    buf ^= 1;
  }
  if (bad && flags) flags->nonfinite = 1;

#pragma unroll
  for (int s = 0; s < SLOTS; ++s)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const double x = warp_sum(acc[s][v]);
      if (lane == 0) red[warp + kWarps * s][v] = x;
    }
  __syncthreads();
  const int G = gridDim.x;
  for (int e = threadIdx.x; e < p * 2; e += kThreads) {
    const int k = e / 2, v = e % 2;
    double x = red[k * R][v];
#pragma unroll
    for (int pr = 1; pr < R; ++pr) x += red[k * R + pr][v];
    partial[(size_t)e * G + blockIdx.x] = x;
  }
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == (unsigned)G - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int e = warp; e < 2 * p; e += kWarps) {
    double x = 0.0;
    for (int c = lane; c < G; c += 32) x += __ldcg(partial + (size_t)e * G + c);
    x = warp_sum(x);
    if (lane == 0) out[e] = x;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// 3 CTAs/SM (<= 8 items per warp, register-capped) loses to the 2-CTA
// variant with whole-tile items at every p >= 8 (tools/kfused.py: p = 26
// 644 vs 568 us) and ties below; kept as an opt-in (knob value 1).
static bool occ3(int p) {
  (void)p;
  return tuning(LSB_TUNE_FUSED_OCC3) == 1;
}

static size_t smem_bytes(int nx, bool pipe) {
  return sizeof(double) * (2 * (kTile + 2 * nx + 2 * kTile) + (pipe ? 2 : 1) * kTile);
}

// the pipelined kernel for 2..4 items per warp, 2 CTAs/SM (tools/kpipe.py,
// 256^3: 3-4% faster there; with one item the stencil chunks have no loads
// to hide under, and at 8 items the extra live registers spill)
static bool use_pipe(int slots) {
  const int knob = tuning(LSB_TUNE_FUSED_PIPE);
  if (knob == 2 || occ3(0)) return false;
  return knob == 1 ? slots <= 8 : (slots >= 2 && slots <= 4);
}

template <class Kern>
static int launch_k(Kern kern, bool pipe, int* occ_nx, int* occ, const lsb_arnoldi& S,
                    const Stencil7& K, int p, int it, cudaStream_t st) {
  const size_t sm = smem_bytes(K.nx, pipe);
  if (*occ_nx != K.nx) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, kThreads, sm);
    if (*occ < 1) *occ = 1;
    *occ_nx = K.nx;
  }
  const int64_t ntiles = (S.n + kTile - 1) / kTile;
  int64_t grid = (int64_t)sm_count() * *occ;
  if (S.ws.grid > 0 && S.ws.grid < grid) grid = S.ws.grid;
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  const cudaError_t le = launch_chain(use_pdl(S.n), kern, dim3((unsigned)grid), dim3(kThreads), sm, st, S.V, S.ld, S.n, p,
               S.V + (int64_t)p * S.ld, K, S.Gloc, S.ws.partial, S.ws.counter, S.flags, it);
  return check_launch("mdot_spmv7", le);
}

template <int R, int SLOTS, int MINB>
static int launch_t(const lsb_arnoldi& S, const Stencil7& K, int p, int it, cudaStream_t st,
                    bool norm) {
  if (norm) {
    static int nx = -1, occ = 0;
    return launch_k(mdot_spmv7_kernel<R, SLOTS, 2, true>, false, &nx, &occ, S, K, p, it, st);
  }
  if constexpr (MINB == 2 && SLOTS <= 8) {
    if (use_pipe(SLOTS)) {
      static int nx = -1, occ = 0;
      return launch_k(mdot_spmv7_pipe_kernel<R, SLOTS, MINB>, true, &nx, &occ, S, K, p, it, st);
    }
  }
  static int nx = -1, occ = 0;
  return launch_k(mdot_spmv7_kernel<R, SLOTS, MINB>, false, &nx, &occ, S, K, p, it, st);
}

template <int R>
static int launch_r(const lsb_arnoldi& S, const Stencil7& K, int p, int it, cudaStream_t st,
                    bool norm) {
  const int s = slots_for(p, R);
  if (occ3(p) && !norm) {   // 3 CTAs/SM, at most 8 items per warp
    if (s <= 1) return launch_t<R, 1, 3>(S, K, p, it, st, norm);
    if (s <= 2) return launch_t<R, 2, 3>(S, K, p, it, st, norm);
    if (s <= 4) return launch_t<R, 4, 3>(S, K, p, it, st, norm);
    return launch_t<R, 8, 3>(S, K, p, it, st, norm);
  }
  if (s <= 1) return launch_t<R, 1, 2>(S, K, p, it, st, norm);
  if (s <= 2) return launch_t<R, 2, 2>(S, K, p, it, st, norm);
  if (s <= 4) return launch_t<R, 4, 2>(S, K, p, it, st, norm);
  if (s <= 8) return launch_t<R, 8, 2>(S, K, p, it, st, norm);
  if (s <= 13) return launch_t<R, 13, 2>(S, K, p, it, st, norm);
  return launch_t<R, 16, 2>(S, K, p, it, st, norm);
}

int launch_lagged_reduce_spmv7(const lsb_arnoldi& S, const lsb_stencil* A, int it, int p,
                               cudaStream_t st, const lsb_halo_wait* hw, bool norm) {
  if (!canonical7(A) || A->nx > kTile) return LSB_EINVAL;
  if ((int64_t)A->nx * A->ny * A->nz != S.n || (S.n & 1) || p < 1 || p > 128 || p + 1 > S.cap)
    return LSB_ERANGE;
  Stencil7 K;
  K.nx = A->nx; K.ny = A->ny; K.plane = A->nx * A->ny;
  K.zlo = A->halo_lo ? -1 : 0;
  K.zhi = A->halo_hi ? A->nz : A->nz - 1;
  K.c0 = A->val[0]; K.c1 = A->val[1]; K.c2 = A->val[2]; K.c3 = A->val[3];
  K.c4 = A->val[4]; K.c5 = A->val[5]; K.c6 = A->val[6];
  K.fx = FastDiv::make((uint32_t)A->nx);
  K.fy = FastDiv::make((uint32_t)A->ny);
  K.lo_valid = A->halo_lo ? -(int64_t)K.plane : 0;
  K.hi_valid = S.n + (A->halo_hi ? K.plane : 0);
  K.shift = 0;
  K.wait_from = INT64_MAX;
  K.sig_lo = K.sig_hi = K.epoch = nullptr;
  K.timeout_ns = 0;
  K.wflags = nullptr;
  if (hw && ((A->halo_lo && hw->sig_lo) || (A->halo_hi && hw->sig_hi))) {
    // tiles that stage ghost rows: the z-1 tile or the row halo below row 0
    // (r0 < plane + nx), the z+1 tile or the row halo past n - 1
    const int64_t ntiles = (S.n + kTile - 1) / kTile;
    const int64_t reach = (int64_t)K.plane + K.nx;
    const int64_t nb_lo = A->halo_lo ? (reach + kTile - 1) / kTile : 0;
    int64_t first_hi = ntiles;
    if (A->halo_hi) {
      first_hi = (S.n - reach - kTile) / kTile;   // conservative: one tile early
      if (S.n - reach - kTile < 0) first_hi = 0;
    }
    const int64_t nb_hi = ntiles - first_hi;
    if (nb_lo + nb_hi >= ntiles) {
      K.shift = 0;
      K.wait_from = 0;           // every tile touches a ghost row: wait up front
    } else {
      K.shift = nb_lo;           // visiting order: interior, upper boundary, lower boundary
      K.wait_from = ntiles - nb_lo - nb_hi;
    }
    K.sig_lo = A->halo_lo ? hw->sig_lo : nullptr;
    K.sig_hi = A->halo_hi ? hw->sig_hi : nullptr;
    K.epoch = hw->epoch;
    K.timeout_ns = hw->timeout_ns;
    K.wflags = hw->flags;
  }
  switch (occ3(p) && !norm ? choose_parts(p, 8) : choose_parts(p)) {
    case 8: return launch_r<8>(S, K, p, it, st, norm);
    case 4: return launch_r<4>(S, K, p, it, st, norm);
    case 2: return launch_r<2>(S, K, p, it, st, norm);
    default: return launch_r<1>(S, K, p, it, st, norm);
  }
}

// lsb_preload: one kernel of this translation unit (its module)
const void* tu_anchor_fused() { return (const void*)mdot_spmv7_kernel<1, 1, 2>; }

}  // namespace lsb
