// K3: the two-sync CGS2 first projection and second reduction in ONE pass
// over the basis (gram_schmidt.py:273-277):
//
//     u /= beta;  w /= beta;  w -= Q r;          (lagged_update, K2)
//     s  = Q^T w                                 (mass_inner_product, MDOT p)
//
// The unfused sequence reads Q twice (8n(p+3) + 8n(p+1) bytes); here every
// CTA stages a tile of T rows of all p columns of Q plus w in shared memory
// by TMA bulk copies (one elected thread, completion counted on a
// per-buffer mbarrier, double-buffered one tile ahead), computes the
// projected rows from shared memory, writes u and w once, and sweeps the
// same staged tile again for Q^T w -- 8n(p+3) bytes per call.
//
//   phase A (rows): thread t owns row t of the tile and evaluates exactly the
//     K2 expression in K2's order (fma chain over k, then the u column), so
//     u and w are bitwise equal to lagged_update's;
//   phase B (columns): (column, lane-rows) items dealt to the 8 warps, one
//     register accumulator per item across all tiles of the CTA, no shuffles
//     in the loop; butterfly at the end and the last CTA sums the per-CTA
//     partials in a fixed order (deterministic).
#include "tile.cuh"

namespace lsb {

namespace {

constexpr int kMaxK3Cols = 110;   // p + 1 staged columns at most (2 stages of 128 rows)
constexpr int kMaxStages = 8;
constexpr size_t kK3Smem = 220 * 1024;   // ring budget (of the 227 KB opt-in)

inline size_t k3_stage_bytes(int p, int T) { return (size_t)(p + 1) * T * sizeof(double); }
inline size_t k3_smem(int p, int T, int ns) {
  return ns * k3_stage_bytes(p, T) + sizeof(double) * (p + 16);   // + coefficients (padded)
}

// Ring of NS stages of T rows x (p+1) columns, NS-1 tiles in flight while one
// is computed: a single 100 KB double buffer leaves the copy engine idle
// half the time (the in-flight bytes drain to zero before the next issue).
template <int SLOTS, int T>
__global__ void __launch_bounds__(kThreads, 2)
lagged_update_reduce_kernel(lsb_arnoldi S, int it, int p, int ks, int ns, int direct, int spread,
                            double* __restrict__ out, double* __restrict__ partial,
                            unsigned* counter) {
  pdl_enter();
  if (gated_off(S.flags, it)) return;
  if (!direct && S.flags && S.flags->broke_iter == it) return;
  static_assert(T % 64 == 0 && (T <= kThreads || T % kThreads == 0), "tile rows");
  constexpr int kRpt = T > kThreads ? T / kThreads : 1;   // rows per thread, phase A
  constexpr int kPairs = T / 64;            // double2 per lane per item
  extern __shared__ __align__(16) double dyn[];
  double* stage_base = dyn;                 // [ns][p+1][T]
  double* sc = dyn + (size_t)ns * (p + 1) * T;
  __shared__ __align__(8) uint64_t bars[kMaxStages];
  __shared__ double red[kWarps * SLOTS];
  __shared__ bool is_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < p; k += kThreads) sc[k] = direct ? S.coef2[k] : S.coef[k];
  if (threadIdx.x == 0) {
    for (int b = 0; b < ns; ++b) mbar_init(&bars[b], 1);
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t ld = S.ld, n = S.n;
  double* __restrict__ u = S.V + (int64_t)(p - 1) * ld;
  double* __restrict__ w = S.V + (int64_t)p * ld;
  const double beta = S.scal[LSB_S_BETA];
  const double cu = sc[p - 1];
  const int cols = p + 1;                   // Q[:, 0..p-1] and w
  auto col_of = [&](int b, int k) { return stage_base + ((size_t)b * cols + k) * T; };

  // stage rows [a, a+T) of every column: lane 0 of warp w issues the bulk
  // copies of columns w, w+8, ... (one thread issuing all p+1 copies puts
  // ~100 cycles per copy on the critical path) and arrives on the buffer's
  // barrier (count 8) with its own byte count.  The (single) ragged last
  // tile is loaded by plain zero-filled loads and arrives with 0 bytes.
  auto stage = [&](int b, int64_t tt) {
    const int64_t a = tt * T;
    if (a + T <= n) {
      if (spread) {
        // one CTA per SM: one copy per thread, threads 128.. first -- for
        // T <= 128 those warps sit out phase A, so the issue overlaps the
        // row work of warps 0..3 (p = 101: 5.7 -> 6.5 TB/s)
        if (threadIdx.x == 0) mbar_arrive_tx(&bars[b], (unsigned)(cols * T * sizeof(double)));
        for (int k = (threadIdx.x + kThreads / 2) % kThreads; k < cols; k += kThreads)
          bulk_g2s(col_of(b, k), S.V + (int64_t)k * ld + a, T * sizeof(double), &bars[b]);
      } else if (lane == 0) {
        // two CTAs per SM: the warp leaders (the other CTA's rows hide it)
        if (warp == 0) mbar_arrive_tx(&bars[b], (unsigned)(cols * T * sizeof(double)));
        for (int k = warp; k < cols; k += kWarps)
          bulk_g2s(col_of(b, k), S.V + (int64_t)k * ld + a, T * sizeof(double), &bars[b]);
      }
    } else {
      for (int e = threadIdx.x; e < cols * T; e += kThreads) {
        const int k = e / T, r = e % T;
        col_of(b, k)[r] = a + r < n ? S.V[(int64_t)k * ld + a + r] : 0.0;
      }
      fence_proxy_async();
      __syncthreads();
      if (threadIdx.x == 0) mbar_arrive_tx(&bars[b], 0u);
    }
  };

  double acc[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) acc[s] = 0.0;

  const int64_t ntiles = (n + T - 1) / T;
  const int64_t G = gridDim.x;
  const int64_t mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / G + 1 : 0;
  for (int s = 0; s < ns - 1 && s < mine; ++s) stage(s, blockIdx.x + s * G);
  unsigned phase = 0;   // bit b: parity of buffer b's next completion
  for (int64_t lt = 0; lt < mine; ++lt) {
    const int buf = (int)(lt % ns);
    mbar_wait(&bars[buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;
    __syncthreads();                        // every warp is done with tile lt-1
    if (lt + ns - 1 < mine) stage((int)((lt + ns - 1) % ns), blockIdx.x + (lt + ns - 1) * G);
    const int64_t a = (blockIdx.x + lt * G) * T;

    // phase A: the K2 row expression; thread t owns rows t, t+256, ... of
    // the tile (independent fma chains interleaved for ILP)
    if (threadIdx.x < T) {
      double accr[kRpt];
#pragma unroll
      for (int i = 0; i < kRpt; ++i) accr[i] = 0.0;
      const int kend = direct ? p : p - 1;
#pragma unroll 4
      for (int k = 0; k < kend; ++k) {
        const double c = sc[k];
        const double* q = col_of(buf, k) + threadIdx.x;
#pragma unroll
        for (int i = 0; i < kRpt; ++i) accr[i] = fma(c, q[i * kThreads], accr[i]);
      }
#pragma unroll
      for (int i = 0; i < kRpt; ++i) {
        const int r = threadIdx.x + i * kThreads;
        if (direct) {   // cgs_project's z - Q s (its fma(-s, q, .) chain is this one negated)
          const double zz = col_of(buf, p)[r] - accr[i];
          if (a + r < n) w[a + r] = zz;
          col_of(buf, p)[r] = a + r < n ? zz : 0.0;
          continue;
        }
        const double uu = __ddiv_rn(col_of(buf, p - 1)[r], beta);
        const double acc1 = fma(cu, uu, accr[i]);
        double ww = col_of(buf, p)[r];
        if (ks) ww = __ddiv_rn(ww, beta);
        ww = ww - acc1;
        if (a + r < n) {
          u[a + r] = uu;
          w[a + r] = ww;
        }
        col_of(buf, p - 1)[r] = a + r < n ? uu : 0.0;
        col_of(buf, p)[r] = a + r < n ? ww : 0.0;
      }
    }
    fence_proxy_async();                    // generic writes before the next TMA into buf
    __syncthreads();

    // phase B: s_k += Q[:, k] . w over this tile, items k = warp + 8 s
    const double2* wt = reinterpret_cast<const double2*>(col_of(buf, p));
    double2 wv[kPairs];
#pragma unroll
    for (int q = 0; q < kPairs; ++q) wv[q] = wt[lane + 32 * q];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int k = warp + kWarps * s;
      if (k < p) {
        const double2* qc = reinterpret_cast<const double2*>(col_of(buf, k));
        double x = 0.0;
#pragma unroll
        for (int q = 0; q < kPairs; ++q) {
          const double2 qv = qc[lane + 32 * q];
          x = fma(qv.x, wv[q].x, x);
          x = fma(qv.y, wv[q].y, x);
        }
        acc[s] += x;
      }
    }
  }

  // CTA totals, per-CTA partials, fixed-order sum in the last CTA
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const double x = warp_sum(acc[s]);
    if (lane == 0) red[warp + kWarps * s] = x;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < p; k += kThreads) partial[(size_t)k * G + blockIdx.x] = red[k];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == (unsigned)G - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int k = warp; k < p; k += kWarps) {
    double x = 0.0;
    for (int c = lane; c < G; c += 32) x += __ldcg(partial + (size_t)k * G + c);
    x = warp_sum(x);
    if (lane == 0) out[k] = x;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// Shared-memory plan (tools/kk3.py sweep on B200, n = 2^24): what matters
// is two resident CTAs per SM -- one sweeps its tile while the other's
// copies land -- with the widest tile that allows it.  So: the largest
// T in {1024, 512, 256, 128} whose two stages fit half the SM (112 KB),
// as many stages as that half holds; past p ~ 54 one CTA of T = 128 rows.
constexpr size_t kK3Half = 112 * 1024;
inline size_t k3_coef(int p) { return sizeof(double) * (p + 16); }
inline bool k3_half_fits(int p, int T) { return 2 * k3_stage_bytes(p, T) + k3_coef(p) <= kK3Half; }

inline int k3_stages(int p, int T) {
  const int cap = tuning(LSB_TUNE_K3_STAGES);
  // the knob asks for exactly `cap` stages out of the whole budget (one CTA
  // per SM when they do not fit half of it)
  const size_t budget = (k3_half_fits(p, T) && cap < 2) ? kK3Half : kK3Smem;
  int ns = (int)((budget - k3_coef(p)) / k3_stage_bytes(p, T));
  if (cap >= 2 && ns > cap) ns = cap;
  return ns < kMaxStages ? ns : kMaxStages;
}

template <int SLOTS, int T>
int launch_k3_t(const lsb_arnoldi& S, int it, int p, int ks, int direct, cudaStream_t st) {
  auto kern = lagged_update_reduce_kernel<SLOTS, T>;
  const int ns = k3_stages(p, T);
  const size_t sm = k3_smem(p, T, ns);
  static size_t configured = 0;
  if (sm > configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
        cudaSuccess)
      return check_launch("lagged_update_reduce-smem");
    configured = sm;
  }
  static int occ_cache[kMaxK3Cols + 1][kMaxStages + 1];   // smem depends on (p, ns)
  int& occ = occ_cache[p][ns];
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, sm);
    if (occ < 1) occ = 1;
  }
  const int64_t ntiles = (S.n + T - 1) / T;
  int64_t grid = (int64_t)sm_count() * occ;
  if (S.ws.grid > 0 && S.ws.grid < grid) grid = S.ws.grid;
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  const int spread = occ < 2;
  // two-sync chain (K5a -> K3 -> K5b -> K4): PDL only for p <= 32 -- at
  // p ~ 50 it cost 3-4% per step at n = 2^21..2^22 (tools/c3_sweep.py A/B)
  const cudaError_t le = launch_chain(use_pdl(S.n) && p <= 32, kern, dim3((unsigned)grid), dim3(kThreads), sm, st, S, it, p, ks, ns, direct, spread, S.Gloc, S.ws.partial,
                                             S.ws.counter);
  return check_launch("lagged_update_reduce", le);
}

template <int T>
int launch_k3_rows(const lsb_arnoldi& S, int it, int p, int ks, int direct, cudaStream_t st) {
  const int s = (p + kWarps - 1) / kWarps;
  if (s <= 1) return launch_k3_t<1, T>(S, it, p, ks, direct, st);
  if (s <= 2) return launch_k3_t<2, T>(S, it, p, ks, direct, st);
  if (s <= 4) return launch_k3_t<4, T>(S, it, p, ks, direct, st);
  if constexpr (T > 256) {
    return LSB_ERANGE;   // wide tiles only for p <= 32
  } else {
    if (s <= 7) return launch_k3_t<7, T>(S, it, p, ks, direct, st);
    if (s <= 10) return launch_k3_t<10, T>(S, it, p, ks, direct, st);
    if (s <= 13) return launch_k3_t<13, T>(S, it, p, ks, direct, st);
    return launch_k3_t<16, T>(S, it, p, ks, direct, st);
  }
}

}  // namespace

// Tile rows for p (0: p above the kernel's column limit).  Knob
// LSB_TUNE_K3_ROWS forces 64..1024 for experiments (512/1024 need p <= 32).
int k3_tile_rows(int p) {
  if (p < 1 || p + 1 > kMaxK3Cols) return 0;
  const int forced = tuning(LSB_TUNE_K3_ROWS);
  if ((forced == 64 || forced == 128 || forced == 192 || forced == 256 ||
       ((forced == 512 || forced == 1024) && p <= 32)) &&
      k3_stages(p, forced) >= 2)
    return forced;
  for (int T = 1024; T >= 128; T /= 2) {
    if ((T <= 256 || p <= 32) && k3_half_fits(p, T)) return T;
    if (T == 256 && k3_half_fits(p, 192) && tuning(LSB_TUNE_K3_ROWS) != 128) return 192;
  }
  if (k3_stages(p, 128) >= 2) return 128;
  return k3_stages(p, 64) >= 2 ? 64 : 0;
}

int launch_lagged_update_reduce(const lsb_arnoldi& S, int it, int p, int ks, int direct, cudaStream_t st) {
  if (S.n <= 0) {
    cudaMemsetAsync(S.Gloc, 0, sizeof(double) * p, st);
    return check_launch("lagged_update_reduce-empty");
  }
  switch (k3_tile_rows(p)) {
    case 1024: return launch_k3_rows<1024>(S, it, p, ks, direct, st);
    case 512: return launch_k3_rows<512>(S, it, p, ks, direct, st);
    case 256: return launch_k3_rows<256>(S, it, p, ks, direct, st);
    case 192: return launch_k3_rows<192>(S, it, p, ks, direct, st);
    case 128: return launch_k3_rows<128>(S, it, p, ks, direct, st);
    case 64: return launch_k3_rows<64>(S, it, p, ks, direct, st);
    default: return LSB_ERANGE;
  }
}

// lsb_preload: one kernel of this translation unit (its module)
const void* tu_anchor_project() { return (const void*)lagged_update_reduce_kernel<1, 128>; }

}  // namespace lsb
