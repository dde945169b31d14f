// Persistent cluster cycle: a whole lagged one-sync GMRES(m) restart cycle
// (Arnoldi iterations 0..m of gmres.py:389-466 with mgs_lvl2,
// gram_schmidt.py:206-245) in ONE launch of ONE thread-block cluster.
//
// At launch-bound sizes (C1: n = 4,096) the per-iteration kernels spend
// their time in launch and grid-reduction latency, not in HBM traffic.  Here
// one control CTA and up to 15 row CTAs form one cluster.  Each row CTA
// holds a contiguous row block of EVERY basis column (and its CSR rows) in
// shared memory; the control CTA holds the whole small state (R, T, the
// rotations, g, the rotated triangle, flags).  Nothing touches HBM during
// the cycle: V and the small state are copied in at launch and out at the
// end, for the cycle epilogue kernels.  Per iteration:
//   row CTAs: SpMV of the own rows (CSR, u of every row read from its
//     owner CTA through distributed shared memory, numpy row order = the
//     K7 bits), partial [Q^T u, Q^T w] of the own rows, pushed into the
//     control CTA's shared memory with st.async (completion counted in
//     bytes on the control CTA's mbarrier: the row CTA does not wait)
//   -> handoff (1): the control CTA waits on its mbarrier, sums the
//      partials in rank order and runs K5: warp 0 the breakdown test, warps
//      1..15 the T column and c = T^T y / beta (persist_small; same
//      arithmetic as mgs_small_body), then pushes c, beta and the flags
//      into every row CTA the same way
//   -> handoff (2): row CTAs wait on their own mbarrier and apply the K2 row
//      update; the control CTA arrives at cluster barrier (3) at once and
//      folds the Givens rotation meanwhile (pipeline2's deferral: a
//      convergence it finds cancels the next iteration at handoff (2), so
//      the stop semantics are exact)
//   -> cluster barrier (3) (the next SpMV reads the updated column).
// Two point-to-point handoffs and one cluster barrier per iteration replace
// four kernel launches and three grid-wide last-CTA reductions (measured on
// this B200, tools/micro: a st.async push + reply round trip ~900 cycles at
// 16 CTAs; a release/acquire cluster barrier 490, 1,057 after a DSMEM
// store).  Only shared memory is written inside the loop, so the barrier's
// release never waits for global stores.
//
// Results: SpMV, beta, T, c, Givens and the K2 row expression follow the
// per-iteration kernels; the mdot sums (per-CTA warp trees + rank-ordered
// cluster sum instead of the K1 tree) and the small T / c dot products
// (warp trees) are summed in a different order, so histories agree with the
// multi-kernel path to rounding (tests/test_gpu_parity.py).
#include <cooperative_groups.h>

#include "small_body.cuh"
#include "tile.cuh"

#ifndef LSB_PERSIST_REFNORM
#define LSB_PERSIST_REFNORM 1
#endif

namespace lsb {

namespace cgx = cooperative_groups;

constexpr int kPT = 512;            // threads per CTA
constexpr int kPWarps = kPT / 32;
constexpr int kPMaxCap = 128;       // basis columns (p + 1 <= cap)
constexpr int kPMaxCluster = 16;
constexpr size_t kPMaxSmem = 200 * 1024;   // + ~10 KB static <= 227 KB

// Phase anatomy (tuning knob LSB_TUNE_PERSIST_TRACE, read back with
// lsb_persist_trace): SM-cycle sums over iterations >= 1 -- [0..4] CTA 1:
// SpMV+dots, wait at barrier 1, wait at barrier 2 (= CTA 0's gather + small
// state), K2, wait at barrier 3 (= the fold beyond K2); [5..7] CTA 0:
// small-state front, T column, c; [8] iterations summed.
constexpr int kTraceSlots = 18;
__device__ long long g_ptrace[kTraceSlots];

__device__ __forceinline__ void cluster_barrier() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// st.async: a store into another CTA's shared memory whose completion is
// counted (in bytes) on that CTA's mbarrier -- the producer does not wait,
// the consumer waits on its own barrier (no cluster-wide rendezvous).
__device__ __forceinline__ uint32_t mapa_u32(const void* local_smem, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"((uint32_t)__cvta_generic_to_shared(local_smem)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v2(uint32_t dst, double a, double b, uint32_t bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
          dst),
      "d"(a), "d"(b), "r"(bar)
      : "memory");
}
// Consumer side of a handoff.  A handoff that never completes is a protocol
// bug (every byte pushed is counted on the consumer's barrier).  The wait is
// bounded in WALL time -- LSB_TUNE_PERSIST_TIMEOUT_S seconds (0: 30 s; < 0:
// unbounded), read through the launch -- so slowness (compute-sanitizer,
// time slicing, a debugger stepping) cannot trip it: a handoff takes ~1 us.
// On expiry the kernel writes -1.0 into the report marker of the mapped log
// (the host's poll raises a clear error from it) and aborts the grid.  It
// cannot return cooperatively: the other CTAs sit at hardware cluster
// barriers, which have no timeout, and a CTA that skipped its part would
// leave them waiting forever.
struct PersistAbort {
  double* marker;       // the current report's marker slot (mapped log), or null
  long long limit_ns;   // <= 0: unbounded
};
__device__ __forceinline__ unsigned long long persist_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, unsigned parity,
                                                      const PersistAbort& ab) {
  unsigned done = 0;
  unsigned spins = 0;
  unsigned long long t0 = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity)
        : "memory");
    if (done || ab.limit_ns <= 0) continue;
    if (++spins == 1024u) t0 = persist_ns();
    if (spins > 1024u && (spins & 1023u) == 0u && (long long)(persist_ns() - t0) > ab.limit_ns) {
      if (ab.marker) {
        *reinterpret_cast<volatile double*>(ab.marker) = -1.0;
        __threadfence_system();
      }
      __trap();
    }
  }
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Row sum in numpy's order with every product load issued before the first
// add: rows of <= 8 / <= 32 entries go through a compile-time plan
// (np_row_sum_fixed) selected by a switch, longer rows through np_row_sum.
template <int C, class Acc>
__device__ __forceinline__ double row_sum_c(const Acc& a) {
  double q[C];
#pragma unroll
  for (int k = 0; k < C; ++k) q[k] = a(k);
  return np_row_sum_fixed<C>(q);
}
template <class Acc>
__device__ __forceinline__ double row_sum_fast(const Acc& a, int cnt) {
  switch (cnt) {
    case 0: return 0.0;
#define LSB_RS(c) case c: return row_sum_c<c>(a);
    LSB_RS(1) LSB_RS(2) LSB_RS(3) LSB_RS(4) LSB_RS(5) LSB_RS(6) LSB_RS(7) LSB_RS(8)
    LSB_RS(9) LSB_RS(10) LSB_RS(11) LSB_RS(12) LSB_RS(13) LSB_RS(14) LSB_RS(15) LSB_RS(16)
    LSB_RS(17) LSB_RS(18) LSB_RS(19) LSB_RS(20) LSB_RS(21) LSB_RS(22) LSB_RS(23) LSB_RS(24)
    LSB_RS(25) LSB_RS(26) LSB_RS(27) LSB_RS(28) LSB_RS(29) LSB_RS(30) LSB_RS(31) LSB_RS(32)
#undef LSB_RS
    default: return np_row_sum(a, cnt);
  }
}

// CSR row products with x = a basis column held, row block by row block, in
// the shared memory of the cluster's CTAs (read through DSMEM).
struct CsrRowAccCluster {
  const int32_t* col;
  const double* val;
  const double* d;
  double* const* peer;   // peer[c] = CTA c's V block (shared memory, DSMEM address)
  size_t coloff;         // column offset inside a block
  FastDiv rdiv;          // division by rows per CTA
  int rows;
  // col / val: this CTA's nonzeros staged in shared memory at launch, or
  // the global arrays (plain loads: the pointers may be either)
  __device__ double operator()(int64_t j) const {
    const uint32_t c = (uint32_t)col[j];
    const uint32_t blk = rdiv.div(c);            // row block; owned by CTA blk + 1
    double xv = peer[blk + 1][coloff + (c - blk * (uint32_t)rows)];
    if (d) xv = __dmul_rn(xv, __ldg(d + c));
    return __dmul_rn(val[j], xv);
  }
};

// The cycle's small state in CTA 0's shared memory: the lsb_arnoldi arrays
// the K5 code touches, copied in at launch and out at the end, so no global
// store is outstanding at a cluster barrier (each barrier.cluster.arrive
// .release would otherwise wait for them to reach L2).
// K5 of the control CTA (gram_schmidt.py:226-245 with krylov_scale; the
// Givens fold is deferred), arranged for latency: warp 0 runs the breakdown
// test (beta, ||R[:p-1,p-1]||, CPython hypot -- gram_schmidt.py:96-106)
// while warps 1..15 speculatively compute the new T column and
// c = T^T y / beta straight into the state.  On a breakdown the cycle ends
// at this iteration and those slots (T[:, p-1], R[:, p], coef) are never
// read again -- the least squares uses the rotated triangle and the host's
// Hessenberg view stops at column p-1.  Same arithmetic as mgs_small_body
// except that the T column and c dot products are warp trees (not serial
// sums).  scratch: cap doubles.
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ void persist_small(const lsb_arnoldi& L, SmallShared& sh, double* scratch, int it,
                              int p, int ks, long long* stamps) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, cap = L.cap;
  constexpr int kW = kPT / 32 - 1;          // speculating warps
  double* Tnew = scratch;                    // T[:p, p-1] (read back by the c sums)
  if (stamps && t == 0) stamps[4] = clock64();
  for (int e = t; e < p; e += kPT) {
    sh.a[e] = L.G[2 * e];
    sh.y[e] = L.G[2 * e + 1];
    if (e < p - 1) sh.col[e] = L.R[(int64_t)e * cap + (p - 1)];
  }
  __syncthreads();
  if (stamps && t == 0) stamps[0] = clock64();
  const double bsq = sh.a[p - 1];
  const double beta = bsq > 0.0 ? sqrt(bsq) : 0.0;
  if (wid == 0) {
    // ---- breakdown test (lagged_front)
    double ss = 0.0;
    for (int j = lane; j < p - 1; j += 32) ss = fma(sh.col[j], sh.col[j], ss);
    ss = warp_sum(ss);
    if (lane == 0) {
      const double tol = breakdown_tol(L, beta, sh.col, p - 1, ss);
      sh.beta = beta;
      sh.tol = tol;
      sh.broke = beta <= tol;
      L.scal[LSB_S_BETA] = beta;
      L.scal[LSB_S_TOL] = tol;
      if (sh.broke) {
        L.flags->broke_iter = it;
        if (it == 0) { L.flags->stop_iter = it; L.flags->status = LSB_STARTUP_BREAKDOWN; }
        sh.col[p - 1] = 0.0;
      } else {
        sh.col[p - 1] = beta;
        L.R[(int64_t)(p - 1) * cap + (p - 1)] = beta;
      }
      if (stamps) stamps[5] = clock64();
    }
  } else {
    // ---- speculative T column and c (mgs_small_body)
    const int u = t - 32;                    // 0 .. 32*kW-1
    for (int e = u; e < p - 1; e += 32 * kW) sh.a[e] = __ddiv_rn(sh.a[e], beta);
    const double ylast = __ddiv_rn(sh.y[p - 1], beta);
    named_bar(1, 32 * kW);
    if (stamps && t == 32) stamps[1] = clock64();
    for (int j = wid - 1; j < p - 1; j += kW) {
      double acc = 0.0;
      for (int l = j + lane; l < p - 1; l += 32) acc = fma(L.T[(int64_t)j * cap + l], sh.a[l], acc);
      acc = warp_sum(acc);
      if (lane == 0) {
        Tnew[j] = -acc;
        L.T[(int64_t)j * cap + (p - 1)] = -acc;
      }
    }
    if (u == 0) {
      Tnew[p - 1] = 1.0;
      L.T[(int64_t)(p - 1) * cap + (p - 1)] = 1.0;
    }
    named_bar(1, 32 * kW);
    if (stamps && t == 32) stamps[2] = clock64();
    for (int j = wid - 1; j < p; j += kW) {
      double acc = 0.0;
      for (int l = lane; l <= j; l += 32) {
        const double tl = j == p - 1 ? Tnew[l] : L.T[(int64_t)l * cap + j];
        acc = fma(tl, l == p - 1 ? ylast : sh.y[l], acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) {
        const double c = ks ? __ddiv_rn(acc, beta) : acc;
        L.coef[j] = c;
        L.R[(int64_t)j * cap + p] = c;
      }
    }
  }
  __syncthreads();
  if (stamps && t == 0) stamps[3] = clock64();
}

// Multi-cycle mode (x != nullptr): after each cycle the kernel also runs the
// cycle epilogue and the next cycle's prologue itself -- the least squares
// (cycle_lsq), x += M^-1 V y (extract), the restart residual b - A x and its
// norm, the restart test -- logging one report per cycle for the host, so a
// whole restarted solve is one launch.
struct PersistSolve {
  double* x;          // local rows of the iterate (global), nullptr: one cycle only
  const double* b;    // local rows of b
  double* log;        // max_cycles reports of kLogStride(m) doubles
  int max_cycles;
  long long timeout_ns;   // handoff wait limit (PersistAbort)
};
__host__ __device__ inline int log_stride(int m) { return 4 + (m + 1) + LSB_S_COUNT + 1; }

__global__ void __launch_bounds__(kPT, 1)
persist_cycle_kernel(lsb_arnoldi S, lsb_csr A, int rows, FastDiv rdiv, int ks, int stage_cap,
                     bool trace, PersistSolve PS) {
  cgx::cluster_group cl = cgx::this_cluster();
  const int crank = (int)cl.block_rank(), csize = (int)cl.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int cap = S.cap, m = S.m;
  const StateLayout SL = StateLayout::make(cap, m);
  extern __shared__ __align__(16) double dyn[];
  double* Vs = dyn;                          // cap columns x rows: own rows of V
  double* xs = Vs + (size_t)cap * rows;      // rows: x (multi-cycle; read remotely at xoff)
  double* bs = xs + rows;                    // rows: b
  double* rs = bs + rows;                    // rows: the restart residual
  const size_t xoff = (size_t)cap * rows;
  double* allp = Vs + (((size_t)(cap + 3) * rows + 1) & ~(size_t)1);   // [16][2*cap]: every CTA's [Q^T u, Q^T w]
                                             // (pushed into CTA 0's copy over DSMEM)
  double* sc = allp + kPMaxCluster * 2 * cap;  // cap: coefficients (row CTAs' copy)
  double* st = sc + cap;                     // SL.total: the small state (CTA 0)
  double* scratch = st + SL.total;           // 2*cap: speculative T column and c (CTA 0)
  double* cval = scratch + 2 * cap;          // stage_cap: this CTA's CSR values
  int32_t* ccol = reinterpret_cast<int32_t*>(cval + stage_cap);   // stage_cap: columns
  int32_t* crp = ccol + stage_cap;           // rows + 1: row offsets into them
  __shared__ SmallShared sh;
  __shared__ double* s_peer[kPMaxCluster];
  // published by CTA 0 before barrier (2): [0] beta, [1] breakdown at this
  // iteration (K2 skipped, cycle over), [2] this iteration runs (0 when the
  // previous iteration's deferred Givens fold stopped the cycle)
  __shared__ double s_pub[3];
  __shared__ __align__(16) double s_pubr[4];   // row CTAs: CTA 0's pushed s_pub
  __shared__ __align__(8) uint64_t mb1, mb2;    // partials in (CTA 0) / coef + pub in (row CTAs)
  __shared__ int s_go, s_stop;
  __shared__ __align__(16) double s_ctl[4];     // row CTAs: pushed epilogue control values
  __shared__ __align__(16) double s_y[kPMaxCap + 2];   // row CTAs: pushed least-squares y
  // CTA 0 is the control CTA (reductions, small state, Givens fold) and
  // owns no rows; row block b lives in CTA b + 1
  const int64_t r0 = crank == 0 ? S.n : (int64_t)(crank - 1) * rows;
  const int64_t r1 = min(r0 + (int64_t)rows, S.n);
  const int nr = r1 > r0 ? (int)(r1 - r0) : 0;
  for (int j = tid; j < nr; j += kPT) Vs[j] = S.V[r0 + j];   // V[:, 0] = r / beta
  // the CTA's CSR rows into shared memory when they fit (read every iteration)
  const int64_t blo = nr ? A.row_ptr[r0] : 0, bhi = nr ? A.row_ptr[r0 + nr] : 0;
  const bool cstaged = bhi - blo <= stage_cap;
  const int32_t* rowp = A.row_ptr;
  const int32_t* colp = A.col_idx;
  const double* valp = A.values;
  if (cstaged) {
    for (int64_t e = tid; e < bhi - blo; e += kPT) {
      cval[e] = A.values[blo + e];
      ccol[e] = A.col_idx[blo + e];
    }
    for (int j = tid; j <= nr; j += kPT) crp[j] = (int32_t)(A.row_ptr[r0 + j] - blo);
    rowp = crp;
    colp = ccol;
    valp = cval;
  }
  const int64_t rbase = cstaged ? 0 : r0;    // row index base into rowp
  if (tid < csize) s_peer[tid] = tid == crank ? Vs : cl.map_shared_rank(Vs, tid);
  lsb_arnoldi L = S;   // CTA 0: the same state, shared-memory resident
  L.R = st + SL.R;
  L.T = st + SL.T;
  L.tri = st + SL.tri;
  L.rot = st + SL.rot;
  L.g = st + SL.g;
  L.res = st + SL.res;
  L.coef = st + SL.coef;
  L.G = st + SL.G;
  L.scal = st + SL.scal;
  L.flags = reinterpret_cast<lsb_flags*>(st + SL.flags);
  L.g_parts = 1;
  if (crank == 0) {
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
  }
  if (tid == 0) {
    const int stop = S.flags->stop_iter, broke = S.flags->broke_iter;
    s_go = !(stop < 0 || (broke >= 0 && broke < 0));   // gated_off(flags, 0)
    s_stop = 0;
  }
  if (tid == 0) {
    mbar_init(&mb1, 1);
    mbar_init(&mb2, 1);
    mbar_fence_init();
  }
  const uint32_t allp0 = mapa_u32(allp + crank * 2 * cap, 0);   // this CTA's slot at CTA 0
  const uint32_t mb1_0 = mapa_u32(&mb1, 0);
  long long tr[kTraceSlots] = {0};
  long long tc = 0;
  bool bad = false;
  int produced = 1;   // basis columns holding data (row CTAs)
  const bool multi = PS.x != nullptr;
  if (multi)
    for (int j = tid; j < nr; j += kPT) {
      xs[j] = PS.x[r0 + j];
      bs[j] = PS.b[r0 + j];
    }
  unsigned ph1 = 0, ph2 = 0;   // completed phases of mb1 / mb2 (parity of the next wait)
  cluster_barrier();

  PersistAbort ab{nullptr, PS.timeout_ns};
  for (int cyc = 0; cyc < (multi ? PS.max_cycles : 1); ++cyc) {
  if (multi) ab.marker = PS.log + (int64_t)cyc * log_stride(m) + 4 + (m + 1) + LSB_S_COUNT;
  produced = 1;
  for (int i = 0; i <= m; ++i) {
    const int p = i + 1;
    __syncthreads();
    if (!s_go) break;    // the cycle was stopped before it began (same in every CTA)
    const bool tw = trace && crank == 1 && tid == 0 && i > 0;
    if (tw) tc = clock64();
    // row CTAs expect this iteration's coefficients + flags from CTA 0
    if (crank != 0 && tid == 0) mbar_arrive_tx(&mb2, (unsigned)(8 * (((p + 1) & ~1) + 4)));
    double* su = Vs + (size_t)(p - 1) * rows;   // u = V[:, p-1], own rows
    double* sw = Vs + (size_t)p * rows;         // w = V[:, p]

    // ---- w = A u on the own rows (V.push(A v_i), gmres.py:411); u of
    // every row from its owner's shared memory
    for (int j = tid; j < nr; j += kPT) {
      const int lo = rowp[rbase + j], hi = rowp[rbase + j + 1];
      const double s = row_sum_fast(CsrRowAccCluster{colp + lo, valp + lo, A.col_scale,
                                                     s_peer, (size_t)(p - 1) * rows, rdiv, rows},
                                    hi - lo);
      if (!isfinite(s)) bad = true;
      sw[j] = s;
    }
    if (tw) { const long long t = clock64(); tr[9] += t - tc; }
    __syncthreads();
    if (tw) { const long long t = clock64(); tr[10] += t - tc; }

    // ---- partial [Q^T u, Q^T w] of the own rows: warp wid takes columns
    // wid, wid + 16, ...; lanes stride the rows
    for (int k = wid; k < p && crank != 0; k += kPWarps) {
      const double* q = Vs + (size_t)k * rows;
      double a = 0.0, b = 0.0;
#pragma unroll 4
      for (int j = lane; j < nr; j += 32) {
        const double qv = q[j];
        a = fma(qv, su[j], a);
        b = fma(qv, sw[j], b);
      }
      a = warp_sum(a);
      b = warp_sum(b);
      if (lane == 0)     // into CTA 0's shared memory, counted on its barrier
        st_async_v2(allp0 + 16u * (uint32_t)k, a, b, mb1_0);
    }
    if (tw) { const long long t = clock64(); tr[0] += t - tc; tc = t; }

    // ---- CTA 0: cluster sum in rank order (the partials already sit in
    // its shared memory), then the K5 small state -- all of it resident in
    // this CTA's shared memory for the whole cycle.  Unless the previous
    // iteration's Givens fold stopped the cycle: then this iteration never
    // happened (its SpMV touched only the shared copy of a column that is
    // not written back).
    const bool tc0 = trace && crank == 0 && tid == 0 && i > 0;
    long long c0a = 0;
    if (tc0) c0a = clock64();
    if (crank == 0) {
      // (1) every row CTA's partials have landed (always waited: no st.async
      // may still be in flight into this CTA when the cycle ends)
      if (tid == 0) mbar_arrive_tx(&mb1, (unsigned)(16 * p * (csize - 1)));
      mbar_wait_acq_cluster(&mb1, ph1++ & 1u, ab);
      if (!s_stop) {
        for (int e = tid; e < 2 * p; e += kPT) {
          double acc = 0.0;
          for (int c = 1; c < csize; ++c) acc += allp[c * 2 * cap + e];
          L.G[e] = acc;
        }
        __syncthreads();
        if (tc0) { const long long t = clock64(); tr[14] += t - c0a; }
        __shared__ long long sm[6];
        persist_small(L, sh, scratch, i, p, ks, (trace && i > 0) ? sm : nullptr);
        if (tc0) { const long long t = clock64(); tr[15] += t - c0a; }
        if (trace && i > 0 && tid == 0 && !sh.broke) {
          tr[5] += sm[1] - sm[0];
          tr[6] += sm[2] - sm[1];
          tr[7] += sm[3] - sm[2];
          tr[9] += sm[0] - sm[4];     // entry -> first sync (control CTA)
          tr[10] += sm[5] - sm[0];    // warp 0: breakdown test done (from the first sync)
        }
      }
      if (tid == 0) {
        s_pub[0] = sh.beta;
        s_pub[1] = sh.broke ? 1.0 : 0.0;
        s_pub[2] = s_stop ? 0.0 : 1.0;
      }
      __syncthreads();
      // (2) push coefficients + flags into every row CTA (st.async, counted
      // on the row CTA's mb2); the full byte count even when stopping
      const int pe = (p + 1) & ~1, per = pe / 2 + 2;
      for (int e = tid; e < (csize - 1) * per; e += kPT) {
        const int c = 1 + e / per, q = e - (c - 1) * per;
        const uint32_t bar = mapa_u32(&mb2, c);
        if (q < pe / 2)
          st_async_v2(mapa_u32(sc + 2 * q, c), L.coef[2 * q], L.coef[2 * q + 1], bar);
        else if (q == pe / 2)
          st_async_v2(mapa_u32(s_pubr, c), s_pub[0], s_pub[1], bar);
        else
          st_async_v2(mapa_u32(s_pubr + 2, c), s_pub[2], 0.0, bar);
      }
    }
    if (tc0) { const long long t = clock64(); tr[11] += t - c0a; c0a = t; }
    const double* pub0 = s_pub;
    if (crank != 0) {
      mbar_wait_acq_cluster(&mb2, ph2++ & 1u, ab);
      pub0 = s_pubr;
    }
    if (tw) { const long long t = clock64(); tr[2] += t - tc; tc = t; }
    if (tc0) { const long long t = clock64(); tr[12] += t - c0a; tr[13] += 1; }
    if (pub0[2] == 0.0) break;             // fold i-1 converged: no iteration i
    if (pub0[1] != 0.0) {                  // breakdown: K2 skipped, cycle over
      if (crank == 0 && i > 0) settle_block(L, sh, i, i, true, /*resident=*/true);
      produced = p + 1;
      break;
    }

    if (crank == 0) {
      // Givens fold of Hessenberg column i-1 (gmres.py:427-435), deferred
      // as in the pipeline2 schedule (gmres.py:444-462): the control CTA
      // arrives at barrier (3) first, so the fold overlaps the row CTAs'
      // K2 and, past the barrier, the next SpMV and partial dots; a
      // convergence it detects cancels the next iteration at barrier (2).
      cluster_arrive();
      if (i > 0) settle_block(L, sh, i, i, false, /*resident=*/true);
      __syncthreads();
      if (tid == 0) s_stop = L.flags->stop_iter <= i;
      cluster_wait();
    } else {
      // ---- K2 on the own rows (gram_schmidt.py:230-242; lagged_update_kernel's
      // row expression)
      const double beta = pub0[0];
      const double cu = sc[p - 1];
      for (int j = tid; j < nr; j += kPT) {
        double acc = 0.0;
        for (int k = 0; k < p - 1; ++k) acc = fma(sc[k], Vs[(size_t)k * rows + j], acc);
        const double uu = __ddiv_rn(su[j], beta);
        su[j] = uu;
        acc = fma(cu, uu, acc);
        double ww = sw[j];
        if (ks) ww = __ddiv_rn(ww, beta);
        sw[j] = ww - acc;
      }
      produced = p + 1;
      if (tw) { const long long t = clock64(); tr[3] += t - tc; tc = t; }
      cluster_barrier();   // (3) the next SpMV reads the updated column
      if (tw) { const long long t = clock64(); tr[4] += t - tc; tr[8] += 1; }
    }
  }
  if (!multi) break;

  // ================= cycle epilogue + next prologue (multi-cycle) =========
  const int pe_y = (cap + 1) & ~1;
  // row CTAs arm for the least-squares push; the control CTA for the
  // residual-norm partials -- before the barrier that precedes those pushes
  if (crank != 0 && tid == 0) mbar_arrive_tx(&mb2, (unsigned)(8 * (pe_y + 2)));
  if (crank == 0 && tid == 0) mbar_arrive_tx(&mb1, (unsigned)(32 * (csize - 1)));
  cluster_barrier();
  if (crank == 0) {
    // (E1) least squares on the rotated triangle (cycle_lsq_kernel,
    // gmres.py:184-192 / 294-297): y into scratch, k and status in flags
    if (wid == 0) {
      const int stop = L.flags->stop_iter;
      const int k = L.flags->status == LSB_GHYSELS_CHECK ? 0 : (stop == LSB_NO_STOP ? m : stop);
      if (lane == 0) L.flags->k = k;
      __syncwarp();
      for (int ii = k - 1; ii >= 0; --ii) {
        const double dd = L.tri[(int64_t)ii * m + ii];
        if (dd == 0.0) {
          if (lane == 0) { L.flags->status = LSB_SINGULAR; L.flags->k = ii; }
          break;
        }
        double acc = 0.0;
        for (int j = ii + 1 + lane; j < k; j += 32) acc = fma(L.tri[(int64_t)ii * m + j], scratch[j], acc);
        acc = warp_sum(acc);
        if (lane == 0) scratch[ii] = __ddiv_rn(L.g[ii] - acc, dd);
        __syncwarp();
      }
    }
    __syncthreads();
    // (E2) y, k and the status into every row CTA
    const int kk = L.flags->k, stt = L.flags->status, per = pe_y / 2 + 1;
    for (int e = tid; e < (csize - 1) * per; e += kPT) {
      const int c = 1 + e / per, q = e - (c - 1) * per;
      const uint32_t bar = mapa_u32(&mb2, c);
      if (q < pe_y / 2)
        st_async_v2(mapa_u32(s_y + 2 * q, c), 2 * q < kk ? scratch[2 * q] : 0.0,
                    2 * q + 1 < kk ? scratch[2 * q + 1] : 0.0, bar);
      else
        st_async_v2(mapa_u32(s_ctl, c), (double)kk, (double)stt, bar);
    }
  } else {
    mbar_wait_acq_cluster(&mb2, ph2++ & 1u, ab);
    // (E3) x += M^-1 V_k y on the own rows (extract_kernel's expression)
    const int kk = (int)s_ctl[0], stt = (int)s_ctl[1];
    if (kk >= 1 && stt != LSB_SINGULAR)
      for (int j = tid; j < nr; j += kPT) {
        double acc = 0.0;
        for (int jj = 0; jj < kk; ++jj) acc = fma(s_y[jj], Vs[(size_t)jj * rows + j], acc);
        if (A.col_scale) acc = __dmul_rn(acc, A.col_scale[r0 + j]);
        xs[j] = xs[j] + acc;
      }
    // the next pushes from the control CTA: the rescale decision
    if (tid == 0) mbar_arrive_tx(&mb2, 16u);
  }
  cluster_barrier();   // x complete everywhere (the residual SpMV reads neighbours' x)
  {
    // (E4) r = b - A x on the own rows (A itself: gmres.py:498), then the
    // (max |r|, sum r^2) partial of norm_partial_kernel
    __shared__ double s_red[kPWarps][2];
    __shared__ int s_bad;
    double am = 0.0, ss = 0.0;
    for (int j = tid; j < nr; j += kPT) {
      const int lo = rowp[rbase + j], hi = rowp[rbase + j + 1];
      const double sx = row_sum_fast(CsrRowAccCluster{colp + lo, valp + lo, nullptr, s_peer, xoff,
                                                      rdiv, rows},
                                     hi - lo);
      if (!isfinite(sx)) bad = true;
      const double v = __dsub_rn(bs[j], sx);
      rs[j] = v;
      am = fmax(am, fabs(v));
      if (isnan(v)) am = v;
      ss = fma(v, v, ss);
    }
    am = warp_max(am);
    ss = warp_sum(ss);
    if (lane == 0) { s_red[wid][0] = am; s_red[wid][1] = ss; }
    const int anybad = __syncthreads_or(bad ? 1 : 0);
    if (crank != 0 && tid == 0) {
      double a = s_red[0][0], q = s_red[0][1];
      for (int w = 1; w < kPWarps; ++w) { a = fmax(a, s_red[w][0]); if (isnan(s_red[w][0])) a = s_red[w][0]; q += s_red[w][1]; }
      st_async_v2(allp0, a, q, mb1_0);
      st_async_v2(allp0 + 16u, anybad ? 1.0 : 0.0, 0.0, mb1_0);
    }
    bad = false;
    (void)s_bad;
  }
  // (E5) the control CTA: the restart norm (norm_finish_kernel), with the
  // exact power-of-two rescale pass when max|r| leaves [2^-450, 2^450]
  __shared__ double s_nrm[3];   // rnorm, rescale flag, scale
  if (crank == 0) {
    mbar_wait_acq_cluster(&mb1, ph1++ & 1u, ab);
    if (tid == 0) {
      double amax = allp[1 * 2 * cap], ssq = allp[1 * 2 * cap + 1];
      int nf = allp[1 * 2 * cap + 2] != 0.0;
      for (int c = 2; c < csize; ++c) {
        amax = fmax(amax, allp[c * 2 * cap]);
        ssq += allp[c * 2 * cap + 1];
        nf |= allp[c * 2 * cap + 2] != 0.0;
      }
      if (nf) L.flags->nonfinite = 1;
      const double lo = 0x1p-450, hi = 0x1p450;
#if LSB_PERSIST_REFNORM
      (void)lo; (void)hi;
      const bool resc = !(amax == 0.0 || isnan(amax));
      const double sc_ = amax;
#else
      const bool resc = !(amax == 0.0 || isnan(amax) || (amax >= lo && amax <= hi));
      double sc_ = 1.0;
      if (resc) {
        int e;
        frexp(amax, &e);
        sc_ = ldexp(1.0, -e);
      }
#endif
      s_nrm[0] = amax == 0.0 ? 0.0 : (isnan(amax) ? amax : sqrt(ssq));
      s_nrm[1] = resc ? 1.0 : 0.0;
      s_nrm[2] = sc_;
      if (resc) mbar_arrive_tx(&mb1, (unsigned)(16 * (csize - 1)));
    }
    __syncthreads();
    for (int c = 1 + tid; c < csize; c += kPT)
      st_async_v2(mapa_u32(s_ctl + 2, c), s_nrm[1], s_nrm[2], mapa_u32(&mb2, c));
    if (s_nrm[1] != 0.0) {
      mbar_wait_acq_cluster(&mb1, ph1++ & 1u, ab);
      if (tid == 0) {
        double q = allp[1 * 2 * cap];
        for (int c = 2; c < csize; ++c) q += allp[c * 2 * cap];
#if LSB_PERSIST_REFNORM
        s_nrm[0] = s_nrm[2] * sqrt(q);
#else
        s_nrm[0] = sqrt(q) / s_nrm[2];
#endif
      }
    }
    __syncthreads();
    // (E6) restart test, the cycle's report, continue or stop
    if (tid == 0) {
      const double rn = s_nrm[0];
      L.scal[LSB_S_RNORM] = rn;
      L.flags->restart_ok = rn <= L.scal[LSB_S_TARGET];
      const bool cont = !L.flags->nonfinite && L.flags->status == LSB_RUNNING &&
                        L.flags->stop_iter == LSB_NO_STOP && !L.flags->restart_ok &&
                        cyc + 1 < PS.max_cycles;
      s_nrm[1] = cont ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int c = 1 + tid; c < csize; c += kPT)
      st_async_v2(mapa_u32(s_ctl, c), s_nrm[1], s_nrm[0], mapa_u32(&mb2, c));
    // the cycle's report (the log may be mapped host memory that the host
    // polls while later cycles run): payload, system fence, then the
    // marker -- 2.0 when another cycle follows, 1.0 for the last one
    if (wid == 0) {
      double* rep = PS.log + (int64_t)cyc * log_stride(m);
      const double* fl = reinterpret_cast<const double*>(L.flags);
      for (int e = lane; e < 4 + (m + 1) + LSB_S_COUNT; e += 32)
        rep[e] = e < 4 ? fl[e] : (e < 5 + m ? L.res[e - 4] : L.scal[e - 5 - m]);
      __threadfence_system();
      __syncwarp();
      if (lane == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile double*>(rep + 4 + (m + 1) + LSB_S_COUNT) =
            s_nrm[1] != 0.0 ? 2.0 : 1.0;
      }
    }
  } else {
    mbar_wait_acq_cluster(&mb2, ph2++ & 1u, ab);         // rescale decision
    if (tid == 0) mbar_arrive_tx(&mb2, 16u);          // next: continue + rnorm
    __syncthreads();
    if (s_ctl[2] != 0.0) {                             // rescaled sum of squares
      __shared__ double s_q[kPWarps];
      const double scl = s_ctl[3];
      double q = 0.0;
      for (int j = tid; j < nr; j += kPT) {
#if LSB_PERSIST_REFNORM
        const double v = __ddiv_rn(rs[j], scl);
#else
        const double v = rs[j] * scl;
#endif
        q = fma(v, v, q);
      }
      q = warp_sum(q);
      if (lane == 0) s_q[wid] = q;
      __syncthreads();
      if (tid == 0) {
        double a = s_q[0];
        for (int w = 1; w < kPWarps; ++w) a += s_q[w];
        st_async_v2(allp0, a, 0.0, mb1_0);
      }
    }
    mbar_wait_acq_cluster(&mb2, ph2++ & 1u, ab);         // continue + rnorm
  }
  __syncthreads();
  const bool cont = (crank == 0 ? s_nrm[1] : s_ctl[0]) != 0.0;
  if (!cont) break;
  // (E7) next cycle's prologue: V[:, 0] = r / beta (scale_div) and a fresh
  // small state with g[0] = beta (cycle_begin_kernel)
  if (crank != 0) {
    const double rn = s_ctl[1];
    for (int j = tid; j < nr; j += kPT) Vs[j] = __ddiv_rn(rs[j], rn);
  } else {
    for (int e = tid; e < cap * cap; e += kPT) { L.R[e] = 0.0; L.T[e] = 0.0; }
    for (int e = tid; e < (m + 1) * m; e += kPT) L.tri[e] = 0.0;
    for (int e = tid; e < 2 * m; e += kPT) L.rot[e] = 0.0;
    for (int e = tid; e <= m; e += kPT) { L.g[e] = 0.0; L.res[e] = 0.0; }
    for (int e = tid; e < cap; e += kPT) L.coef[e] = 0.0;
    __syncthreads();
    if (tid == 0) {
      L.g[0] = L.scal[LSB_S_RNORM];
      L.flags->stop_iter = LSB_NO_STOP;
      L.flags->status = LSB_RUNNING;
      L.flags->broke_iter = -1;
      L.flags->k = 0;
      L.flags->restart_ok = 0;
      s_stop = 0;
    }
  }
  cluster_barrier();   // V[:, 0] everywhere, state reset
  }   // cycles
  if (!multi && bad)
    atomicOr(reinterpret_cast<int*>(cl.map_shared_rank(L.flags, 0)) + 4, 1);  // nonfinite
  if (multi) {
    for (int j = tid; j < nr; j += kPT) PS.x[r0 + j] = xs[j];
  }
  // the basis columns this cycle produced, own rows, back to HBM
  for (int k = 0; k < produced; ++k)
    for (int j = tid; j < nr; j += kPT) S.V[(int64_t)k * S.ld + r0 + j] = Vs[(size_t)k * rows + j];
  // no CTA may exit while a peer can still touch its shared memory
  cluster_barrier();
  if (crank == 0) {    // the small state back to HBM for the cycle epilogue
    copy_d(S.R, L.R, cap * cap);
    copy_d(S.T, L.T, cap * cap);
    copy_d(S.tri, L.tri, (m + 1) * m);
    copy_d(S.rot, L.rot, 2 * m);
    copy_d(S.g, L.g, m + 1);
    copy_d(S.res, L.res, m + 1);
    copy_d(S.coef, L.coef, cap);
    copy_d(S.G, L.G, 2 * cap);
    copy_d(S.scal, L.scal, LSB_S_COUNT);
    if (tid < (int)(sizeof(lsb_flags) / sizeof(int)))
      reinterpret_cast<int*>(S.flags)[tid] = reinterpret_cast<const int*>(L.flags)[tid];
  }
  if (trace && tid == 0 && (crank == 1 || crank == 0)) {
    if (crank == 1) {
      for (int k = 0; k < 5; ++k) g_ptrace[k] = tr[k];
      g_ptrace[9] = tr[9];
      g_ptrace[10] = tr[10];
    }
    else
      for (int k = 5; k < 8; ++k) g_ptrace[k] = tr[k];
    if (crank == 0) {
      for (int k = 11; k < 16; ++k) g_ptrace[k] = tr[k];
      g_ptrace[6 + 10] = tr[9];
      g_ptrace[6 + 11] = tr[10];
    }
    if (crank == 1) g_ptrace[8] = tr[8];
  }
}

// Cluster shape for (n, cap, m): one control CTA + up to 15 row CTAs of
// ~256 rows, each CTA holding its rows of all cap basis columns plus the
// small state in shared memory.  Returns the CTA count, 0 if no fit.
static int persist_plan(int64_t n, int cap, int m, int* rows_out, size_t* smem_out,
                        int* stage_out = nullptr) {
  if (n < 1 || cap < 2 || cap > kPMaxCap || cap > kSmall || m + 2 > cap) return 0;
  int csize = 1 + (int)((n + 255) / 256);
  const int forced = tuning(LSB_TUNE_PERSIST_CTAS);
  if (forced >= 2 && forced <= kPMaxCluster) csize = forced;
  if (csize < 2) csize = 2;
  if (csize > kPMaxCluster) csize = kPMaxCluster;
  const int64_t rows = (n + csize - 2) / (csize - 1);
  const size_t smem = sizeof(double) * ((size_t)(cap + 3) * rows + 1 + (2 * kPMaxCluster + 3) * cap +
                                        StateLayout::make(cap, m).total);
  if (smem > kPMaxSmem) return 0;
  // what is left stages the CTA's CSR rows (12 B per nonzero + row offsets)
  int64_t stage = ((int64_t)kPMaxSmem - (int64_t)smem - 4 * (rows + 2)) / 12;
  stage = stage < 0 ? 0 : (stage > (1 << 20) ? (1 << 20) : stage);
  stage &= ~(int64_t)1;                      // keeps the int32 arrays 8-byte aligned
  *rows_out = (int)rows;
  *smem_out = smem + 12 * (size_t)stage + 4 * (size_t)(rows + 2);
  if (stage_out) *stage_out = (int)stage;
  return csize;
}

int persist_trace(long long* out, int count) {
  if (count > kTraceSlots) count = kTraceSlots;
  if (cudaMemcpyFromSymbol(out, g_ptrace, sizeof(long long) * count) != cudaSuccess)
    return check_launch("persist_trace");
  return LSB_OK;
}

int persist_fits(int64_t n, int cap) {
  int rows;
  size_t sm;
  return persist_plan(n, cap, cap - 2, &rows, &sm) > 0;
}

int launch_cycle_persistent(const lsb_arnoldi& S, const lsb_csr* A, int ks, cudaStream_t st,
                            double* x, const double* b, double* log, int max_cycles) {
  if (x && (!b || !log || max_cycles < 1)) return LSB_EINVAL;
  if (!A || S.g_parts != 1 || S.m + 2 > S.cap || A->n_rows != S.n || A->n_cols != S.n ||
      A->x_lo != 0 || A->nnz >= (1LL << 31))
    return LSB_ERANGE;
  int rows = 0, stage = 0;
  size_t smem = 0;
  const int csize = persist_plan(S.n, S.cap, S.m, &rows, &smem, &stage);
  if (!csize) return LSB_ERANGE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(persist_cycle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kPMaxSmem);
    cudaFuncSetAttribute(persist_cycle_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)csize, 1, 1);
  cfg.blockDim = dim3(kPT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const lsb_csr Av = *A;
  const bool trace = tuning(LSB_TUNE_PERSIST_TRACE) == 1;
  const int tmo = tuning(LSB_TUNE_PERSIST_TIMEOUT_S);
  const long long limit = tmo < 0 ? 0LL : (long long)(tmo ? tmo : 30) * 1000000000LL;
  const PersistSolve ps{x, b, log, x ? max_cycles : 1, limit};
  const cudaError_t le = cudaLaunchKernelEx(&cfg, persist_cycle_kernel, S, Av, rows,
                                            FastDiv::make((uint32_t)rows), ks, stage, trace, ps);
  return check_launch("cycle_persistent", le);
}

// lsb_preload: one kernel of this translation unit (its module)
const void* tu_anchor_persist() { return (const void*)persist_cycle_kernel; }

}  // namespace lsb
