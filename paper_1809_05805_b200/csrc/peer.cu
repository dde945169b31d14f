// Peer-memory collectives for the row-partitioned solve (one rank per GPU).
//
// The multi-rank Arnoldi iteration has exactly two exchange steps
// (SURVEY §8(e)): the all-gather of every rank's partial
// reduction vector (one per reduction event: 2p doubles for the one-sync
// fused reduction, gram_schmidt.py:195-203 / kernels.py:328-347) and the
// stencil's ghost z-planes before each SpMV.  Both are tiny next to the
// HBM passes of an iteration (a few KB, and one plane per neighbour), so
// what matters is latency and staying inside the CUDA graph -- not
// bandwidth.  Instead of NCCL calls issued from the host between kernels,
// each step is one kernel that writes straight into the peers' memory over
// NVLink / NVSwitch (the buffers are mapped into this process with CUDA IPC,
// or are plain device pointers when the ranks share a process) and
// signals with a release store of a monotonically increasing epoch; the
// consumer spins on its own (local) signal word with acquire loads.  The
// epochs live in device memory and are advanced by the kernels themselves,
// so a captured cycle graph replays without host involvement.
//
//   all-gather: rank r stores its `count` doubles (+ its nonfinite flag)
//     into slot r of every rank's mailbox (double-buffered by epoch parity:
//     a peer can be one exchange ahead, never two, because reaching exchange
//     e+1 needs this rank's signal of e+1, which it sends only after it has
//     consumed exchange e), signals, waits for all size signals of this
//     epoch, copies the size slots into `out` in rank order.  The caller
//     sums them in that fixed order on the device (small_body.cuh), so every
//     rank holds bit-identical small state whatever the interconnect does.
//   halo: every CTA stores its share of the first / last owned plane into
//     the ghost plane of rank-1 / rank+1's copy of the same vector; the last
//     CTA to finish (grid counter) signals both neighbours and waits for
//     their signals -- the next kernel on the stream reads complete ghosts.
//     A ghost region of a basis column is rewritten only in the next
//     restart cycle, after many all-gathers, so it is never overwritten
//     while its reader still needs it.
//
// A wait that does not complete within the timeout (a dead peer) records
// LSB_COMM_TIMEOUT in flags->comm_error and the error word and returns; the
// host raises at its next report -- no trap, no sticky context error.
#include "common.cuh"

namespace lsb {

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_release_sys(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_volatile(const double* p) {
  return *reinterpret_cast<const volatile double*>(p);
}

// Spin until *sig >= e; false on timeout.
__device__ bool wait_signal(const int64_t* sig, int64_t e, int64_t timeout_ns) {
  if (ld_acquire_sys(sig) >= e) return true;
  const uint64_t t0 = global_ns();
  unsigned k = 0;
  while (ld_acquire_sys(sig) < e) {
    if ((++k & 255u) == 0 && (int64_t)(global_ns() - t0) > timeout_ns) return false;
    __nanosleep(32);
  }
  return true;
}

__device__ void record_timeout(const lsb_peer& P, lsb_flags* flags) {
  P.epoch[2] = LSB_COMM_TIMEOUT;
  if (flags) flags->comm_error = LSB_COMM_TIMEOUT;
}

constexpr int kPeerThreads = 256;

__global__ void __launch_bounds__(kPeerThreads)
peer_allgather_kernel(lsb_peer P, const double* __restrict__ local, int count,
                      double* __restrict__ out, int out_stride, lsb_flags* flags) {
  __shared__ int64_t s_e;
  __shared__ int s_fail;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_e = P.epoch[0] + 1;
    s_fail = 0;
  }
  __syncthreads();
  const int64_t e = s_e;
  const size_t par = (size_t)(e & 1);
  const double nf = (flags && *((volatile const int*)&flags->nonfinite)) ? 1.0 : 0.0;
  // 1. my slot in every rank's mailbox (remote stores over NVLink)
  for (int q = 0; q < P.size; ++q) {
    double* dst = P.mbox[q] + (par * P.size + P.rank) * (size_t)P.slot;
    for (int i = tid; i < count; i += kPeerThreads) dst[i] = local[i];
    if (tid == 0) dst[count] = nf;
  }
  __threadfence_system();
  __syncthreads();
  // 2. signal every rank (thread q -> rank q), then wait for every rank's
  // signal in my own signal words (thread q <- rank q)
  if (tid < P.size) {
    st_release_sys(P.sig[tid] + P.rank, e);
    if (!wait_signal(P.sig[P.rank] + tid, e, P.timeout_ns)) s_fail = 1;
  }
  __syncthreads();
  if (s_fail) {
    if (tid == 0) record_timeout(P, flags);
    return;
  }
  __threadfence();
  // 3. the size slots in rank order
  const double* mine = P.mbox[P.rank] + par * P.size * (size_t)P.slot;
  for (int q = 0; q < P.size; ++q)
    for (int i = tid; i < count; i += kPeerThreads)
      out[(size_t)q * out_stride + i] = ld_volatile(mine + (size_t)q * P.slot + i);
  if (tid < P.size && flags && ld_volatile(mine + (size_t)tid * P.slot + count) != 0.0)
    flags->nonfinite = 1;   // every rank reports a NaN/Inf any rank's SpMV saw
  if (tid == 0) P.epoch[0] = e;
}

template <class T>
__global__ void __launch_bounds__(kPeerThreads)
peer_halo_kernel(lsb_peer P, const T* __restrict__ lo_src, T* lo_dst, const T* __restrict__ hi_src,
                 T* hi_dst, int64_t cnt, lsb_flags* flags) {
  const int64_t stride = (int64_t)gridDim.x * kPeerThreads;
  for (int64_t i = (int64_t)blockIdx.x * kPeerThreads + threadIdx.x; i < cnt; i += stride) {
    if (lo_dst) lo_dst[i] = lo_src[i];
    if (hi_dst) hi_dst[i] = hi_src[i];
  }
  __threadfence_system();
  __syncthreads();
  __shared__ bool s_last;
  __shared__ int s_fail;
  if (threadIdx.x == 0) {
    s_last = atomicAdd(P.counter, 1u) == gridDim.x - 1;
    s_fail = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t e = P.epoch[1] + 1;
  const int r = P.rank;
  // sig[size] = "from below" (rank-1 wrote my lower ghost), sig[size+1] =
  // "from above" (rank+1 wrote my upper ghost)
  if (threadIdx.x == 0 && r > 0) st_release_sys(P.sig[r - 1] + P.size + 1, e);
  if (threadIdx.x == 1 && r < P.size - 1) st_release_sys(P.sig[r + 1] + P.size, e);
  if (threadIdx.x == 0 && r > 0 && !wait_signal(P.sig[r] + P.size, e, P.timeout_ns)) s_fail = 1;
  if (threadIdx.x == 1 && r < P.size - 1 && !wait_signal(P.sig[r] + P.size + 1, e, P.timeout_ns))
    s_fail = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_fail) record_timeout(P, flags);
    P.epoch[1] = e;
    *P.counter = 0u;
  }
}

static bool peer_ok(const lsb_peer* P) {
  if (!P || P->size < 1 || P->size > LSB_PEER_MAX || P->rank < 0 || P->rank >= P->size ||
      !P->epoch || !P->counter)
    return false;
  for (int q = 0; q < P->size; ++q)
    if (!P->mbox[q] || !P->sig[q]) return false;
  return true;
}

static lsb_peer with_default_timeout(const lsb_peer* P) {
  lsb_peer Q = *P;
  if (Q.timeout_ns <= 0) Q.timeout_ns = 60LL * 1000 * 1000 * 1000;
  return Q;
}

int launch_peer_allgather(const lsb_peer* P, const double* local, int count, double* out,
                          int out_stride, lsb_flags* flags, cudaStream_t st) {
  if (!peer_ok(P) || count < 0 || count + 1 > P->slot || out_stride < count || !local || !out)
    return LSB_EINVAL;
  peer_allgather_kernel<<<1, kPeerThreads, 0, st>>>(with_default_timeout(P), local, count, out,
                                                    out_stride, flags);
  return check_launch("peer_allgather");
}

int launch_peer_halo(const lsb_peer* P, const double* lo_src, double* lo_dst,
                     const double* hi_src, double* hi_dst, int64_t plane, lsb_flags* flags,
                     cudaStream_t st) {
  if (!peer_ok(P) || plane < 0) return LSB_EINVAL;
  if ((P->rank > 0) != (lo_dst != nullptr) || (P->rank < P->size - 1) != (hi_dst != nullptr) ||
      (lo_dst && !lo_src) || (hi_dst && !hi_src))
    return LSB_EINVAL;
  const lsb_peer Q = with_default_timeout(P);
  auto al16 = [](const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; };
  const bool vec = plane % 2 == 0 && al16(lo_src) && al16(lo_dst) && al16(hi_src) && al16(hi_dst);
  const int64_t cnt = vec ? plane / 2 : plane;
  int64_t want = (cnt + kPeerThreads - 1) / kPeerThreads;
  const int64_t cap = 2 * (int64_t)sm_count();
  const int grid = (int)(want < 1 ? 1 : (want > cap ? cap : want));
  if (vec)
    peer_halo_kernel<double2><<<grid, kPeerThreads, 0, st>>>(
        Q, reinterpret_cast<const double2*>(lo_src), reinterpret_cast<double2*>(lo_dst),
        reinterpret_cast<const double2*>(hi_src), reinterpret_cast<double2*>(hi_dst), cnt, flags);
  else
    peer_halo_kernel<double><<<grid, kPeerThreads, 0, st>>>(Q, lo_src, lo_dst, hi_src, hi_dst,
                                                            cnt, flags);
  return check_launch("peer_halo");
}

// lsb_preload: one kernel of this translation unit (its module)
const void* tu_anchor_peer() { return (const void*)peer_allgather_kernel; }

}  // namespace lsb
