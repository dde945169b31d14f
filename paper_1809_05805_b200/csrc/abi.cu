// extern "C" entry points of liblsb200 (declared in include/lsb200.h).
#include <stdio.h>
#include <string.h>

#include "reduce.cuh"

namespace lsb {

static thread_local char g_err[512] = "";
static int g_sms = 0;
static int g_tune[LSB_TUNE_COUNT] = {0};

int tuning(int key) { return (key >= 0 && key < LSB_TUNE_COUNT) ? g_tune[key] : 0; }

int sm_count() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms < 1) g_sms = 1;
  }
  return g_sms;
}

int check_launch(const char* what, cudaError_t launch_status) {
  if (launch_status != cudaSuccess) {
    cudaGetLastError();   // clear the recorded copy
    snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(launch_status));
    return LSB_ECUDA;
  }
  return check_launch(what);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
    return LSB_ECUDA;
  }
  return LSB_OK;
}

// launchers defined in the other translation units
int launch_mdot(const double*, int64_t, int64_t, int, const double*, const double*, double*,
                const lsb_workspace*, const lsb_flags*, int, cudaStream_t);
int launch_maxpy(const double*, const double*, int64_t, int64_t, int, const double*, int, double*,
                 const lsb_flags*, int, cudaStream_t);
int launch_lagged_update(const lsb_arnoldi&, int, int, int, cudaStream_t,
                         const lsb_halo_push* = nullptr);
int launch_lagged_correct(const lsb_arnoldi&, int, int, cudaStream_t);
int launch_lagged_update_reduce(const lsb_arnoldi&, int, int, int, int, cudaStream_t);
int k3_tile_rows(int);
int launch_mgs1_pass(const lsb_arnoldi&, int, int, int, int, cudaStream_t);
int launch_mgs1_passes(const lsb_arnoldi&, int, int, int, cudaStream_t);
int launch_cgs_project(const lsb_arnoldi&, int, int, int, int, cudaStream_t);
int launch_norm_partial(const double*, int64_t, double*, const lsb_workspace*, const lsb_flags*,
                        int, cudaStream_t);
int launch_norm_finish(const double*, int, int, const double*, int64_t, double*,
                       const lsb_workspace*, const lsb_flags*, int, cudaStream_t);
int launch_norm_scaled_partial(const double*, int, int, const double*, int64_t, double*,
                               const lsb_workspace*, cudaStream_t);
int launch_norm_finish_scaled(const double*, const double*, int, int, int, double*, cudaStream_t);
int launch_scale_div(const double*, int64_t, const double*, double*, const lsb_flags*, int, int,
                     cudaStream_t);
int launch_extract(const lsb_arnoldi&, double*, const double*, cudaStream_t);
int launch_stencil(const lsb_stencil*, const double*, const double*, double*, lsb_flags*, int,
                   cudaStream_t);
int launch_csr(const lsb_csr*, const double*, const double*, double*, lsb_flags*, int,
               cudaStream_t);
int launch_csr_dict(const lsb_csr_dict*, const double*, const double*, double*, lsb_flags*, int,
                    cudaStream_t);
int launch_mgs_lvl2_small(const lsb_arnoldi&, int, int, int, int, cudaStream_t);
int launch_cycle_persistent(const lsb_arnoldi&, const lsb_csr*, int, cudaStream_t, double*,
                            const double*, double*, int);
int persist_fits(int64_t, int);
int persist_trace(long long*, int);
int launch_cgs2_small_a(const lsb_arnoldi&, int, int, int, int, cudaStream_t);
int launch_cgs2_small_b(const lsb_arnoldi&, int, int, cudaStream_t);
int launch_collect_coef(const lsb_arnoldi&, int, int, int, cudaStream_t, int = 1, int = 0);
int launch_direct_small(const lsb_arnoldi&, int, int, int, int, cudaStream_t);
int launch_cycle_begin(const lsb_arnoldi&, cudaStream_t);
int launch_cycle_lsq(const lsb_arnoldi&, cudaStream_t);
int launch_restart_check(const lsb_arnoldi&, int, cudaStream_t);
int launch_givens_update(double*, double*, double*, int, const double*, int, double*, cudaStream_t);
int launch_lagged_reduce_spmv7(const lsb_arnoldi&, const lsb_stencil*, int, int, cudaStream_t,
                               const lsb_halo_wait* = nullptr, bool = false);
int launch_trial_lsq(const lsb_arnoldi&, int, double*, cudaStream_t);
int launch_ghysels_small(const lsb_arnoldi&, int, int, int, cudaStream_t, int = 1, int = 0);
int launch_settle(const lsb_arnoldi&, int, int, cudaStream_t);
int launch_trial_combine(const lsb_arnoldi&, int, const double*, const double*, double*,
                         const double*, cudaStream_t);
int launch_back_substitute(const double*, const double*, int, int, double*, int*, cudaStream_t);
int launch_cycle_grid(const lsb_arnoldi&, const lsb_csr*, int, double*, int64_t, cudaStream_t);
int grid_fits(int64_t, int);
int grid_trace(long long*, int);
int launch_sum_parts(const double*, int, int, int, double*, const lsb_flags*, int, cudaStream_t);
int launch_peer_allgather(const lsb_peer*, const double*, int, double*, int, lsb_flags*,
                          cudaStream_t);
int launch_peer_halo(const lsb_peer*, const double*, double*, const double*, double*, int64_t,
                     lsb_flags*, cudaStream_t);

// cuMemGetAddressRange through the runtime's driver entry point (no link
// dependency on libcuda: the library must load on hosts without a driver)
typedef int (*mem_range_fn)(unsigned long long*, size_t*, unsigned long long);
static mem_range_fn mem_range() {
  static mem_range_fn f = nullptr;
  if (!f) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<mem_range_fn>(p);
  }
  return f;
}
const void* tu_anchor_fused();
const void* tu_anchor_mdot();
const void* tu_anchor_project();
const void* tu_anchor_spmv();
const void* tu_anchor_peer();
const void* tu_anchor_persist();
const void* tu_anchor_small();
const void* tu_anchor_update();
const void* tu_anchor_gridcycle();

template <class F>
static F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

static int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return LSB_OK;
  snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
  return LSB_ECUDA;
}

static inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace lsb

using namespace lsb;

extern "C" {

const char* lsb_version(void) { return "lsb200 0.1 sm_100a"; }

int lsb_set_tuning(int32_t key, int32_t value) {
  if (key < 0 || key >= LSB_TUNE_COUNT) return -1;
  const int old = g_tune[key];
  g_tune[key] = value;
  return old;
}
const char* lsb_last_error(void) { return g_err; }
int lsb_sm_count(void) { return sm_count(); }
int32_t lsb_max_columns(void) { return 128; }

int64_t lsb_partial_len(int32_t pmax) {
  // grid <= sm_count * 8 CTAs (mdot occupancy is lower), entries <= 2*min(pmax,128)
  int64_t e = 2 * (int64_t)(pmax < 128 ? (pmax > 2 ? pmax : 2) : 128);
  return (int64_t)sm_count() * 8 * e + 64;
}

int lsb_spmv_csr(const lsb_csr* A, const double* x, const double* b, double* y, lsb_flags* flags,
                 int32_t it, void* stream) {
  if (!A || !x || !y) return LSB_EINVAL;
  return launch_csr(A, x, b, y, flags, it, S_(stream));
}

int lsb_spmv_csr_dict(const lsb_csr_dict* A, const double* x, const double* b, double* y,
                      lsb_flags* flags, int32_t it, void* stream) {
  if (!A || !x || !y) return LSB_EINVAL;
  return launch_csr_dict(A, x, b, y, flags, it, S_(stream));
}

int lsb_spmv_stencil(const lsb_stencil* S, const double* x, const double* b, double* y,
                     lsb_flags* flags, int32_t it, void* stream) {
  if (!S || !x || !y) return LSB_EINVAL;
  return launch_stencil(S, x, b, y, flags, it, S_(stream));
}

int lsb_mdot(const double* X, int64_t ld, int64_t n, int32_t p, const double* u, const double* w,
             double* out, const lsb_workspace* ws, const lsb_flags* flags, int32_t it,
             void* stream) {
  if (p < 0 || n < 0 || !ws || !out) return LSB_EINVAL;
  if (p > 0 && (!aligned16(X) || (ld & 1) || !aligned16(u) || (w && !aligned16(w))))
    return LSB_EINVAL;
  return launch_mdot(X, ld, n, p, u, w, out, ws, flags, it, S_(stream));
}

int lsb_maxpy(const double* y, const double* X, int64_t ld, int64_t n, int32_t p,
              const double* alpha, int32_t alpha_sign, double* out, const lsb_flags* flags,
              int32_t it, void* stream) {
  if (p < 0 || n < 0) return LSB_EINVAL;
  if (!aligned16(y) || !aligned16(out) || (p > 0 && (!aligned16(X) || (ld & 1))))
    return LSB_EINVAL;
  return launch_maxpy(y, X, ld, n, p, alpha, alpha_sign, out, flags, it, S_(stream));
}

int lsb_norm_partial(const double* x, int64_t n, double* out2, const lsb_workspace* ws,
                     const lsb_flags* flags, int32_t it, void* stream) {
  if (n < 0 || !ws) return LSB_EINVAL;
  return launch_norm_partial(x, n, out2, ws, flags, it, S_(stream));
}

int lsb_norm_finish(const double* parts, int32_t nparts, int32_t part_stride, const double* x,
                    int64_t n, double* out, const lsb_workspace* ws, const lsb_flags* flags,
                    int32_t it, void* stream) {
  if (nparts < 1 || !ws || (nparts > 1 && part_stride < 2)) return LSB_EINVAL;
  return launch_norm_finish(parts, nparts, part_stride, x, n, out, ws, flags, it, S_(stream));
}

int lsb_norm_scaled_partial(const double* parts, int32_t nparts, int32_t part_stride,
                            const double* x, int64_t n, double* out2, const lsb_workspace* ws,
                            void* stream) {
  if (nparts < 1 || !ws || !parts || !out2 || (nparts > 1 && part_stride < 2)) return LSB_EINVAL;
  return launch_norm_scaled_partial(parts, nparts, part_stride, x, n, out2, ws, S_(stream));
}

int lsb_norm_finish_scaled(const double* parts, const double* parts2, int32_t nparts,
                           int32_t part_stride, int32_t part2_stride, double* out, void* stream) {
  if (nparts < 1 || !parts || !parts2 || !out || (nparts > 1 && (part_stride < 2 || part2_stride < 1)))
    return LSB_EINVAL;
  return launch_norm_finish_scaled(parts, parts2, nparts, part_stride, part2_stride, out,
                                   S_(stream));
}

int lsb_scale_div(const double* x, int64_t n, const double* s, double* out,
                  const lsb_flags* flags, int32_t it, void* stream) {
  return launch_scale_div(x, n, s, out, flags, it, 0, S_(stream));
}

static int check_arnoldi(const lsb_arnoldi* S) {
  if (!S || !S->V || !S->flags || !S->scal || (S->ld & 1) || !aligned16(S->V)) return LSB_EINVAL;
  return LSB_OK;
}

int lsb_lagged_reduce(const lsb_arnoldi* S, int32_t it, int32_t p, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (p < 1 || p + 1 > S->cap) return LSB_ERANGE;
  const double* u = S->V + (int64_t)(p - 1) * S->ld;
  const double* w = S->V + (int64_t)p * S->ld;
  return launch_mdot(S->V, S->ld, S->n, p, u, w, S->Gloc, &S->ws, S->flags, it, S_(stream));
}

int lsb_lagged_reduce_spmv7(const lsb_arnoldi* S, const lsb_stencil* A, int32_t it, int32_t p,
                            void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (!A) return LSB_EINVAL;
  return launch_lagged_reduce_spmv7(*S, A, it, p, S_(stream));
}

int lsb_lagged_reduce_spmv7_norm(const lsb_arnoldi* S, const lsb_stencil* A, int32_t it, int32_t p,
                            void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (!A) return LSB_EINVAL;
  return launch_lagged_reduce_spmv7(*S, A, it, p, S_(stream), nullptr, true);
}

int lsb_mgs_lvl2_small(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                       int32_t givens_col, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_mgs_lvl2_small(*S, it, p, krylov_scale, givens_col, S_(stream));
}

int lsb_cycle_persistent(const lsb_arnoldi* S, const lsb_csr* A, int32_t krylov_scale,
                         void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (!A) return LSB_EINVAL;
  return launch_cycle_persistent(*S, A, krylov_scale, S_(stream), nullptr, nullptr, nullptr, 1);
}

int lsb_solve_persistent(const lsb_arnoldi* S, const lsb_csr* A, int32_t krylov_scale, double* x,
                         const double* b, double* log, int32_t max_cycles, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (!A || !x || !b || !log || max_cycles < 1) return LSB_EINVAL;
  return launch_cycle_persistent(*S, A, krylov_scale, S_(stream), x, b, log, max_cycles);
}

int lsb_cycle_persistent_fits(int64_t n, int32_t cap) { return persist_fits(n, cap); }

int lsb_persist_trace(int64_t* out, int32_t count) {
  if (!out || count < 0) return LSB_EINVAL;
  return persist_trace((long long*)out, count);
}

int lsb_cgs2_lvl2_small_a(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                          int32_t givens_col, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (!S->L) return LSB_EINVAL;
  return launch_cgs2_small_a(*S, it, p, krylov_scale, givens_col, S_(stream));
}

int lsb_cgs2_lvl2_small_b(const lsb_arnoldi* S, int32_t it, int32_t p, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_cgs2_small_b(*S, it, p, S_(stream));
}

int lsb_lagged_update(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                      void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (p < 1 || p + 1 > S->cap) return LSB_ERANGE;
  return launch_lagged_update(*S, it, p, krylov_scale, S_(stream));
}

int lsb_lagged_update_reduce(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                             void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (p < 1 || p + 1 > S->cap || !k3_tile_rows(p)) return LSB_ERANGE;
  if (!S->Gloc) return LSB_EINVAL;
  return launch_lagged_update_reduce(*S, it, p, krylov_scale, 0, S_(stream));
}

int lsb_lagged_correct(const lsb_arnoldi* S, int32_t it, int32_t p, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (p < 1 || p + 1 > S->cap) return LSB_ERANGE;
  return launch_lagged_correct(*S, it, p, S_(stream));
}

int lsb_mgs1_pass(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t k, int32_t p,
                  void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (k < 0 || k > p || col < p || col >= S->cap) return LSB_ERANGE;
  return launch_mgs1_pass(*S, it, col, k, p, S_(stream));
}

int lsb_mgs1_passes(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (p < 0 || col < p || col >= S->cap) return LSB_ERANGE;
  return launch_mgs1_passes(*S, it, col, p, S_(stream));
}

int lsb_collect_coef(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t accumulate,
                     void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_collect_coef(*S, it, p, accumulate, S_(stream));
}

int lsb_cgs_project(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p, int32_t want_norm,
                    void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (col < p || col >= S->cap) return LSB_ERANGE;
  return launch_cgs_project(*S, it, col, p, want_norm, S_(stream));
}

int lsb_cgs_project_reduce(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p,
                           void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (col != p || col >= S->cap || !k3_tile_rows(p)) return LSB_ERANGE;
  if (!S->Gloc) return LSB_EINVAL;
  return launch_lagged_update_reduce(*S, it, p, 0, 1, S_(stream));
}

int lsb_direct_small(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  const int gc = S->m > 0 ? col : 0;
  return launch_direct_small(*S, it, col, p, gc, S_(stream));
}

int lsb_settle(const lsb_arnoldi* S, int32_t it, int32_t col, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_settle(*S, it, col, S_(stream));
}

int lsb_ghysels_small(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_ghysels_small(*S, it, col, p, S_(stream));
}

int lsb_ghysels_small_pairs(const lsb_arnoldi* S, int32_t it, int32_t col, int32_t p,
                            void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_ghysels_small(*S, it, col, p, S_(stream), 2, 1);
}

int lsb_direct_normalize(const lsb_arnoldi* S, int32_t it, int32_t col, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  double* z = S->V + (int64_t)col * S->ld;
  return launch_scale_div(z, S->n, S->scal + LSB_S_BETA, z, S->flags, it, 1, S_(stream));
}

int lsb_cycle_begin(const lsb_arnoldi* S, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_cycle_begin(*S, S_(stream));
}

int lsb_cycle_lsq(const lsb_arnoldi* S, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_cycle_lsq(*S, S_(stream));
}

int lsb_cycle_extract(const lsb_arnoldi* S, double* x, const double* col_scale, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_extract(*S, x, col_scale, S_(stream));
}

int lsb_trial_lsq(const lsb_arnoldi* S, int32_t it, double* y, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_trial_lsq(*S, it, y, S_(stream));
}

int lsb_trial_combine(const lsb_arnoldi* S, int32_t it, const double* x, const double* y,
                      double* xt, const double* col_scale, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_trial_combine(*S, it, x, y, xt, col_scale, S_(stream));
}

int lsb_restart_check(const lsb_arnoldi* S, int32_t first, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_restart_check(*S, first, S_(stream));
}

int lsb_gram_row(const lsb_arnoldi* S, int32_t it, int32_t row, int32_t ncols, double* gram,
                 int64_t gram_ld, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (ncols < 1 || row < 0 || row >= S->cap) return LSB_ERANGE;
  const double* u = S->V + (int64_t)row * S->ld;
  return launch_mdot(S->V, S->ld, S->n, ncols, u, nullptr, gram + (int64_t)row * gram_ld, &S->ws,
                     S->flags, it, S_(stream));
}

int lsb_givens_update(double* rot, double* g, double* tri, int32_t m, const double* h, int32_t i,
                      double* res_out, void* stream) {
  return launch_givens_update(rot, g, tri, m, h, i, res_out, S_(stream));
}

int lsb_back_substitute(const double* tri, const double* g, int32_t m, int32_t k, double* y,
                        int32_t* status, void* stream) {
  return launch_back_substitute(tri, g, m, k, y, status, S_(stream));
}

int lsb_peer_allgather(const lsb_peer* P, const double* local, int32_t count, double* out,
                       int32_t out_stride, lsb_flags* flags, void* stream) {
  return launch_peer_allgather(P, local, count, out, out_stride, flags, (cudaStream_t)stream);
}

int lsb_peer_halo(const lsb_peer* P, const double* lo_src, double* lo_dst, const double* hi_src,
                  double* hi_dst, int64_t plane, lsb_flags* flags, void* stream) {
  return launch_peer_halo(P, lo_src, lo_dst, hi_src, hi_dst, plane, flags, (cudaStream_t)stream);
}

int lsb_ipc_export(const void* ptr, void* handle64, int64_t* offset) {
  if (!ptr || !handle64 || !offset) return LSB_EINVAL;
  mem_range_fn f = mem_range();
  if (!f) {
    snprintf(g_err, sizeof g_err, "lsb_ipc_export: cuMemGetAddressRange unavailable");
    return LSB_ECUDA;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (f(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0) {
    snprintf(g_err, sizeof g_err, "lsb_ipc_export: cuMemGetAddressRange failed");
    return LSB_ECUDA;
  }
  cudaIpcMemHandle_t h;
  const int rc = cuda_status(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base), "cudaIpcGetMemHandle");
  if (rc) return rc;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, sizeof h);
  *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
  return LSB_OK;
}

int lsb_ipc_open(const void* handle64, void** base) {
  if (!handle64 || !base) return LSB_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h);
  return cuda_status(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess),
                     "cudaIpcOpenMemHandle");
}

int lsb_ipc_close(void* base) {
  if (!base) return LSB_EINVAL;
  return cuda_status(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle");
}

int lsb_sum_parts(const double* parts, int32_t nparts, int32_t stride, int32_t count,
                  double* out, const lsb_flags* flags, int32_t it, void* stream) {
  if (!parts || !out || nparts < 1 || stride < count) return LSB_EINVAL;
  return launch_sum_parts(parts, nparts, stride, count, out, flags, it, S_(stream));
}

int lsb_cycle_grid(const lsb_arnoldi* S, const lsb_csr* A, int32_t krylov_scale, double* part,
                   int64_t part_len, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_cycle_grid(*S, A, krylov_scale, part, part_len, S_(stream));
}

int lsb_cycle_grid_fits(int64_t n, int32_t cap) { return grid_fits(n, cap); }

int lsb_grid_trace(int64_t* out, int32_t count) {
  return out ? grid_trace(reinterpret_cast<long long*>(out), count) : LSB_EINVAL;
}

int lsb_lagged_update_push(const lsb_arnoldi* S, int32_t it, int32_t p, int32_t krylov_scale,
                           const lsb_halo_push* hp, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (!hp) return LSB_EINVAL;
  return launch_lagged_update(*S, it, p, krylov_scale, S_(stream), hp);
}

int lsb_lagged_reduce_spmv7_halo(const lsb_arnoldi* S, const lsb_stencil* A, int32_t it,
                                 int32_t p, const lsb_halo_wait* hw, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  if (!hw || !hw->epoch) return LSB_EINVAL;
  return launch_lagged_reduce_spmv7(*S, A, it, p, S_(stream), hw);
}

int lsb_collect_coef_pairs(const lsb_arnoldi* S, int32_t it, int32_t p, void* stream) {
  if (int rc = check_arnoldi(S)) return rc;
  return launch_collect_coef(*S, it, p, 0, S_(stream), 2, 1);
}

int lsb_preload(void) {
  // Load every kernel of every module of the library now.  Under CUDA's
  // lazy loading a kernel's first launch loads it, and loading waits for
  // the context to go idle -- which never happens while an exchange kernel
  // of this context spins on a peer whose progress needs that launch (ranks
  // sharing one device).  Also keeps first-launch latency out of timings.
  typedef int (*get_module_fn)(void**, void*);
  typedef int (*count_fn)(unsigned*, void*);
  typedef int (*enum_fn)(void**, unsigned, void*);
  typedef int (*load_fn)(void*);
  static const get_module_fn get_module = driver_fn<get_module_fn>("cuFuncGetModule");
  static const count_fn count = driver_fn<count_fn>("cuModuleGetFunctionCount");
  static const enum_fn enumerate = driver_fn<enum_fn>("cuModuleEnumerateFunctions");
  static const load_fn load = driver_fn<load_fn>("cuFuncLoad");
  if (!get_module || !count || !enumerate || !load) {
    snprintf(g_err, sizeof g_err, "lsb_preload: driver lacks cuModuleEnumerateFunctions/cuFuncLoad");
    return -LSB_ECUDA;
  }
  const void* anchors[] = {tu_anchor_fused(), tu_anchor_mdot(), tu_anchor_project(),
                           tu_anchor_spmv(), tu_anchor_peer(), tu_anchor_persist(),
                           tu_anchor_small(), tu_anchor_update(), tu_anchor_gridcycle()};
  int loaded = 0;
  for (const void* a : anchors) {
    cudaFunction_t f;
    int rc = cuda_status(cudaGetFuncBySymbol(&f, a), "cudaGetFuncBySymbol");
    if (rc) return -rc;
    void* mod = nullptr;
    unsigned n = 0;
    if (get_module(&mod, (void*)f) || count(&n, mod)) {
      snprintf(g_err, sizeof g_err, "lsb_preload: cannot enumerate a module");
      return -LSB_ECUDA;
    }
    void* fs[512];
    if (n > 512) n = 512;
    if (enumerate(fs, n, mod)) {
      snprintf(g_err, sizeof g_err, "lsb_preload: cuModuleEnumerateFunctions failed");
      return -LSB_ECUDA;
    }
    for (unsigned k = 0; k < n; ++k)
      if (load(fs[k]) == 0) ++loaded;
  }
  return loaded;
}

}  // extern "C"
