"""ctypes binding of liblsb200.so (include/lsb200.h).

The library is the only compute path: if it is missing or cannot be loaded
every entry point raises ``LsbUnavailable`` -- there is no CPU fallback.
Structures below mirror the C structs field for field.
"""

from __future__ import annotations

import ctypes as C
import os
import warnings

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LSB200_LIB", os.path.join(_HERE, "liblsb200.so"))

OK, EINVAL, ECUDA, ERANGE = 0, 1, 2, 3
RUNNING, CONVERGED, BREAKDOWN, STARTUP_BREAKDOWN, SINGULAR, GHYSELS_CHECK = 0, 1, 2, 3, 4, 5
NO_STOP = 0x7FFFFFFF

# scalar slots (LSB_S_*)
S_BETA, S_TARGET, S_DENOM, S_RNORM, S_RELTOL, S_BTF, S_AMAX, S_SSQ, S_TOL, S_RAD = range(10)
S_COUNT = 16
MAX_OFF = 27
# lsb_set_tuning keys (include/lsb200.h LSB_TUNE_*)
TUNE_FUSED_OCC3, TUNE_FORCE_PARTS, TUNE_ROW_CTAS_PER_SM = 1, 2, 3
TUNE_K3_ROWS, TUNE_K3_STAGES, TUNE_CSR_THREAD_ROW = 4, 5, 6
TUNE_PERSIST_TRACE, TUNE_PERSIST_CTAS, TUNE_FUSED_PIPE, TUNE_CSR_DICT, TUNE_PDL = 7, 8, 9, 10, 11
TUNE_PERSIST_TIMEOUT_S = 12
TUNE_GRID_OCC, TUNE_GRID_TRACE, TUNE_S27_MARCH, TUNE_MGS1_GRID = 13, 14, 15, 16
TUNE_S27_TILE_Z = 17


class LsbUnavailable(RuntimeError):
    """liblsb200.so is not built / not loadable: no compute path exists."""


class LsbError(RuntimeError):
    """A liblsb200 entry point returned an error status."""


class Flags(C.Structure):
    _fields_ = [("stop_iter", C.c_int32), ("status", C.c_int32), ("broke_iter", C.c_int32),
                ("k", C.c_int32), ("nonfinite", C.c_int32), ("restart_ok", C.c_int32),
                ("comm_error", C.c_int32), ("pad", C.c_int32)]


FLAGS_INTS = C.sizeof(Flags) // 4


class Workspace(C.Structure):
    _fields_ = [("partial", C.c_void_p), ("counter", C.c_void_p), ("grid", C.c_int32),
                ("pad", C.c_int32)]


class CsrDict(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("val_idx", C.c_void_p), ("off_idx", C.c_void_p),
                ("val_tab", C.c_void_p), ("off_tab", C.c_void_p), ("n_val", C.c_int32),
                ("n_off", C.c_int32), ("col_scale", C.c_void_p), ("row0", C.c_int64),
                ("x_lo", C.c_int64)]


class Csr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p),
                ("col_scale", C.c_void_p), ("row0", C.c_int64), ("x_lo", C.c_int64)]


class Stencil(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("noff", C.c_int32),
                ("halo_lo", C.c_int32), ("halo_hi", C.c_int32),
                ("dx", C.c_int32 * MAX_OFF), ("dy", C.c_int32 * MAX_OFF),
                ("dz", C.c_int32 * MAX_OFF), ("val", C.c_double * MAX_OFF),
                ("col_scale", C.c_void_p)]


class Arnoldi(C.Structure):
    _fields_ = [("V", C.c_void_p), ("ld", C.c_int64), ("n", C.c_int64), ("n_global", C.c_int64),
                ("cap", C.c_int32), ("m", C.c_int32),
                ("R", C.c_void_p), ("T", C.c_void_p), ("L", C.c_void_p),
                ("rot", C.c_void_p), ("g", C.c_void_p), ("tri", C.c_void_p),
                ("coef", C.c_void_p), ("coef2", C.c_void_p),
                ("G", C.c_void_p), ("g_parts", C.c_int32), ("g_stride", C.c_int32),
                ("Gloc", C.c_void_p), ("scal", C.c_void_p), ("res", C.c_void_p),
                ("flags", C.c_void_p), ("ws", Workspace)]


PEER_MAX = 16
COMM_TIMEOUT = 1


class Peer(C.Structure):
    _fields_ = [("rank", C.c_int32), ("size", C.c_int32), ("slot", C.c_int32), ("pad", C.c_int32),
                ("timeout_ns", C.c_int64), ("mbox", C.c_void_p * PEER_MAX),
                ("sig", C.c_void_p * PEER_MAX), ("epoch", C.c_void_p), ("counter", C.c_void_p)]


class HaloPush(C.Structure):
    _fields_ = [("lo_dst", C.c_void_p), ("hi_dst", C.c_void_p), ("plane", C.c_int64),
                ("sig_lo", C.c_void_p), ("sig_hi", C.c_void_p), ("epoch", C.c_void_p),
                ("counter", C.c_void_p)]


class HaloWait(C.Structure):
    _fields_ = [("sig_lo", C.c_void_p), ("sig_hi", C.c_void_p), ("epoch", C.c_void_p),
                ("timeout_ns", C.c_int64), ("flags", C.c_void_p)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64

_SIGS = {
    "lsb_version": ([], C.c_char_p),
    "lsb_set_tuning": ([_I32, _I32], C.c_int),
    "lsb_last_error": ([], C.c_char_p),
    "lsb_sm_count": ([], C.c_int),
    "lsb_partial_len": ([_I32], _I64),
    "lsb_max_columns": ([], _I32),
    "lsb_spmv_csr": ([_P, _P, _P, _P, _P, _I32, _P], C.c_int),
    "lsb_spmv_csr_dict": ([_P, _P, _P, _P, _P, _I32, _P], C.c_int),
    "lsb_norm_scaled_partial": ([_P, _I32, _I32, _P, _I64, _P, _P, _P], C.c_int),
    "lsb_norm_finish_scaled": ([_P, _P, _I32, _I32, _I32, _P, _P], C.c_int),
    "lsb_spmv_stencil": ([_P, _P, _P, _P, _P, _I32, _P], C.c_int),
    "lsb_mdot": ([_P, _I64, _I64, _I32, _P, _P, _P, _P, _P, _I32, _P], C.c_int),
    "lsb_maxpy": ([_P, _P, _I64, _I64, _I32, _P, _I32, _P, _P, _I32, _P], C.c_int),
    "lsb_norm_partial": ([_P, _I64, _P, _P, _P, _I32, _P], C.c_int),
    "lsb_norm_finish": ([_P, _I32, _I32, _P, _I64, _P, _P, _P, _I32, _P], C.c_int),
    "lsb_scale_div": ([_P, _I64, _P, _P, _P, _I32, _P], C.c_int),
    "lsb_lagged_reduce": ([_P, _I32, _I32, _P], C.c_int),
    "lsb_lagged_reduce_spmv7": ([_P, _P, _I32, _I32, _P], C.c_int),
    "lsb_lagged_reduce_spmv7_norm": ([_P, _P, _I32, _I32, _P], C.c_int),
    "lsb_mgs_lvl2_small": ([_P, _I32, _I32, _I32, _I32, _P], C.c_int),
    "lsb_cgs2_lvl2_small_a": ([_P, _I32, _I32, _I32, _I32, _P], C.c_int),
    "lsb_cgs2_lvl2_small_b": ([_P, _I32, _I32, _P], C.c_int),
    "lsb_lagged_update": ([_P, _I32, _I32, _I32, _P], C.c_int),
    "lsb_lagged_update_reduce": ([_P, _I32, _I32, _I32, _P], C.c_int),
    "lsb_lagged_correct": ([_P, _I32, _I32, _P], C.c_int),
    "lsb_mgs1_pass": ([_P, _I32, _I32, _I32, _I32, _P], C.c_int),
    "lsb_mgs1_passes": ([_P, _I32, _I32, _I32, _P], C.c_int),
    "lsb_collect_coef": ([_P, _I32, _I32, _I32, _P], C.c_int),
    "lsb_collect_coef_pairs": ([_P, _I32, _I32, _P], C.c_int),
    "lsb_cgs_project": ([_P, _I32, _I32, _I32, _I32, _P], C.c_int),
    "lsb_cgs_project_reduce": ([_P, _I32, _I32, _I32, _P], C.c_int),
    "lsb_direct_small": ([_P, _I32, _I32, _I32, _P], C.c_int),
    "lsb_direct_normalize": ([_P, _I32, _I32, _P], C.c_int),
    "lsb_ghysels_small": ([_P, _I32, _I32, _I32, _P], C.c_int),
    "lsb_ghysels_small_pairs": ([_P, _I32, _I32, _I32, _P], C.c_int),
    "lsb_settle": ([_P, _I32, _I32, _P], C.c_int),
    "lsb_cycle_persistent": ([_P, _P, _I32, _P], C.c_int),
    "lsb_solve_persistent": ([_P, _P, _I32, _P, _P, _P, _I32, _P], C.c_int),
    "lsb_cycle_persistent_fits": ([C.c_int64, _I32], C.c_int),
    "lsb_cycle_grid": ([_P, _P, _I32, _P, _I64, _P], C.c_int),
    "lsb_cycle_grid_fits": ([C.c_int64, _I32], C.c_int),
    "lsb_grid_trace": ([_P, _I32], C.c_int),
    "lsb_persist_trace": ([_P, _I32], C.c_int),
    "lsb_cycle_begin": ([_P, _P], C.c_int),
    "lsb_cycle_lsq": ([_P, _P], C.c_int),
    "lsb_cycle_extract": ([_P, _P, _P, _P], C.c_int),
    "lsb_restart_check": ([_P, _I32, _P], C.c_int),
    "lsb_trial_lsq": ([_P, _I32, _P, _P], C.c_int),
    "lsb_trial_combine": ([_P, _I32, _P, _P, _P, _P, _P], C.c_int),
    "lsb_gram_row": ([_P, _I32, _I32, _I32, _P, _I64, _P], C.c_int),
    "lsb_givens_update": ([_P, _P, _P, _I32, _P, _I32, _P, _P], C.c_int),
    "lsb_back_substitute": ([_P, _P, _I32, _I32, _P, _P, _P], C.c_int),
    "lsb_peer_allgather": ([_P, _P, _I32, _P, _I32, _P, _P], C.c_int),
    "lsb_peer_halo": ([_P, _P, _P, _P, _P, _I64, _P, _P], C.c_int),
    "lsb_ipc_export": ([_P, _P, _P], C.c_int),
    "lsb_ipc_open": ([_P, _P], C.c_int),
    "lsb_ipc_close": ([_P], C.c_int),
    "lsb_preload": ([], C.c_int),
    "lsb_sum_parts": ([_P, _I32, _I32, _I32, _P, _P, _I32, _P], C.c_int),
    "lsb_lagged_update_push": ([_P, _I32, _I32, _I32, _P, _P], C.c_int),
    "lsb_lagged_reduce_spmv7_halo": ([_P, _P, _I32, _I32, _P, _P], C.c_int),
}

EXPORTS = tuple(_SIGS)

_lib = None


def load(path=None):
    """Load (once) and type the library; raises LsbUnavailable if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise LsbUnavailable(
            f"{p} not found: build it with `python -m paper_1809_05805_b200.build` "
            "(there is no CPU fallback)")
    try:
        lib = C.CDLL(p)
    except OSError as e:  # pragma: no cover
        raise LsbUnavailable(f"cannot load {p}: {e}") from e
    for name, (argt, rest) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = argt
        fn.restype = rest
    # LSB_TUNE="key=value,..." (experiments): tuning knobs set at load;
    # malformed or unknown entries are reported and skipped
    for item in filter(None, os.environ.get("LSB_TUNE", "").split(",")):
        key, _, val = item.partition("=")
        try:
            k, v = int(key), int(val)
        except ValueError:
            warnings.warn(f"LSB_TUNE: ignoring malformed entry {item!r}")
            continue
        if lib.lsb_set_tuning(k, v) != 0:
            warnings.warn(f"LSB_TUNE: unknown tuning key {k}")
    if path is None:
        _lib = lib
    return lib


def check(rc, what):
    if rc != OK:
        msg = load().lsb_last_error().decode(errors="replace")
        raise LsbError(f"{what} failed with status {rc}: {msg}")


def call(name, *args):
    rc = getattr(load(), name)(*args)
    if rc != OK:
        check(rc, name)
    return rc
