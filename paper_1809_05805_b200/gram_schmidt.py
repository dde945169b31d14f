"""Drop-in orthogonalizers of lowsync.gram_schmidt (reference
gram_schmidt.py), on B200.

Same signatures, mutation contract (lagged kernels update two basis columns
and the FactorState in place and return None; direct kernels return fresh
(q, r_col, r_diag)), ledger events and HappyBreakdown semantics (raised
before the lagged column is normalised).  Each call is a short sequence of
liblsb200 launches; standalone calls synchronise once to surface
HappyBreakdown, the solver engine (engine.py) chains the same kernels
without any synchronisation.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _abi
from . import _dev as D
from .errors import HappyBreakdown
from .kernels import FUSED, KrylovBasis, ReductionLedger, mdot_pair, maxpy, norm2

__all__ = ["FactorState", "HappyBreakdown", "cgs_iterated", "mgs_level1", "cgs2_two_sync",
           "mgs_lvl2", "cgs2_lvl2", "apply_T", "qr_factorize"]

_RESET = None


def _reset_flags(flags):
    global _RESET
    if _RESET is None:
        _RESET = torch.tensor([_abi.NO_STOP, 0, -1, 0, 0, 0, 0, 0], dtype=torch.int32)
    flags.copy_(_RESET, non_blocking=False)


class _Scratch:
    """Per-(state) small device buffers for standalone kernel calls."""

    def __init__(self, cap, dev):
        f = dict(dtype=D.F64, device=dev)
        self.coef = torch.zeros(cap + 2, **f)
        self.coef2 = torch.zeros(cap + 2, **f)
        self.G = torch.zeros(2 * (cap + 2), **f)
        self.scal = torch.zeros(_abi.S_COUNT, **f)
        self.flags = torch.zeros(_abi.FLAGS_INTS, dtype=torch.int32, device=dev)
        self.ws = D.Workspace(max(cap + 2, 8), dev)

    def struct(self, Vptr, ld, n, cap, R=None, T=None, L=None):
        return _abi.Arnoldi(
            V=Vptr, ld=ld, n=n, n_global=n, cap=cap, m=0, R=D.ptr(R).value if R is not None else None,
            T=D.ptr(T).value if T is not None else None, L=D.ptr(L).value if L is not None else None,
            rot=None, g=None, tri=None, coef=self.coef.data_ptr(), coef2=self.coef2.data_ptr(),
            G=self.G.data_ptr(), g_parts=1, g_stride=2 * cap, Gloc=self.G.data_ptr(),
            scal=self.scal.data_ptr(), res=None, flags=self.flags.data_ptr(),
            ws=_abi.Workspace(self.ws.partial.data_ptr(), self.ws.counter.data_ptr(), 0, 0))


class FactorState:
    """R, T (compact-WY) and L (CGS2) factors (gram_schmidt.py:70-93).

    Default: numpy arrays like the reference (tests read and write
    state.R / .T / .L in place; the kernels stage them on the device and
    write them back); ``device="cuda"``: CUDA tensors the kernels update in
    place."""

    def __init__(self, capacity, device=None):
        self.capacity = int(capacity)
        self.host = device is None
        shp = (capacity, capacity)
        if self.host:
            self.R, self.T, self.L = np.zeros(shp), np.zeros(shp), np.zeros(shp)
        else:
            dev = D.require_cuda()
            self.R, self.T, self.L = (torch.zeros(shp, dtype=D.F64, device=dev) for _ in range(3))
        self.active = 0
        self._sc = None

    def reset(self):
        for a in (self.R, self.T, self.L):
            a[...] = 0.0
        self.active = 0

    def scratch(self):
        if self._sc is None:
            self._sc = _Scratch(self.capacity, D.require_cuda())
        return self._sc


def _dev_factors(state):
    """(R, T, L) as device tensors: the state's own, or staged copies."""
    if not state.host:
        return state.R, state.T, state.L
    dev = D.require_cuda()
    return tuple(torch.as_tensor(np.ascontiguousarray(a)).to(dev) for a in (state.R, state.T,
                                                                              state.L))


def _write_back(state, dR, dT, dL):
    if state.host:
        for a, d in ((state.R, dR), (state.T, dT), (state.L, dL)):
            a[...] = d.cpu().numpy()


def _lagged(V, state, j, ledger, krylov_scale, btf, eligible, two):
    """Host-mode basis / factors (the reference's numpy storage) run on
    staged device copies; the two columns and the factors the kernels change
    are written back, so the mutation contract is the reference's."""
    if j > V.n_cols:
        raise ValueError(f"cannot view {j} of {V.n_cols} columns")
    if not (V.host or state.host):
        return _lagged_dev(V, state, j, ledger, krylov_scale, btf, eligible, two,
                           state.R, state.T, state.L)
    Vd = V.device_copy() if V.host else V
    dR, dT, dL = _dev_factors(state)
    try:
        _lagged_dev(Vd, state, j, ledger, krylov_scale, btf, eligible, two, dR, dT, dL)
    finally:
        _write_back(state, dR, dT, dL)
        if V.host:
            p = j - 1
            V.store[:, p - 1:p + 1] = Vd.store[p - 1:p + 1, : V.n].t().cpu().numpy()
            V.lag = Vd.lag


def _lagged_dev(V, state, j, ledger, krylov_scale, btf, eligible, two, Rt, Tt, Lt):
    p = j - 1
    sc = state.scratch()
    S = sc.struct(V.ptr(0), V.ld, V.n, state.capacity, Rt, Tt, Lt)
    ref = C.byref(S)
    st = D.stream()
    _reset_flags(sc.flags)
    sc.scal[_abi.S_BTF] = float(btf)
    ledger.record(FUSED, 2 * p, eligible)
    _abi.call("lsb_lagged_reduce", ref, 0, p, st)
    if not two:
        _abi.call("lsb_mgs_lvl2_small", ref, 0, p, int(bool(krylov_scale)), 0, st)
        _abi.call("lsb_lagged_update", ref, 0, p, int(bool(krylov_scale)), st)
    else:
        _abi.call("lsb_cgs2_lvl2_small_a", ref, 0, p, int(bool(krylov_scale)), 0, st)
    fl = sc.flags.cpu()
    if int(fl[2]) == 0:  # broke_iter: HappyBreakdown before normalising u
        sv = sc.scal.cpu().numpy()
        raise HappyBreakdown(p - 1, float(sv[_abi.S_BETA]), float(sv[_abi.S_TOL]),
                             r_col=Rt[: p - 1, p - 1].cpu().numpy().copy())
    if two:
        from .kernels import MDOT
        ledger.record(MDOT, p, False)
        if p + 1 <= 110:   # K3: w -= Q r and s = Q^T w in one pass over Q
            _abi.call("lsb_lagged_update_reduce", ref, 0, p, int(bool(krylov_scale)), st)
        else:
            _abi.call("lsb_lagged_update", ref, 0, p, int(bool(krylov_scale)), st)
            _abi.call("lsb_mdot", C.c_void_p(V.ptr(0)), V.ld, V.n, p, C.c_void_p(V.ptr(p)), None,
                      D.ptr(sc.G), sc.ws.ref(), None, 0, st)
        _abi.call("lsb_cgs2_lvl2_small_b", ref, 0, p, st)
        _abi.call("lsb_lagged_correct", ref, 0, p, st)
    state.active = p
    V.lag = 1


def mgs_lvl2(V, state, j, ledger, krylov_scale=False, breakdown_tol_factor=1.0,
             overlap_eligible=False):
    """Lagged compact-WY MGS, one reduction per column (gram_schmidt.py:206-245):
    K1 (one pass over Q: [Q^T u, Q^T w]) -> K5 (beta, breakdown, T column,
    c = T^T y) -> K2 (u/beta and w - Q c in one pass)."""
    if j < 2:
        state.active = max(state.active, 0)
        return
    _lagged(V, state, j, ledger, krylov_scale, breakdown_tol_factor, overlap_eligible, False)


def cgs2_lvl2(V, state, j, ledger, krylov_scale=False, breakdown_tol_factor=1.0,
              overlap_eligible=False):
    """Lagged Ruhe-style CGS2, two reductions (gram_schmidt.py:248-280)."""
    if j < 2:
        return
    _lagged(V, state, j, ledger, krylov_scale, breakdown_tol_factor, overlap_eligible, True)


def _columns(Q):
    if isinstance(Q, KrylovBasis):
        return Q.view(Q.n_cols)
    if not isinstance(Q, torch.Tensor):
        Q = np.asarray(Q, dtype=np.float64)
    if Q.ndim != 2:
        raise ValueError("basis must be a 2-d column block")
    return Q


def _work_store(Q, a):
    """(p+1, ld) device store holding Q's columns then the work vector."""
    dev = D.require_cuda()
    Qt = Q if isinstance(Q, torch.Tensor) else torch.as_tensor(Q)
    n, p = Qt.shape
    av = D.to_device_vector(a, n)
    ld = D.round_up(max(n, 2), 32)
    store = torch.zeros((p + 1, ld), dtype=D.F64, device=dev)
    if p:
        store[:p, :n].copy_(Qt.to(dev, D.F64).t())
    store[p, :n].copy_(av)
    return store, n, p, ld


def _direct(Q, a, ledger, btf, passes):
    host = D.is_host(a) and D.is_host(Q if not isinstance(Q, KrylovBasis) else np.zeros(0))
    Q = _columns(Q)
    store, n, p, ld = _work_store(Q, a)
    sc = _Scratch(p + 1, store.device)
    S = sc.struct(store.data_ptr(), ld, n, p + 1)
    ref = C.byref(S)
    st = D.stream()
    _reset_flags(sc.flags)
    sc.scal[_abi.S_BTF] = float(btf)
    from .kernels import DOT, MDOT, NORM
    zp = C.c_void_p(store.data_ptr() + 8 * ld * p)
    if passes == 0:  # level-1 MGS: p fused axpy+dot passes, then the norm pass
        for k in range(p):
            ledger.record(DOT, 1)
        _abi.call("lsb_mgs1_passes", ref, 0, p, p, st)   # one cooperative launch
    else:
        fused_next = False   # Q^T z of this pass already produced by the previous projection
        for ps in range(passes if p else 0):
            ledger.record(MDOT, p)
            if not fused_next:
                _abi.call("lsb_mdot", C.c_void_p(store.data_ptr()), ld, n, p, zp, None,
                          D.ptr(sc.G), sc.ws.ref(), None, 0, st)
            _abi.call("lsb_collect_coef", ref, 0, p, int(ps > 0), st)
            fused_next = ps < passes - 1 and p + 1 <= 110
            if fused_next:   # z -= Q s and the next pass's Q^T z in one read of Q
                _abi.call("lsb_cgs_project_reduce", ref, 0, p, p, st)
            else:
                _abi.call("lsb_cgs_project", ref, 0, p, p, int(ps == passes - 1), st)
        if not p:
            _abi.call("lsb_norm_partial", zp, n, D.ptr(sc.G), sc.ws.ref(), None, 0, st)
    ledger.record(NORM, 1)
    _abi.call("lsb_norm_finish", D.ptr(sc.G), 1, 2, zp, n,
              C.c_void_p(sc.scal.data_ptr() + 8 * _abi.S_BETA), sc.ws.ref(), None, 0, st)
    _abi.call("lsb_direct_small", ref, 0, p, p, st)
    fl = sc.flags.cpu()
    sv = sc.scal.cpu().numpy()
    r_diag = float(sv[_abi.S_BETA])
    r_col = sc.coef[:p].clone()
    if int(fl[2]) == 0:
        raise HappyBreakdown(p, r_diag, float(sv[_abi.S_TOL]), r_col=r_col.cpu().numpy())
    _abi.call("lsb_direct_normalize", ref, 0, p, st)
    q = store[p, :n].clone()
    return D.out_like(q, host), D.out_like(r_col, host), r_diag


def mgs_level1(Q, a, ledger, breakdown_tol_factor=1.0):
    """Level-1 MGS: p single dots + the norm, p + 1 reductions
    (gram_schmidt.py:144-160).  Each pass fuses the previous rank-1 update
    with the next dot (K8), so z is read and written once per pass."""
    return _direct(Q, a, ledger, breakdown_tol_factor, 0)


def cgs_iterated(Q, a, passes, ledger, breakdown_tol_factor=1.0):
    """Classical GS with re-orthogonalisation passes, passes + 1 reductions
    (gram_schmidt.py:118-141)."""
    if passes < 1:
        raise ValueError("passes must be >= 1")
    return _direct(Q, a, ledger, breakdown_tol_factor, passes)


def cgs2_two_sync(Q, state, a, q_prev, ledger, breakdown_tol_factor=1.0):
    """Two-synchronisation CGS2 (gram_schmidt.py:163-192), composed from the
    device primitives (not on the GMRES path)."""
    host = D.is_host(a)
    Qd, _, _ = D.colmajor(_columns(Q))
    n, p = Qd.shape
    work = D.to_device_vector(a, n, copy=True)
    if p == 0:
        r_col = torch.zeros(0, dtype=D.F64, device=work.device)
    else:
        B = mdot_pair(Qd, work, D.to_device_vector(q_prev, n), ledger)
        y, ell = B[:, 0], B[:, 1]
        if p >= 2:
            state.L[p - 1, : p - 1] = ell[: p - 1] if not state.host else ell[: p - 1].cpu().numpy()
        Ls = state.L[:p, :p]
        Ls = Ls if isinstance(Ls, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(Ls))
        Ls = Ls.to(work.device)
        r_col = y - Ls @ y - Ls.T @ y
        work = maxpy(work, Qd, -r_col)
        state.active = p
    r_diag = norm2(work, ledger)
    _check_breakdown(n, r_diag, r_col.cpu().numpy(), breakdown_tol_factor, p)
    return D.out_like(work / r_diag, host), D.out_like(r_col, host), r_diag


def _check_breakdown(n, r_diag, r_col, factor, column):
    """gram_schmidt.py:96-106 (host scalars; used by the composed kernels)."""
    import math
    r_col = np.asarray(r_col.cpu() if isinstance(r_col, torch.Tensor) else r_col)
    eps = float(np.finfo(np.float64).eps)
    pre = math.hypot(r_diag, float(np.linalg.norm(r_col))) if len(r_col) else r_diag
    tol = factor * eps * math.sqrt(n) * pre
    if r_diag <= tol:
        raise HappyBreakdown(column, r_diag, tol, r_col=np.array(r_col, copy=True))


def apply_T(state, y, transpose=False, path="wy"):
    """Projector correction of the active block (gram_schmidt.py:283-299)."""
    from .errors import DimensionError
    k = state.active
    host = D.is_host(y)
    yv = D.to_device_vector(y)
    if yv.shape[0] != k:
        raise DimensionError(f"expected length {k}, got {yv.shape[0]}")
    def blk(M):
        M = M[:k, :k]
        M = M if isinstance(M, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(M))
        return M.to(yv.device)

    if path == "wy":
        T = blk(state.T)
        out = (T.T @ yv) if transpose else (T @ yv)
    elif path == "cgs2":
        L = blk(state.L)
        out = yv - L @ yv - L.T @ yv
    else:
        raise ValueError(f"unknown path {path!r}")
    return D.out_like(out, host)


_QR_METHODS = ("cgs1", "cgs2", "mgs", "cgs2_two_sync", "mgs_wy", "cgs2_wy")


def qr_factorize(M, method="mgs", ledger=None, breakdown_tol_factor=1.0):
    """Column-by-column QR through any kernel (gram_schmidt.py:305-358);
    returns host (Q, R) like the reference."""
    if method not in _QR_METHODS:
        raise ValueError(f"method must be one of {_QR_METHODS}")
    M = np.asarray(M, dtype=np.float64)
    n, k = M.shape
    if ledger is None:
        ledger = ReductionLedger()
    basis = KrylovBasis(n, k)
    state = FactorState(max(k, 1))
    if method in ("mgs_wy", "cgs2_wy"):
        kernel = mgs_lvl2 if method == "mgs_wy" else cgs2_lvl2
        basis.push(M[:, 0])
        basis.lag = 1
        for j in range(2, k + 1):
            basis.push(M[:, j - 1])
            kernel(basis, state, j, ledger, breakdown_tol_factor=breakdown_tol_factor)
        u = basis.column(k - 1)
        r_diag = norm2(u, ledger)
        _check_breakdown(n, r_diag, state.R[: k - 1, k - 1], breakdown_tol_factor, k - 1)
        u /= r_diag
        state.R[k - 1, k - 1] = r_diag
        basis.lag = 0
        return basis.view(k).copy(), state.R[:k, :k].copy()
    R = np.zeros((k, k))
    for jcol in range(k):
        a = M[:, jcol]
        Qv = basis.view(jcol)
        if method == "cgs1":
            q, r_col, r_diag = cgs_iterated(Qv, a, 1, ledger, breakdown_tol_factor)
        elif method == "cgs2":
            q, r_col, r_diag = cgs_iterated(Qv, a, 2, ledger, breakdown_tol_factor)
        elif method == "mgs":
            q, r_col, r_diag = mgs_level1(Qv, a, ledger, breakdown_tol_factor)
        else:
            q_prev = basis.column(jcol - 1) if jcol else np.zeros(n)
            q, r_col, r_diag = cgs2_two_sync(Qv, state, a, q_prev, ledger, breakdown_tol_factor)
        R[:jcol, jcol] = np.asarray(r_col)
        R[jcol, jcol] = r_diag
        basis.push(q)
    return basis.view(k).copy(), R
