"""Drop-in primitives of lowsync.kernels (reference kernels.py), on B200.

Same names, signatures, ledger semantics and error types as the reference.
Arithmetic runs in liblsb200 (sm_100a); numpy inputs are uploaded and the
results handed back as numpy, CUDA tensors stay on the device.

Reductions record exactly one ledger event (kind, scalar_count,
overlap_eligible) per call, as kernels.py:59-95 specifies -- the ledger is
host bookkeeping and costs nothing on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from . import _dev as D
from .errors import DimensionError, NonFiniteError

EPS = float(np.finfo(np.float64).eps)

MDOT = "mdot"
NORM = "norm"
FUSED = "fused_mdot_norm"
DOT = "dot"
_KINDS = (MDOT, NORM, FUSED, DOT)


def as_vector(x, n=None):
    """Device float64 vector, optionally length-checked (kernels.py:35-42)."""
    return D.to_device_vector(x, n)


def require_finite(v, label="vector"):
    t = v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v, dtype=np.float64))
    if not bool(torch.isfinite(t).all()):
        raise NonFiniteError(f"{label} contains NaN or Inf")
    return v


# ---------------------------------------------------------------- ledger
@dataclass
class ReductionEvent:
    iteration: int
    kind: str
    scalar_count: int
    overlap_eligible: bool = False


class ReductionLedger:
    """Append-only log of global-reduction events (kernels.py:59-95)."""

    def __init__(self):
        self.events: list[ReductionEvent] = []
        self.iteration = 0

    def record(self, kind, scalar_count, overlap_eligible=False):
        if kind not in _KINDS:
            raise ValueError(f"unknown reduction kind {kind!r}")
        self.events.append(ReductionEvent(self.iteration, kind, int(scalar_count),
                                          bool(overlap_eligible)))

    def __len__(self):
        return len(self.events)

    def events_in_iteration(self, iteration):
        return [e for e in self.events if e.iteration == iteration]

    def counts_per_iteration(self):
        out: dict[int, int] = {}
        for e in self.events:
            out[e.iteration] = out.get(e.iteration, 0) + 1
        return out

    def counts_by_kind(self):
        out = {k: 0 for k in _KINDS}
        for e in self.events:
            out[e.kind] += 1
        return out


# ---------------------------------------------------------------- matrices
class CsrMatrix:
    """Host CSR (int64 indices, float64 values; kernels.py:98-203) with a
    lazily uploaded device copy (int32 indices) used by the K7 kernel."""

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self._dev = None
        self.validate()

    def validate(self):
        nnz = self.values.shape[0]
        rp, ci = self.row_ptr, self.col_idx
        if rp.shape[0] != self.n_rows + 1:
            raise ValueError("row_ptr must have length n_rows + 1")
        if ci.shape[0] != nnz:
            raise ValueError("col_idx and values must have equal length")
        if rp[0] != 0 or rp[-1] != nnz:
            raise ValueError("row_ptr must start at 0 and end at nnz")
        if np.any(np.diff(rp) < 0):
            raise ValueError("row_ptr must be non-decreasing")
        if nnz and (ci.min() < 0 or ci.max() >= self.n_cols):
            raise ValueError("column index out of range")
        if nnz > 1:
            same_row = np.ones(nnz - 1, dtype=bool)
            starts = rp[1:-1]
            starts = starts[(starts > 0) & (starts < nnz)]
            same_row[starts - 1] = False
            bad = (np.diff(ci) <= 0) & same_row
            if np.any(bad):
                k = int(np.argmax(bad))
                row = int(np.searchsorted(rp, k, side="right") - 1)
                raise ValueError(f"column indices not strictly increasing in row {row}")

    @property
    def nnz(self):
        return self.values.shape[0]

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    @classmethod
    def from_dense(cls, M, drop_tol=0.0):
        M = np.asarray(M, dtype=np.float64)
        if M.ndim != 2:
            raise ValueError("from_dense needs a 2-d array")
        r, c = np.nonzero(np.abs(M) > drop_tol)
        ptr = np.zeros(M.shape[0] + 1, dtype=np.int64)
        np.cumsum(np.bincount(r, minlength=M.shape[0]), out=ptr[1:])
        return cls(M.shape[0], M.shape[1], ptr, c, M[r, c])

    @classmethod
    def from_coo(cls, n_rows, n_cols, rows, cols, vals):
        """Duplicates summed, rows sorted (kernels.py:159-177)."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        if rows.size:
            head = np.empty(rows.size, dtype=bool)
            head[0] = True
            head[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
            grp = np.cumsum(head) - 1
            summed = np.zeros(int(grp[-1]) + 1)
            np.add.at(summed, grp, vals)
            rows, cols, vals = rows[head], cols[head], summed
        ptr = np.zeros(n_rows + 1, dtype=np.int64)
        if rows.size:
            np.cumsum(np.bincount(rows, minlength=n_rows), out=ptr[1:])
        return cls(n_rows, n_cols, ptr, cols, vals)

    @classmethod
    def diagonal(cls, diag):
        diag = np.asarray(diag, dtype=np.float64)
        n = diag.shape[0]
        return cls(n, n, np.arange(n + 1), np.arange(n), diag.copy())

    def diagonal_values(self):
        d = np.zeros(min(self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        hit = (rows == self.col_idx) & (rows < d.shape[0])
        d[rows[hit]] = self.values[hit]
        return d

    def frobenius_norm(self):
        return float(np.sqrt(np.dot(self.values, self.values)))

    def to_dense(self):
        M = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        M[rows, self.col_idx] = self.values
        return M

    # -- device side
    def device_op(self):
        if self._dev is None:
            from .operators import CsrOperator
            self._dev = CsrOperator(self)
        return self._dev


class KrylovBasis:
    """Column store of the Krylov basis (kernels.py:206-253).

    Two storage modes:
      * default (``device=None``): the reference's own storage -- a
        Fortran-order numpy array; ``view`` / ``column`` / ``columns`` alias
        it (the reference tests mutate columns through them,
        test_gram_schmidt.py:375-383).  The lagged kernels stage it into a
        device copy, run there and write the columns they change back
        (gram_schmidt._lagged): reference semantics at the API level.
      * ``device="cuda"``: HBM, (capacity, ld) with column j contiguous at
        ptr(j) = base + 8*ld*j, ld a multiple of 32 doubles; views are CUDA
        tensors and the kernels work in place (the solver engine keeps its
        own basis the same way)."""

    def __init__(self, n, capacity, ld=None, device=None):
        if capacity < 1:
            raise ValueError("capacity must be at least 1")
        self.n = int(n)
        self.capacity = int(capacity)
        self.host = device is None
        self.n_cols = 0
        self.lag = 0
        if self.host:
            self.ld = self.n
            self.store = np.zeros((self.n, self.capacity), order="F")
            return
        dev = D.require_cuda()
        self.ld = int(ld) if ld else D.round_up(max(self.n, 2), 32)
        self.store = torch.zeros((self.capacity, self.ld), dtype=D.F64,
                                 device=dev if device in (True, "cuda") else device)

    @property
    def columns(self):
        if self.host:
            return self.store
        return self.store[:, : self.n].t()

    def ptr(self, j=0):
        if self.host:
            raise TypeError("host-mode KrylovBasis has no device pointer (see device_copy)")
        return self.store.data_ptr() + 8 * self.ld * j

    def device_copy(self):
        """Device-mode copy of a host-mode basis (same columns and lag)."""
        V = KrylovBasis(self.n, self.capacity, device="cuda")
        if self.n_cols:
            V.store[: self.n_cols, : self.n].copy_(torch.from_numpy(
                np.ascontiguousarray(self.store[:, : self.n_cols].T)))
        V.n_cols, V.lag = self.n_cols, self.lag
        return V

    def push(self, vec):
        if self.n_cols >= self.capacity:
            raise ValueError("basis is at capacity")
        if self.host:
            v = vec.detach().cpu().numpy() if isinstance(vec, torch.Tensor) else np.asarray(
                vec, dtype=np.float64)
            if v.ndim != 1 or v.shape[0] != self.n:
                raise DimensionError(f"expected length {self.n}, got {tuple(v.shape)}")
            self.store[:, self.n_cols] = v
        else:
            v = vec if isinstance(vec, torch.Tensor) else torch.as_tensor(
                np.asarray(vec, dtype=np.float64))
            if v.dim() != 1 or v.shape[0] != self.n:
                raise DimensionError(f"expected length {self.n}, got {tuple(v.shape)}")
            self.store[self.n_cols, : self.n].copy_(v)
        self.n_cols += 1
        return self.n_cols - 1

    def view(self, p):
        if p < 0 or p > self.n_cols:
            raise ValueError(f"cannot view {p} of {self.n_cols} columns")
        if self.host:
            return self.store[:, :p]
        return self.store[:p, : self.n].t()

    def column(self, j):
        if j < 0 or j >= self.n_cols:
            raise IndexError(f"column {j} of {self.n_cols}")
        if self.host:
            return self.store[:, j]
        return self.store[j, : self.n]

    def reset(self):
        self.n_cols = 0
        self.lag = 0

    def check_normalized(self):
        """Columns up to n_cols - lag have unit norm within 4 eps sqrt(n)
        (kernels.py:246-253); the norms come from the device norm kernel."""
        tol = 4.0 * EPS * np.sqrt(self.n)
        k = self.n_cols - self.lag
        for j in range(max(k, 0)):
            nrm = float(_device_norm(D.to_device_vector(self.column(j))).item())
            if abs(nrm - 1.0) > tol:
                raise ValueError(f"column {j} has norm {nrm!r}, outside unit tolerance")
        return True


# ---------------------------------------------------------------- primitives
def spmv(A, x):
    """y = A x, bitwise equal to the reference row sums (kernels.py:256-272)."""
    host = D.is_host(x)
    op = A if hasattr(A, "apply") else A.device_op()
    xv = D.to_device_vector(x, op.n_cols)
    y = torch.empty(op.n_rows, dtype=D.F64, device=xv.device)
    flags = torch.zeros(_abi.FLAGS_INTS, dtype=torch.int32, device=xv.device)
    op.apply(xv, y, flags=flags)
    if int(flags[4].item()):
        raise NonFiniteError("spmv result contains NaN or Inf")
    return D.out_like(y, host)


def _reduce_ptrs(X):
    Xv, xp, ld = D.colmajor(X)
    return Xv, xp, ld


def mass_inner_product(X, y, ledger, overlap_eligible=False):
    """X^T y, one 'mdot' event; p == 0 is a silent no-op (kernels.py:301-312)."""
    host = D.is_host(X)
    Xv, xp, ld = _reduce_ptrs(X)
    n, p = Xv.shape
    if p == 0:
        return np.zeros(0) if host else torch.zeros(0, dtype=D.F64, device=Xv.device)
    yv = D.to_device_vector(y, n)
    ledger.record(MDOT, p, overlap_eligible)
    out = torch.empty(p, dtype=D.F64, device=Xv.device)
    ws = D.default_workspace()
    _abi.call("lsb_mdot", xp, ld, n, p, D.ptr(yv), None, D.ptr(out), ws.ref(), None, 0, D.stream())
    return D.out_like(out, host)


def fused_mdot_norm(X, y, z, ledger, overlap_eligible=False):
    """(X^T y, ||z||) in one 'fused_mdot_norm' event of p+1 scalars
    (kernels.py:315-325); both partial sets travel in one device pass each."""
    host = D.is_host(X)
    Xv, xp, ld = _reduce_ptrs(X)
    n, p = Xv.shape
    yv = D.to_device_vector(y, n)
    zv = D.to_device_vector(z, n)
    ledger.record(FUSED, p + 1, overlap_eligible)
    ws = D.default_workspace()
    out = torch.empty(p, dtype=D.F64, device=yv.device)
    if p:
        _abi.call("lsb_mdot", xp, ld, n, p, D.ptr(yv), None, D.ptr(out), ws.ref(), None, 0,
                  D.stream())
    nrm = _device_norm(zv, ws)
    return D.out_like(out, host), float(nrm.item())


def mdot_pair(X, u, w, ledger, kind=MDOT, overlap_eligible=False):
    """[X^T u, X^T w] as (p, 2) with one event of 2p scalars, X read once
    (kernels.py:328-347)."""
    host = D.is_host(X)
    Xv, xp, ld = _reduce_ptrs(X)
    n, p = Xv.shape
    if p == 0:
        return np.zeros((0, 2)) if host else torch.zeros((0, 2), dtype=D.F64, device=Xv.device)
    uv = D.to_device_vector(u, n)
    wv = D.to_device_vector(w, n)
    ledger.record(kind, 2 * p, overlap_eligible)
    out = torch.empty((p, 2), dtype=D.F64, device=uv.device)
    ws = D.default_workspace()
    _abi.call("lsb_mdot", xp, ld, n, p, D.ptr(uv), D.ptr(wv), D.ptr(out), ws.ref(), None, 0,
              D.stream())
    return D.out_like(out, host)


def maxpy(y, X, alpha):
    """y + X alpha as a new array, reduction-free (kernels.py:350-362)."""
    host = D.is_host(y)
    Xv, xp, ld = _reduce_ptrs(X)
    n, p = Xv.shape
    yv = D.to_device_vector(y, n if p else None)
    if p == 0:
        return D.out_like(yv.clone(), host)
    av = D.to_device_vector(alpha, p)
    out = torch.empty(n, dtype=D.F64, device=yv.device)
    _abi.call("lsb_maxpy", D.ptr(yv), xp, ld, n, p, D.ptr(av), 1, D.ptr(out), None, 0, D.stream())
    return D.out_like(out, host)


def _device_norm(v, ws=None):
    """||v||_2 into a device scalar (overflow-safe, deterministic)."""
    ws = ws or D.default_workspace()
    parts = torch.empty(2, dtype=D.F64, device=v.device)
    out = torch.empty(1, dtype=D.F64, device=v.device)
    n = v.shape[0]
    _abi.call("lsb_norm_partial", D.ptr(v), n, D.ptr(parts), ws.ref(), None, 0, D.stream())
    _abi.call("lsb_norm_finish", D.ptr(parts), 1, 2, D.ptr(v), n, D.ptr(out), ws.ref(), None, 0,
              D.stream())
    return out


def dot(x, y, ledger):
    """Single inner product, one 'dot' event (kernels.py:275-280)."""
    xv = D.to_device_vector(x)
    yv = D.to_device_vector(y, xv.shape[0])
    ledger.record(DOT, 1)
    out = torch.empty(1, dtype=D.F64, device=xv.device)
    ws = D.default_workspace()
    n = xv.shape[0]
    if n == 0:
        return 0.0
    _abi.call("lsb_mdot", D.ptr(xv), D.round_up(max(n, 2), 2), n, 1, D.ptr(yv), None, D.ptr(out),
              ws.ref(), None, 0, D.stream())
    return float(out.item())


def norm2(x, ledger, overlap_eligible=False):
    """Euclidean norm, overflow-safe, one 'norm' event (kernels.py:283-289)."""
    xv = D.to_device_vector(x)
    if bool(torch.isnan(xv).any()):
        raise NonFiniteError("norm2 input contains NaN")
    ledger.record(NORM, 1, overlap_eligible)
    if xv.shape[0] == 0:
        return 0.0
    return float(_device_norm(xv).item())
