"""Device operators that feed the Arnoldi loop: K7 CSR and K6 box stencils.

Both reproduce the reference SpMV (kernels.py:256-272) bit for bit.  The
stencil operators are matrix-free (16 B/row of compulsory HBM traffic) and
duck-type the reference CsrMatrix (n_rows, n_cols, nnz, row_ptr, col_idx,
values, to_dense, diagonal_values, frobenius_norm), materialising the CSR
arrays only if a caller asks for them.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _abi
from . import _dev as D


class CsrOperator:
    """Device copy of a CsrMatrix with 32-bit indices."""

    def __init__(self, A, col_scale=None):
        dev = D.require_cuda()
        if A.nnz >= 2 ** 31 or A.n_rows >= 2 ** 31:
            raise ValueError("CSR kernel supports nnz < 2^31")
        self.n_rows, self.n_cols = A.n_rows, A.n_cols
        self.row_ptr = torch.as_tensor(A.row_ptr.astype(np.int32), device=dev)
        self.col_idx = torch.as_tensor(A.col_idx.astype(np.int32), device=dev)
        self.values = torch.as_tensor(A.values, device=dev)
        self.col_scale = col_scale
        self.halo = 0
        self.c = _abi.Csr(A.n_rows, A.n_cols, A.nnz, self.row_ptr.data_ptr(),
                          self.col_idx.data_ptr(), self.values.data_ptr(),
                          col_scale.data_ptr() if col_scale is not None else None, 0, 0)
        self._dictionary()

    @classmethod
    def row_block(cls, row_ptr, col_idx, values, row0, halo):
        """Rows [row0, row0 + n) of a global CSR matrix (row_ptr rebased to
        0, GLOBAL column indices): x is the owned rows with `halo` ghost rows
        on either side, the kernel indexes it by (col - row0), so ghost
        columns land in the padding the halo exchange fills."""
        from types import SimpleNamespace
        n = len(row_ptr) - 1
        A = SimpleNamespace(n_rows=n, n_cols=n, nnz=int(len(values)), row_ptr=np.asarray(row_ptr),
                            col_idx=np.asarray(col_idx), values=np.asarray(values, np.float64))
        op = object.__new__(cls)
        dev = D.require_cuda()
        op.n_rows = op.n_cols = n
        op.row_ptr = torch.as_tensor(A.row_ptr.astype(np.int32), device=dev)
        op.col_idx = torch.as_tensor(A.col_idx.astype(np.int32), device=dev)
        op.values = torch.as_tensor(A.values, device=dev)
        op.col_scale = None
        op.halo = int(halo)
        op.row0 = int(row0)
        op._diag = None
        rows = np.repeat(np.arange(n), np.diff(A.row_ptr)) + row0
        hit = A.col_idx == rows
        d = np.zeros(n)
        d[rows[hit] - row0] = A.values[hit]
        op._diag = d
        op.c = _abi.Csr(n, n, A.nnz, op.row_ptr.data_ptr(), op.col_idx.data_ptr(),
                        op.values.data_ptr(), None, int(row0), int(row0))
        op._dictionary()
        return op

    def diagonal_values(self):
        d = getattr(self, "_diag", None)
        if d is None:
            raise AttributeError("diagonal_values of a device-only CSR operator")
        return d

    # nnz from which the dictionary form pays for its one-time build
    DICT_MIN_NNZ = 1 << 20

    def _dictionary(self):
        """Dictionary-coded copy (lsb_csr_dict) when the values have at most
        256 distinct bit patterns and the column offsets col - row at most 256
        distinct values: the SpMV then streams 2 bytes per nonzero instead of
        12, bitwise the same y.  LSB_CSR_DICT=0 never, =1 always (any size)."""
        self.cd = None
        mode = os.environ.get("LSB_CSR_DICT", "auto")
        nnz = int(self.values.shape[0])
        if mode == "0" or nnz == 0 or (mode != "1" and nnz < self.DICT_MIN_NNZ):
            return
        try:
            self._build_dictionary()
        except torch.cuda.OutOfMemoryError:   # the build's sort temporaries: keep plain CSR
            self.cd = None
            torch.cuda.empty_cache()

    def _build_dictionary(self):
        bits = self.values.view(torch.int64)          # exact: -0.0, NaN payloads kept
        vt, vi = torch.unique(bits, return_inverse=True)
        if vt.numel() > 256:
            return
        counts = self.row_ptr[1:].to(torch.int64) - self.row_ptr[:-1].to(torch.int64)
        rows = torch.repeat_interleave(torch.arange(self.n_rows, device=bits.device), counts)
        rows += int(self.c.row0)          # row-block partition: offsets from global rows
        ot, oi = torch.unique(self.col_idx.to(torch.int64) - rows, return_inverse=True)
        del rows
        if ot.numel() > 256 or ot.abs().max() >= 2 ** 31:
            return
        # padded to whole 32-bit words (+1): the warp-staged kernel copies
        # the index bytes of a 32-row segment with word loads
        pad = (-vi.numel()) % 4 + 4
        self.cd_val_idx = torch.nn.functional.pad(vi.to(torch.uint8), (0, pad))
        self.cd_off_idx = torch.nn.functional.pad(oi.to(torch.uint8), (0, pad))
        self.cd_val_tab = vt.view(torch.float64).contiguous()
        self.cd_off_tab = ot.to(torch.int32)
        self.cd = self._dict_struct(self.col_scale)

    def _dict_struct(self, col_scale):
        return _abi.CsrDict(self.c.n_rows, self.c.n_cols, self.c.nnz, self.row_ptr.data_ptr(),
                            self.cd_val_idx.data_ptr(), self.cd_off_idx.data_ptr(),
                            self.cd_val_tab.data_ptr(), self.cd_off_tab.data_ptr(),
                            int(self.cd_val_tab.numel()), int(self.cd_off_tab.numel()),
                            col_scale.data_ptr() if col_scale is not None else None,
                            self.c.row0, self.c.x_lo)

    @classmethod
    def from_device(cls, n_rows, n_cols, row_ptr, col_idx, values, col_scale=None):
        """Wrap CSR arrays already resident on the device (int32 row_ptr and
        col_idx, float64 values), e.g. a stencil's CSR built on the GPU
        (StencilMatrix.device_csr) for matrices too large to stage via numpy."""
        op = object.__new__(cls)
        op.n_rows, op.n_cols = int(n_rows), int(n_cols)
        op.row_ptr, op.col_idx, op.values = row_ptr, col_idx, values
        op.col_scale = col_scale
        op.halo = 0
        op.c = _abi.Csr(op.n_rows, op.n_cols, int(values.shape[0]), row_ptr.data_ptr(),
                        col_idx.data_ptr(), values.data_ptr(),
                        col_scale.data_ptr() if col_scale is not None else None, 0, 0)
        op._dictionary()
        return op

    def with_scale(self, col_scale):
        op = object.__new__(CsrOperator)
        op.__dict__.update(self.__dict__)
        op.col_scale = col_scale
        op.c = _abi.Csr(self.c.n_rows, self.c.n_cols, self.c.nnz, self.c.row_ptr, self.c.col_idx,
                        self.c.values, col_scale.data_ptr() if col_scale is not None else None,
                        self.c.row0, self.c.x_lo)
        if self.cd is not None:
            op.cd = self._dict_struct(col_scale)
        return op

    @property
    def h2d_bytes(self):
        return 4 * (self.n_rows + 1) + 12 * int(self.values.shape[0])

    def apply_ptr(self, xp, yp, bp=None, flagsp=None, it=-1, stream=None):
        if self.cd is not None:
            _abi.call("lsb_spmv_csr_dict", C.byref(self.cd), xp, bp, yp, flagsp, it,
                      stream or D.stream())
            return
        _abi.call("lsb_spmv_csr", C.byref(self.c), xp, bp, yp, flagsp, it, stream or D.stream())

    def apply(self, x, y, b=None, flags=None, it=-1):
        self.apply_ptr(D.ptr(x), D.ptr(y), D.ptr(b), D.ptr(flags), it)


def _offsets_7():
    offs = [((0, 0, 0), 6.0)]
    for ax in range(3):
        for s in (-1, 1):
            d = [0, 0, 0]
            d[ax] = s
            offs.append((tuple(d), -1.0))
    return offs


def _offsets_5():
    return [((0, 0, 0), 4.0), ((-1, 0, 0), -1.0), ((1, 0, 0), -1.0), ((0, -1, 0), -1.0),
            ((0, 1, 0), -1.0)]


def convdiff27_offsets(pe=0.5):
    """27-point convection-diffusion: centre 26,
    every neighbour -1, face neighbours also carry central convection
    pe*(dx+dy+dz), i.e. -1+pe downstream and -1-pe upstream."""
    offs = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                if dx == dy == dz == 0:
                    offs.append(((0, 0, 0), 26.0))
                elif abs(dx) + abs(dy) + abs(dz) == 1:
                    offs.append(((dx, dy, dz), -1.0 + pe * (dx + dy + dz)))
                else:
                    offs.append(((dx, dy, dz), -1.0))
    return offs


class StencilMatrix:
    """Constant-coefficient Dirichlet stencil on an nx x ny x nz box,
    row i = (iz*ny + iy)*nx + ix; the CSR it stands for has each row's
    columns in increasing order, exactly what CsrMatrix.from_coo builds
    from the same triples (so gen_laplace2d's matrix is reproduced)."""

    def __init__(self, dims, offsets, name="stencil"):
        self.dims = tuple(int(d) for d in dims)
        nx, ny, nz = self.dims
        self.name = name
        key = lambda o: (o[0][2] * ny + o[0][1]) * nx + o[0][0]  # noqa: E731
        self.offsets = sorted(offsets, key=key)
        self.n_rows = self.n_cols = nx * ny * nz
        self._csr = None
        self._dev = None
        self._dev_csr = None

    # -- CsrMatrix duck typing (materialised lazily, host only)
    def _materialise(self):
        if self._csr is None:
            from .kernels import CsrMatrix
            nx, ny, nz = self.dims
            ix = np.arange(nx); iy = np.arange(ny); iz = np.arange(nz)
            pres, lins, vals = [], [], []
            for (dx, dy, dz), v in self.offsets:
                mx = (ix + dx >= 0) & (ix + dx < nx)
                my = (iy + dy >= 0) & (iy + dy < ny)
                mz = (iz + dz >= 0) & (iz + dz < nz)
                pres.append((mz[:, None, None] & my[None, :, None] & mx[None, None, :]).ravel())
                lins.append((dz * ny + dy) * nx + dx)
                vals.append(v)
            P = np.stack(pres, axis=1)
            ptr = np.zeros(self.n_rows + 1, dtype=np.int64)
            np.cumsum(P.sum(axis=1), out=ptr[1:])
            cols = (np.arange(self.n_rows, dtype=np.int64)[:, None] + np.array(lins)[None, :])[P]
            v = np.broadcast_to(np.array(vals, dtype=np.float64)[None, :], P.shape)[P]
            self._csr = CsrMatrix(self.n_rows, self.n_cols, ptr, cols, v)
        return self._csr

    @property
    def nnz(self):
        nx, ny, nz = self.dims
        tot = 0
        for (dx, dy, dz), _ in self.offsets:
            tot += (nx - abs(dx)) * (ny - abs(dy)) * (nz - abs(dz))
        return tot

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    @property
    def row_ptr(self):
        return self._materialise().row_ptr

    @property
    def col_idx(self):
        return self._materialise().col_idx

    @property
    def values(self):
        return self._materialise().values

    def to_csr(self):
        return self._materialise()

    def to_dense(self):
        return self._materialise().to_dense()

    def diagonal_values(self):
        c = [v for (o, v) in self.offsets if o == (0, 0, 0)]
        return np.full(self.n_rows, c[0] if c else 0.0)

    def frobenius_norm(self):
        nx, ny, nz = self.dims
        s = 0.0
        for (dx, dy, dz), v in self.offsets:
            s += (nx - abs(dx)) * (ny - abs(dy)) * (nz - abs(dz)) * v * v
        return float(np.sqrt(s))

    def device_csr(self):
        """The same CSR as _materialise(), built directly in device memory
        (int32 indices) and wrapped as a K7 CsrOperator: the CSR form of
        configs 2/5 at N=256 (450M nonzeros for the 27-point operator).
        Built once per matrix and cached."""
        if self._dev_csr is not None:
            return self._dev_csr
        dev = D.require_cuda()
        nx, ny, nz = self.dims
        n = self.n_rows
        if n + max(abs((o[2] * ny + o[1]) * nx + o[0]) for o, _ in self.offsets) >= 2 ** 31 \
                or self.nnz >= 2 ** 31:
            raise ValueError("device CSR needs 32-bit indices")
        ix = torch.arange(nx, device=dev)
        iy = torch.arange(ny, device=dev)
        iz = torch.arange(nz, device=dev)
        cnt = torch.zeros(n, dtype=torch.int32, device=dev)
        masks = []
        for (dx, dy, dz), _ in self.offsets:
            mx = (ix + dx >= 0) & (ix + dx < nx)
            my = (iy + dy >= 0) & (iy + dy < ny)
            mz = (iz + dz >= 0) & (iz + dz < nz)
            m = (mz[:, None, None] & my[None, :, None] & mx[None, None, :]).reshape(-1)
            masks.append(m)
            cnt += m.to(torch.int32)
        row_ptr = torch.zeros(n + 1, dtype=torch.int32, device=dev)
        torch.cumsum(cnt, 0, out=row_ptr[1:])
        del cnt
        nnz = int(row_ptr[-1])
        col_idx = torch.empty(nnz, dtype=torch.int32, device=dev)
        values = torch.empty(nnz, dtype=D.F64, device=dev)
        rows = torch.arange(n, dtype=torch.int32, device=dev)
        fill = row_ptr[:-1].clone()          # next free slot of every row
        for ((dx, dy, dz), v), m in zip(self.offsets, masks):   # column order
            r = rows[m]
            pos = fill[m].long()
            col_idx[pos] = r + ((dz * ny + dy) * nx + dx)
            values[pos] = v
            fill[m] += 1
            del r, pos
        self._dev_csr = CsrOperator.from_device(n, n, row_ptr, col_idx, values)
        return self._dev_csr

    def device_op(self):
        if self._dev is None:
            self._dev = StencilOperator(self)
        return self._dev


class StencilOperator:
    """K6 launcher; optional z-slab partition (rows of planes [z0, z0+nzl))
    with ghost planes supplied by the caller next to x."""

    def __init__(self, S, col_scale=None, z0=0, nz_local=None):
        D.require_cuda()
        nx, ny, nz = S.dims
        nzl = nz if nz_local is None else nz_local
        self.stencil = S
        self.n_rows = self.n_cols = nx * ny * nzl
        self.plane = nx * ny
        self.halo_lo = int(z0 > 0)
        self.halo_hi = int(z0 + nzl < nz)
        self.halo = self.plane if (self.halo_lo or self.halo_hi) else 0
        self.col_scale = col_scale
        c = _abi.Stencil()
        c.nx, c.ny, c.nz, c.noff = nx, ny, nzl, len(S.offsets)
        c.halo_lo, c.halo_hi = self.halo_lo, self.halo_hi
        for k, ((dx, dy, dz), v) in enumerate(S.offsets):
            c.dx[k], c.dy[k], c.dz[k], c.val[k] = dx, dy, dz, v
        c.col_scale = col_scale.data_ptr() if col_scale is not None else None
        self.c = c
        self.h2d_bytes = 0

    def diagonal_values(self):
        """This slab's rows of the diagonal (the centre coefficient)."""
        c = [v for (o, v) in self.stencil.offsets if o == (0, 0, 0)]
        return np.full(self.n_rows, c[0] if c else 0.0)

    def with_scale(self, col_scale):
        op = object.__new__(StencilOperator)
        op.__dict__.update(self.__dict__)
        c = _abi.Stencil()
        C.pointer(c)[0] = self.c
        c.col_scale = col_scale.data_ptr() if col_scale is not None else None
        op.c = c
        op.col_scale = col_scale
        return op

    def apply_ptr(self, xp, yp, bp=None, flagsp=None, it=-1, stream=None):
        _abi.call("lsb_spmv_stencil", C.byref(self.c), xp, bp, yp, flagsp, it, stream or D.stream())

    def apply(self, x, y, b=None, flags=None, it=-1):
        self.apply_ptr(D.ptr(x), D.ptr(y), D.ptr(b), D.ptr(flags), it)


def laplace2d(nx):
    """5-point Laplacian (reference harness.py:119-136) as a stencil."""
    return StencilMatrix((nx, nx, 1), _offsets_5(), "laplace2d")


def laplace3d(N, dims=None):
    """7-point Laplacian, the 3D analogue."""
    return StencilMatrix(dims or (N, N, N), _offsets_7(), "laplace3d")


def convdiff27(N, pe=0.5, dims=None):
    """27-point convection-diffusion."""
    return StencilMatrix(dims or (N, N, N), convdiff27_offsets(pe), "convdiff27")


def device_operator(A):
    if hasattr(A, "device_op"):
        return A.device_op()
    if hasattr(A, "apply_ptr"):
        return A
    raise TypeError(f"unsupported operator {type(A).__name__}")
