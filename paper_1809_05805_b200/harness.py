"""Problem generators (reference harness.py:105-149) plus the 3D problems of
BASELINE.json configs 2-5.  Matrices come back as device-ready operators:
stencil problems as matrix-free StencilMatrix (K6), everything else as
CsrMatrix (K7); both reproduce the reference SpMV bit for bit."""

from __future__ import annotations

import numpy as np

from .kernels import CsrMatrix, spmv
from .operators import StencilMatrix, convdiff27, laplace2d, laplace3d


class MatrixMarketError(ValueError):
    """Malformed or unsupported Matrix Market content (harness.py:37-38)."""


def load_matrix_market(path):
    """Matrix Market coordinate file -> CsrMatrix (device CSR on first use).

    Same acceptance rules as the reference loader (harness.py:41-102): real
    or integer, general or symmetric (expanded), 1-based indices, entry count
    checked, duplicates summed, rows sorted.  The entry block is parsed with
    one vectorised numpy conversion instead of a per-line Python loop, so
    thermal1-class files load in seconds.
    """
    with open(path, "r", encoding="ascii", errors="replace") as fh:
        header = fh.readline()
        body = fh.read()
    tok = header.strip().split()
    if len(tok) != 5 or tok[0].lower() != "%%matrixmarket":
        raise MatrixMarketError(f"malformed header: {header.strip()!r}")
    obj, fmt, fld, sym = (t.lower() for t in tok[1:])
    if obj != "matrix":
        raise MatrixMarketError(f"unsupported object {obj!r}")
    if fmt != "coordinate":
        raise MatrixMarketError(f"only coordinate format is supported, got {fmt!r}")
    if fld in ("complex", "pattern"):
        raise MatrixMarketError(f"{fld} fields are not supported, real data required")
    if fld not in ("real", "integer"):
        raise MatrixMarketError(f"unknown field type {fld!r}")
    if sym not in ("general", "symmetric"):
        raise MatrixMarketError(f"unsupported symmetry {sym!r}")
    lines = [s for s in (ln.strip() for ln in body.splitlines()) if s and not s.startswith("%")]
    if not lines:
        raise MatrixMarketError("missing size line")
    parts = lines[0].split()
    if len(parts) != 3:
        raise MatrixMarketError(f"bad size line: {lines[0]!r}")
    n_rows, n_cols, nnz = (int(p) for p in parts)
    entries = lines[1:]
    if len(entries) != nnz:
        raise MatrixMarketError(f"declared {nnz} entries, found {len(entries)}")
    if nnz:
        flat = " ".join(entries).split()
        if len(flat) != 3 * nnz:
            bad = next(s for s in entries if len(s.split()) != 3)
            raise MatrixMarketError(f"bad entry line: {bad!r}")
        arr = np.array(flat, dtype=np.float64).reshape(nnz, 3)
        i = arr[:, 0].astype(np.int64) - 1
        j = arr[:, 1].astype(np.int64) - 1
        v = arr[:, 2]
    else:
        i = j = np.zeros(0, dtype=np.int64)
        v = np.zeros(0)
    out = (i < 0) | (i >= n_rows) | (j < 0) | (j >= n_cols)
    if np.any(out):
        k = int(np.argmax(out))
        raise MatrixMarketError(f"entry ({i[k] + 1}, {j[k] + 1}) out of range")
    if sym == "symmetric":
        off = i != j
        # interleave each off-diagonal mirror right after its entry, as the
        # reference appends them, so duplicate sums keep the same order
        order = np.argsort(np.concatenate([2 * np.arange(nnz), 2 * np.nonzero(off)[0] + 1]),
                           kind="stable")
        i, j = np.concatenate([i, j[off]])[order], np.concatenate([j, i[off]])[order]
        v = np.concatenate([v, v[off]])[order]
    return CsrMatrix.from_coo(n_rows, n_cols, i, j, v)


def gen_simoncini(n=100, first=1e-8):
    """diag(first, 2, ..., n) (harness.py:105-116)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    d = np.arange(1, n + 1, dtype=np.float64)
    d[0] = first
    return CsrMatrix.diagonal(d)


def gen_laplace2d(nx=10):
    """5-point Dirichlet Laplacian on nx x nx (harness.py:119-136), matrix-free."""
    if nx < 1:
        raise ValueError("nx must be >= 1")
    return laplace2d(nx)


def gen_laplace3d(N=32, dims=None):
    """7-point Dirichlet Laplacian on N^3 (configs 2 and 4)."""
    return laplace3d(N, dims)


def gen_convdiff27(N=16, pe=0.5, dims=None):
    """27-point convection-diffusion on N^3 (config 5)."""
    return convdiff27(N, pe, dims)


def gen_rhs(kind, A, seed=None):
    """Unit-norm seeded Gaussian or the image of all-ones (harness.py:139-149);
    host numpy, like the reference."""
    if kind == "ones_image":
        return spmv(A, np.ones(A.n_cols))
    if kind == "random":
        if seed is None:
            raise ValueError("random rhs requires a seed")
        b = np.random.default_rng(seed).standard_normal(A.n_rows)
        return b / np.linalg.norm(b)
    raise ValueError(f"unknown rhs kind {kind!r}")


__all__ = ["gen_simoncini", "gen_laplace2d", "gen_laplace3d", "gen_convdiff27", "gen_rhs",
           "StencilMatrix", "MatrixMarketError", "load_matrix_market"]
