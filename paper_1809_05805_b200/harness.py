"""Problem generators (reference harness.py:105-149) plus the 3D problems of
BASELINE.json configs 2-5.  Matrices come back as device-ready operators:
stencil problems as matrix-free StencilMatrix (K6), everything else as
CsrMatrix (K7); both reproduce the reference SpMV bit for bit."""

from __future__ import annotations

import numpy as np

from .kernels import CsrMatrix, spmv
from .operators import StencilMatrix, convdiff27, laplace2d, laplace3d


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
           "StencilMatrix"]
