"""Exception types of the drop-in surface (same names and bases as lowsync)."""


class DimensionError(ValueError):
    """Operand shapes are incompatible (reference kernels.py:27-28)."""


class NonFiniteError(ArithmeticError):
    """A NaN or Inf appeared where the contract requires finite values
    (reference kernels.py:31-32)."""


class HappyBreakdown(Exception):
    """The projected column vanished (reference gram_schmidt.py:54-67)."""

    def __init__(self, column, norm, tol, r_col=None):
        super().__init__(f"column {column} has residual norm {norm:.3e} <= {tol:.3e}")
        self.column = column
        self.norm = norm
        self.tol = tol
        self.r_col = r_col


class SingularHessenberg(Exception):
    """The rotated triangle has a zero diagonal (reference gmres.py:180-181)."""
