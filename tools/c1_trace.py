"""LSB_TRACE phase timestamps of full C1 solves (2D 64^2, one-sync
GMRES(30), tol 1e-6, 365 iterations): where the end-to-end time goes
between engine setup, prologue, the 13 cycles and the result."""

import os
import sys

os.environ["LSB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1809_05805_b200 as P  # noqa: E402

A = P.gen_laplace2d(64)
b = P.gen_rhs("random", A, 42)
cfg = P.GmresConfig(restart_m=30, max_restarts=200, rel_tol=1e-6, method="one_sync_mgs")
for _ in range(4):
    x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
