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

# untraced wall time (the trace synchronises at every mark, which hides the
# overlap of the host's report replay with the device's later cycles)
import time  # noqa: E402

import torch  # noqa: E402

os.environ.pop("LSB_TRACE")
for meth in ("one_sync_mgs", "pipeline2"):
    cfg = P.GmresConfig(restart_m=30, max_restarts=200, rel_tol=1e-6, method=meth)
    for _ in range(3):
        P.solve(A, b, config=cfg, diagnostics_every=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 50
    for _ in range(reps):
        x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
    dt = (time.perf_counter() - t0) / reps
    print(f"{meth}: solve() wall {1e3 * dt:.2f} ms per solve, {h.iterations} iterations, "
          f"{h.iterations / dt:.0f} it/s")
