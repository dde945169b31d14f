"""Launch-bound regime: full C1 (2D 64^2, one-sync GMRES(30), tol 1e-6, 365
iterations) and 3D 32^3 solves through solve(); iterations/s on the device
(graph-replayed cycles) vs the reference's single-thread CPU rate."""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402


def rate(A, m, tol, meth, reps=5):
    b = P.gen_rhs("random", A, 42)
    cfg = P.GmresConfig(restart_m=m, max_restarts=500, rel_tol=tol, method=meth)
    x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
        best = min(best, time.perf_counter() - t0)
    return h.iterations, h.iterations / best, best


for name, A, m, tol in (("C1 laplace2d64", P.gen_laplace2d(64), 30, 1e-6),
                        ("laplace3d32", P.gen_laplace3d(32), 50, 1e-6)):
    for meth in ("one_sync_mgs", "two_sync_cgs2", "mgs_l1", "cgs2"):
        its, r, t = rate(A, m, tol, meth)
        print(f"{name:16s} {meth:14s} {its:5d} it  {1e3 * t:8.2f} ms  {r:10.0f} it/s")
