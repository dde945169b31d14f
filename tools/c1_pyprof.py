"""cProfile of repeated C1 solves (host-side cost of the launch-bound path)."""

import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1809_05805_b200 as P  # noqa: E402

A = P.gen_laplace2d(64)
b = P.gen_rhs("random", A, 42)
cfg = P.GmresConfig(restart_m=30, max_restarts=200, rel_tol=1e-6, method="one_sync_mgs")
for _ in range(3):
    P.solve(A, b, config=cfg, diagnostics_every=0)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    P.solve(A, b, config=cfg, diagnostics_every=0)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(40)
st.sort_stats("tottime").print_stats(25)
