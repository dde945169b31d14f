"""Host latency of small solves through the drop-in API (the reference's
acceptance criterion 1 runs six GMRES(36) solves of a 36-unknown problem,
diagnostics on, within one second).  Prints per-solver wall times, cold
and warm, and the top of a cProfile of the cold pass."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_05805_b200 as P  # noqa: E402

P._dev.require_cuda()
A = P.gen_laplace2d(6)
b = P.gen_rhs("random", A, 42)
cfg = P.GmresConfig(restart_m=36, max_restarts=1, rel_tol=1e-12)
SOLVERS = {"mgs_l1": P.gmres_mgs_l1, "cgs2": P.gmres_cgs2, "two_sync": P.gmres_two_sync,
           "one_sync": P.gmres_one_sync, "pipeline2": P.gmres_pipeline2,
           "cgs1_ghysels": P.gmres_cgs1_ghysels}


def once(tag):
    t0 = time.perf_counter()
    for name, fn in SOLVERS.items():
        t = time.perf_counter()
        fn(A, b, config=cfg, ledger=P.ReductionLedger())
        print(f"{tag} {name}: {1e3 * (time.perf_counter() - t):.1f} ms")
    print(f"{tag} total {1e3 * (time.perf_counter() - t0):.1f} ms")


pr = cProfile.Profile()
pr.enable()
once("cold")
pr.disable()
once("warm")
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
