"""Config 2 to convergence: 256^3 7-point, GMRES(50), tol 1e-6, through the
drop-in solve() with host b and host x (the reference needs 1,749
iterations / 35 cycles, 65 min on one host core -- tests/golden).  Reports
iterations, wall time and Arnoldi it/s for the lagged methods.

    python tools/c2_converge.py [--methods one_sync_mgs,two_sync_cgs2,pipeline2]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--methods", default="one_sync_mgs,pipeline2,two_sync_cgs2")
    ap.add_argument("--N", type=int, default=256)
    a = ap.parse_args()
    A = P.gen_laplace3d(a.N)
    b = P.gen_rhs("random", A, 42)
    out = {}
    for meth in a.methods.split(","):
        cfg = P.GmresConfig(restart_m=50, max_restarts=100, rel_tol=1e-6, method=meth)
        x, h = P.solve(A, b, config=cfg, diagnostics_every=0)      # warm (allocations)
        h.release()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
        dt = time.perf_counter() - t0
        out[meth] = {"iterations": h.iterations, "cycles": len(h.cycle_starts),
                     "outcome": h.outcome, "final_true_rel_res": h.final_true_rel_res,
                     "seconds": round(dt, 3), "it_s": round(h.iterations / dt, 1)}
        print(meth, out[meth], flush=True)
        h.release()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
