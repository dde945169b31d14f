"""Run the prologue and N one-sync GMRES(50) cycles on 256^3 (config 2) for
ncu captures (launch order per iteration: stencil7 SpMV, mdot K1, small K5,
lagged_update K2).

    python tools/profile_cycle.py [--cycles 1] [--N 256] [--method one_sync_mgs]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=1)
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--method", default="one_sync_mgs")
    ap.add_argument("--graph", action="store_true")
    a = ap.parse_args()
    A = P.gen_laplace3d(a.N)
    b = np.random.default_rng(42).standard_normal(A.n_rows)
    b /= np.linalg.norm(b)
    eng = Engine(A, 50, a.method, 1e-14, use_graph=a.graph)
    eng.load(torch.as_tensor(b).cuda())
    eng.prologue()
    for _ in range(a.cycles):
        rep = eng.cycle()
    torch.cuda.synchronize()
    print("cycles", a.cycles, "launches/cycle", eng.launches_per_cycle, "res", rep.res[-1])


if __name__ == "__main__":
    main()
