"""Launch-bound regime anatomy at C1 (2D 64^2, GMRES(30)): device time per
graph-replayed cycle vs the whole solve() wall time, per method.

    python tools/c1_profile.py [--N 64] [--m 30]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--m", type=int, default=30)
    ap.add_argument("--cycles", type=int, default=20)
    ap.add_argument("--methods", default="one_sync_mgs,two_sync_cgs2,mgs_l1,cgs2")
    a = ap.parse_args()
    A = P.gen_laplace2d(a.N)
    b = np.asarray(P.gen_rhs("random", A, 42))
    for meth in a.methods.split(","):
        eng = Engine(A, a.m, meth, 1e-300, use_graph=True)
        eng.load(torch.as_tensor(b).cuda())
        eng.prologue()
        eng.cycle()
        eng.cycle()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(a.cycles):
            eng.cycle()
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / a.cycles
        dev = e0.elapsed_time(e1) / a.cycles / 1e3
        print(f"{meth:14s} launches/cycle {eng.launches_per_cycle:4d}  device {1e6 * dev / a.m:6.2f} us/it"
              f"  wall {1e6 * wall / a.m:6.2f} us/it  ({a.m / dev:8.0f} it/s device)", flush=True)
        del eng


if __name__ == "__main__":
    main()
