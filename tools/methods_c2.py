"""Steady-state GMRES(50) cycle rate of every orthogonalization method at
256^3 (config 2), next to each method's HBM ceiling from SURVEY §8(a)'s
algorithmic bytes per iteration (+16n for an unfused stencil SpMV).

    python tools/methods_c2.py [--N 256] [--cycles 3]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200.engine import Engine  # noqa: E402

PEAK = 6551.4e9
M = 50


def bytes_per_cycle(method, n):
    """Algorithmic bytes: SURVEY §8(a) table, p = i+1 (lagged) or i (direct)."""
    tot = 0
    for i in range(1, M + 1):
        if method in ("one_sync_mgs", "pipeline2"):
            p = i + 1
            tot += 8 * n * (2 * p + 4)             # SpMV fused into K1
        elif method == "two_sync_cgs2":
            p = i + 1
            tot += 8 * n * (3 * p + 6)
        elif method == "cgs2":
            tot += 8 * n * (3 * i + 7) + 16 * n
        elif method == "mgs_l1":
            tot += 8 * n * (4 * i + 3) + 16 * n
        elif method == "cgs1_ghysels":
            tot += 8 * n * (2 * i + 4) + 16 * n
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--cycles", type=int, default=3)
    ap.add_argument("--methods", default="one_sync_mgs,pipeline2,two_sync_cgs2,cgs2,mgs_l1,cgs1_ghysels")
    a = ap.parse_args()
    A = P.gen_laplace3d(a.N)
    n = A.n_rows
    b = np.random.default_rng(42).standard_normal(n)
    b /= np.linalg.norm(b)
    bd = torch.as_tensor(b).cuda()
    out = {}
    for meth in a.methods.split(","):
        eng = Engine(A, M, meth, 1e-14, use_graph=True)
        eng.load(bd)
        eng.prologue()
        eng.cycle()
        eng.cycle()                                   # capture + warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        its = 0
        for _ in range(a.cycles):
            rep = eng.cycle()
            its += len(rep.res) if hasattr(rep, "res") else M
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.cycles
        ceil_ms = bytes_per_cycle(meth, n) / PEAK * 1e3
        out[meth] = {"ms_per_cycle": round(ms, 2), "it_s": round(M * 1e3 / ms, 1),
                     "hbm_ceiling_ms": round(ceil_ms, 2), "frac": round(ceil_ms / ms, 3)}
        print(meth, out[meth], flush=True)
        del eng
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
