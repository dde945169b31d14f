"""Phase anatomy of the persistent cluster cycle (lsb_cycle_persistent) at
C1: per-iteration time split into SpMV+dots / barrier 1 / gather / small
state / barrier 2 / K2 / barrier 3, from CTA 0's globaltimer stamps.

    python tools/persist_trace.py [--N 64] [--m 30]
"""

import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200 import _abi  # noqa: E402
from paper_1809_05805_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=64)
    ap.add_argument("--m", type=int, default=30)
    ap.add_argument("--ctas", type=int, default=0, help="cluster size (0 auto)")
    a = ap.parse_args()
    lib = _abi.load()
    lib.lsb_set_tuning(_abi.TUNE_PERSIST_CTAS, a.ctas)
    A = P.gen_laplace2d(a.N)
    b = np.asarray(P.gen_rhs("random", A, 42))
    eng = Engine(A, a.m, "one_sync_mgs", 1e-300, use_graph=False)
    assert eng.persistent
    eng.load(torch.as_tensor(b).cuda())
    eng.prologue()
    eng.cycle()
    lib.lsb_set_tuning(_abi.TUNE_PERSIST_TRACE, 1)
    eng.cycle()
    torch.cuda.synchronize()
    lib.lsb_set_tuning(_abi.TUNE_PERSIST_TRACE, 0)
    n = 10 * (a.m + 1)
    buf = (C.c_int64 * n)()
    _abi.call("lsb_persist_trace", buf, n)
    t = np.array(buf, dtype=np.float64).reshape(a.m + 1, 10)
    names = ["spmv+dots", "barrier1", "gather", "small", "k2", "barrier3+gate"]
    d = np.zeros((a.m, 6))
    for i in range(a.m):
        seg = [t[i, 1] - t[i, 0], t[i, 2] - t[i, 1], t[i, 3] - t[i, 2], t[i, 4] - t[i, 3],
               t[i, 5] - t[i, 4], t[i + 1, 0] - t[i, 5]]
        d[i] = seg
    print("mean ns per iteration:", {k: round(float(v), 1) for k, v in zip(names, d[1:].mean(0))})
    print("total us per iteration:", round(float(d[1:].sum(1).mean()) / 1e3, 2))
    sm = np.stack([t[2:a.m, 6] - t[2:a.m, 3], t[2:a.m, 7] - t[2:a.m, 6], t[2:a.m, 8] - t[2:a.m, 7],
                   t[2:a.m, 9] - t[2:a.m, 8], t[2:a.m, 4] - t[2:a.m, 9]], 1)
    print("small-state split ns (front, T col, c, settle sync, givens+tail):",
          [round(float(v), 1) for v in sm.mean(0)])


if __name__ == "__main__":
    main()
