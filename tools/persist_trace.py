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
    buf = (C.c_int64 * 18)()
    _abi.call("lsb_persist_trace", buf, 18)
    t = np.array(buf, dtype=np.float64)
    its = max(t[8], 1)
    names = ["row CTA: spmv+dots", "wait b1", "wait b2 (gather+small)", "K2", "wait b3 (fold)",
             "ctl: a/beta", "ctl: T col", "ctl: c + join"]
    print("mean SM cycles per iteration:", {k: round(float(v) / its, 1) for k, v in zip(names, t[:8])})
    print("row-CTA total cycles per iteration:", round(float(t[:5].sum()) / its, 1))
    c0 = max(t[13], 1)
    print("control CTA: B1 exit -> B2 arrive", round(float(t[11]) / c0, 1), "cycles; B2 arrive -> exit",
          round(float(t[12]) / c0, 1), "| gather done at", round(float(t[14]) / c0, 1),
          "small done at", round(float(t[15]) / c0, 1), "| small: entry->sync", round(float(t[16]) / c0, 1),
          "warp0 tol chain done at", round(float(t[17]) / c0, 1), "after the first sync")
    print("row CTA: thread 0's SpMV rows done at", round(float(t[9]) / its, 1),
          "cycles, SpMV of the whole CTA done at", round(float(t[10]) / its, 1))


if __name__ == "__main__":
    main()
