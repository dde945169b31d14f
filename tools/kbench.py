"""Kernel micro-benchmark at C2 scale (n = 256^3): average device time and
algorithmic GB/s of the hot kernels at several p, for each tuning variant.

    python tools/kbench.py [--reps 20]
"""

import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200 import _abi  # noqa: E402
from paper_1809_05805_b200 import _dev as D  # noqa: E402
from paper_1809_05805_b200.engine import Engine  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ps", default="2,10,26,51")
    a = ap.parse_args()
    lib = _abi.load()
    A = P.gen_laplace3d(256)
    eng = Engine(A, 50, "one_sync_mgs", 1e-14, use_graph=False)
    n = eng.n
    g = torch.Generator(device="cuda").manual_seed(0)
    eng.Vstore[:, :n].normal_(generator=g)
    eng.Vstore.mul_(1.0 / n ** 0.5)
    eng.flags.copy_(torch.tensor([_abi.NO_STOP, 0, -1, 0, 0, 0, 0, 0], dtype=torch.int32))
    eng.scal[_abi.S_BETA] = 1.0
    eng.coef.fill_(1e-3)
    st = D.stream()
    S = eng.Sref
    rows = []
    for p in [int(x) for x in a.ps.split(",")]:
        byt1 = 8 * n * (p + 1)
        byt2 = 8 * n * (p + 3)
        for tv in (0, 1):
            lib.lsb_set_tuning(_abi.LSB_TUNE_FUSED_OCC3 if hasattr(_abi, "LSB_TUNE_FUSED_OCC3")
                               else 1, tv)
            t = timed(lambda: lib.lsb_lagged_reduce_spmv7(S, C.byref(eng.op.c), 0, p, st), a.reps)
            rows.append((f"fused K1+SpMV occ3={tv}", p, t, byt1 / t / 1e6))
        lib.lsb_set_tuning(1, 0)
        t = timed(lambda: lib.lsb_lagged_reduce(S, 0, p, st), a.reps)
        rows.append(("K1 mdot", p, t, byt1 / t / 1e6))
        t = timed(lambda: lib.lsb_lagged_update(S, 0, p, 0, st), a.reps)
        rows.append(("K2 lagged_update", p, t, byt2 / t / 1e6))
        t = timed(lambda: lib.lsb_mgs_lvl2_small(S, 0, p, 1, 0, st), a.reps)
        rows.append(("K5 small", p, t, 0.0))
    t = timed(lambda: eng.op.apply_ptr(eng.col_ptr(0), eng.col_ptr(1), None, None, -1, st), a.reps)
    rows.append(("K6 stencil7", 0, t, 16 * n / t / 1e6))
    for name, p, t, gbs in rows:
        print(f"{name:28s} p={p:3d}  {1e3 * t:9.1f} us  {gbs:8.1f} GB/s")


if __name__ == "__main__":
    main()
