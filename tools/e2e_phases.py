"""Break down the end-to-end solve(A, b_host) call at 256^3 into phases."""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200 import _dev as D  # noqa: E402
from paper_1809_05805_b200.engine import Engine  # noqa: E402


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


def main():
    A = P.gen_laplace3d(256)
    b = np.random.default_rng(42).standard_normal(A.n_rows)
    b /= np.linalg.norm(b)
    cfg = P.GmresConfig(restart_m=50, max_restarts=1, rel_tol=1e-14)
    for rep in range(3):
        t0 = t()
        bd = D.to_device_vector(b, A.n_rows)
        t1 = t()
        eng = Engine(A, 50, "one_sync_mgs", 1e-14, use_graph=True)
        t2 = t()
        eng.load(bd)
        r = eng.prologue()
        t3 = t()
        r = eng.cycle()
        t4 = t()
        x = eng.x_view().clone().cpu().numpy()
        t5 = t()
        del eng
        x2, h = P.solve(A, b, config=cfg, diagnostics_every=0)
        h.release()
        t6 = t()
        print(f"rep {rep}: h2d {1e3*(t1-t0):.1f} ms, engine {1e3*(t2-t1):.1f}, prologue {1e3*(t3-t2):.1f},"
              f" cycle {1e3*(t4-t3):.1f}, d2h {1e3*(t5-t4):.1f}, full solve() {1e3*(t6-t5):.1f}")
    pin = torch.empty(A.n_rows, dtype=torch.float64).pin_memory()
    t0 = t()
    pin.copy_(torch.from_numpy(b))
    t1 = t()
    g = pin.cuda(non_blocking=True)
    t2 = t()
    print(f"numpy->pinned {1e3*(t1-t0):.1f} ms, pinned->device {1e3*(t2-t1):.1f} ms")


if __name__ == "__main__":
    main()
