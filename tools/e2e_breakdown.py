"""Where the end-to-end solve(A, b_numpy) -> x_numpy time goes at C2
(256^3, GmresConfig(50, 1 cycle)), with the engine reused across calls as in
the bench: LSB_TRACE phase marks (synchronised) for a few warm calls, plus
the raw host<->device copy rates of the staging pipeline."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200 import _dev as D  # noqa: E402


def main():
    A = P.gen_laplace3d(256)
    b = np.random.default_rng(42).standard_normal(A.n_rows)
    b /= np.linalg.norm(b)
    cfg = P.GmresConfig(restart_m=50, max_restarts=1, rel_tol=1e-14)
    for _ in range(2):
        x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
        h.release()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
        h.release()
        ts.append(time.perf_counter() - t0)
    print(f"solve() wall per call: {', '.join(f'{1e3 * t:.1f}' for t in ts)} ms")
    os.environ["LSB_TRACE"] = "1"
    for _ in range(2):
        x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
        h.release()
    del os.environ["LSB_TRACE"]
    n = A.n_rows
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = D.h2d(b, torch.device("cuda"))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        hb = D.HostBuffer(n)
        y = D.d2h(d, hb.get())
        t2 = time.perf_counter()
        out = np.empty(n)
        t3 = time.perf_counter()
        out[:] = b
        t4 = time.perf_counter()
        print(f"h2d staged {1e3 * (t1 - t0):.1f} ms ({8 * n / (t1 - t0) / 1e9:.1f} GB/s), "
              f"d2h staged {1e3 * (t2 - t1):.1f} ms ({8 * n / (t2 - t1) / 1e9:.1f} GB/s), "
              f"host memcpy {1e3 * (t4 - t3):.1f} ms ({8 * n / (t4 - t3) / 1e9:.1f} GB/s), "
              f"cpus {os.cpu_count()}, torch threads {torch.get_num_threads()}")


if __name__ == "__main__":
    main()
