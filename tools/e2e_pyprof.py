"""cProfile of the bench's e2e call (solve(A, b_host) -> x_host, 256^3,
one GMRES(50) cycle): where the host time around the device cycle goes."""

import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402

A = P.gen_laplace3d(256)
b = np.random.default_rng(42).standard_normal(A.n_rows)
b /= np.linalg.norm(b)
cfg = P.GmresConfig(restart_m=50, max_restarts=1, rel_tol=1e-14, method="one_sync_mgs")


def once():
    x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
    h.release()


for _ in range(2):
    once()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    once()
print("e2e ms per solve", (time.perf_counter() - t0) / 5 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    once()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
