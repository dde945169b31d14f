"""LSB_TRACE phase timestamps of the bench's e2e call: solve(A, b_host) ->
x_host at 256^3, one GMRES(50) cycle."""

import os
import sys

os.environ["LSB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200 import _dev  # noqa: E402

if len(sys.argv) > 1:           # staging chunk, log2 doubles (default 22 = 32 MB)
    _dev._CHUNK = 1 << int(sys.argv[1])
    print("chunk", _dev._CHUNK * 8 >> 20, "MB")

A = P.gen_laplace3d(256)
b = np.random.default_rng(42).standard_normal(A.n_rows)
b /= np.linalg.norm(b)
cfg = P.GmresConfig(restart_m=50, max_restarts=1, rel_tol=1e-14, method="one_sync_mgs")
for _ in range(4):
    x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
    h.release()
