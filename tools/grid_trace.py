"""Phase anatomy of the grid-persistent cycle (LSB_TUNE_GRID_TRACE=1): 3D
7-point N^3 one-sync GMRES(50), ns per phase per iteration on CTA 0."""
import ctypes as C
import os
import sys

os.environ["LSB_TUNE"] = "14=1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200 import _abi  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
A = P.gen_laplace3d(N)
b = P.gen_rhs("random", A, 42)
cfg = P.GmresConfig(restart_m=50, max_restarts=1, rel_tol=1e-14)
P.solve(A, b, config=cfg, diagnostics_every=0)
lib = _abi.load()
buf = (C.c_int64 * 8)()
lib.lsb_grid_trace(buf, 8)
for _ in range(3):
    x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
torch.cuda.synchronize()
lib.lsb_grid_trace(buf, 8)
its = 3 * 50
names = ["spmv", "sync1", "dots", "sync2+sums+sync3", "K5(cta0)", "sync4", "K2", "sync5"]
print(" ".join(f"{n} {buf[k] / its / 1000:.2f}us" for k, n in enumerate(names)),
      f"total {sum(buf) / its / 1000:.2f}us/it")
