import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1809_05805_b200 as P
A = P.gen_laplace3d(256); n = A.n_rows
b = np.random.default_rng(42).standard_normal(n); b /= np.linalg.norm(b)
cfg = P.GmresConfig(restart_m=50, max_restarts=1, rel_tol=1e-14)
def e2e_once():
    x, h = P.solve(A, b, config=cfg, diagnostics_every=0)
    assert h.iterations == 50 and isinstance(x, np.ndarray)
    h.release()
for i in range(7):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e2e_once()
    print(f"call {i}: {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
