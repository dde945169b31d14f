import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1809_05805_b200 as P
from paper_1809_05805_b200 import _dev as D
from paper_1809_05805_b200.engine import Engine
A = P.gen_laplace3d(256); n = A.n_rows
b = np.random.default_rng(42).standard_normal(n); b /= np.linalg.norm(b)
eng = Engine(A, 50, "one_sync_mgs", 1e-14)
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(4):
    t0 = T()
    bd = D.to_device_vector(b, n); t1 = T()
    eng.reset(1e-14, 1.0); t2 = T()
    eng.load(bd); t3 = T()
    hb = D.HostBuffer(n); t4 = time.perf_counter()
    rep_ = eng.prologue(); t5 = T()
    r = eng.cycle(); t6 = T()
    x = eng.x_view().clone(); t7 = T()
    y = D.out_like(x, True, hb); t8 = time.perf_counter()
    print(f"h2d {1e3*(t1-t0):.2f} reset {1e3*(t2-t1):.2f} load {1e3*(t3-t2):.2f} hostbuf {1e3*(t4-t3):.2f} prologue {1e3*(t5-t4):.2f} cycle {1e3*(t6-t5):.2f} clone {1e3*(t7-t6):.2f} d2h {1e3*(t8-t7):.2f}")
