import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
import paper_1809_05805_b200 as P
from paper_1809_05805_b200.engine import Engine
A = P.gen_laplace2d(64)
for _ in range(5): Engine(A, 30, "one_sync_mgs", 1e-6)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100): e = Engine(A, 30, "one_sync_mgs", 1e-6)
torch.cuda.synchronize()
print("Engine() us", (time.perf_counter() - t0) / 100 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(100): e = Engine(A, 30, "one_sync_mgs", 1e-6)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
