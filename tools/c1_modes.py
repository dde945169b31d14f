import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1809_05805_b200 as P
G = np.load("tests/golden/c1_laplace2d64.npz")
A = P.gen_laplace2d(64); b = P.gen_rhs("random", A, 42)
for meth in ["one_sync_mgs"]:
    for persist, whole in (("0","0"),("1","0"),("1","1")):
        os.environ["LSB_PERSISTENT"]=persist; os.environ["LSB_PERSISTENT_SOLVE"]=whole
        cfg = P.GmresConfig(restart_m=30, max_restarts=200, rel_tol=1e-6, method=meth)
        x, h = P.solve(A, b, config=cfg, ledger=P.ReductionLedger(), diagnostics_every=0)
        c = h.implicit_curve(); cu = G[meth+"__curve"]
        rel = np.abs(c-cu)/np.abs(cu)
        starts = h.cycle_starts
        print(meth, persist, whole, len(c), "max", rel.max(), "at", int(np.argmax(rel)),
              "per-cycle-start", ["%.1e" % rel[s] for s in starts[1:6]])
        ends = starts[1:] + [len(c)]
        print("   per-cycle max", " ".join("%.0e" % rel[a:e].max() for a, e in zip(starts, ends)))
