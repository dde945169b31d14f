"""Achieved parity per case: max relative deviation of the implicit-residual
curve from the reference's golden run (and the reference's own
summation-reorder floor where one was measured), iteration counts, ledger
equality.  Writes a markdown table (the committed copy: profiles/).

    python tools/parity_report.py [--out gpurun_out/parity.md] [--big]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def run(A, b, meth, m, restarts, tol, env=None):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        led = P.ReductionLedger()
        cfg = P.GmresConfig(restart_m=m, max_restarts=restarts, rel_tol=tol, method=meth)
        t0 = time.perf_counter()
        x, h = P.solve(A, b, config=cfg, ledger=led, diagnostics_every=0)
        dt = time.perf_counter() - t0
        h.release()
        return h, led, dt
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def row(case, meth, G, h, led, floor=None, dt=None):
    p = meth + "__"
    c, cr = h.implicit_curve(), G[p + "curve"]
    same = len(c) == len(cr)
    dev = float(np.max(np.abs(c - cr) / cr)) if same else float("nan")
    ledger = same and [e.kind for e in led.events] == list(G[p + "ev_kind"]) and \
        [e.scalar_count for e in led.events] == list(G[p + "ev_count"])
    return {"case": case, "method": meth, "iterations": len(c), "ref_iterations": len(cr),
            "max_rel_dev": dev, "floor": floor, "ledger_equal": bool(ledger),
            "outcome": h.outcome, "seconds": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity.md"))
    ap.add_argument("--big", action="store_true", help="include C2 256^3 and C5 N=128")
    a = ap.parse_args()
    rows = []
    floors = json.load(open(os.path.join(GOLD, "reorder_floor.json")))
    G = np.load(os.path.join(GOLD, "c1_laplace2d64.npz"))
    A = P.gen_laplace2d(64)
    b = P.gen_rhs("random", A, 42)
    for meth in ("one_sync_mgs", "two_sync_cgs2", "mgs_l1", "cgs2", "pipeline2"):
        modes = [("", {})]
        if meth in ("one_sync_mgs", "pipeline2"):
            modes = [(" whole-solve launch", {"LSB_PERSISTENT": "1", "LSB_PERSISTENT_SOLVE": "1"}),
                     (" cluster cycle", {"LSB_PERSISTENT": "1", "LSB_PERSISTENT_SOLVE": "0"}),
                     (" per-iteration", {"LSB_PERSISTENT": "0"})]
        for tag, env in modes:
            h, led, dt = run(A, b, meth, 30, 200, 1e-6, env)
            rows.append(row("C1 2D 64^2 GMRES(30)" + tag, meth, G, h, led, 5.3e-11, dt))
    G = np.load(os.path.join(GOLD, "laplace3d32.npz"))
    A = P.gen_laplace3d(32)
    b = P.gen_rhs("random", A, 42)
    for meth in ("one_sync_mgs", "two_sync_cgs2", "mgs_l1", "cgs2", "pipeline2"):
        h, led, dt = run(A, b, meth, 50, 50, 1e-6)
        rows.append(row("3D 7-pt 32^3 GMRES(50)", meth, G, h, led, None, dt))
    G = np.load(os.path.join(GOLD, "laplace3d32_ghysels.npz"))
    for tag, env in ((" SpMV+norm fused", {}), (" unfused", {"LSB_FUSE_DIRECT": "0"})):
        h, led, dt = run(A, b, "cgs1_ghysels", 50, 50, 1e-6, env)
        rows.append(row("3D 7-pt 32^3 GMRES(50) (bar 1e-7)" + tag, "cgs1_ghysels", G, h, led,
                        None, dt))
    G = np.load(os.path.join(GOLD, "laplace3d64.npz"))
    A = P.gen_laplace3d(64)
    b = P.gen_rhs("random", A, 42)
    for meth in ("one_sync_mgs", "two_sync_cgs2"):
        h, led, dt = run(A, b, meth, 50, 100, 1e-6)
        rows.append(row("3D 7-pt 64^3 GMRES(50)", meth, G, h, led, None, dt))
    Ns = (16, 64, 128) if a.big else (16, 64)
    for N in Ns:
        G = np.load(os.path.join(GOLD, f"convdiff27_{N}.npz"))
        A = P.gen_convdiff27(N)
        b = P.gen_rhs("random", A, 42)
        meths = ("one_sync_mgs", "two_sync_cgs2", "mgs_l1") + (("cgs2",) if N == 16 else ())
        for meth in meths:
            h, led, dt = run(A, b, meth, 100, 20 if N == 16 else 30, 1e-10)
            fl = floors.get(f"convdiff27_{N}", {}).get(meth)
            rows.append(row(f"C5 27-pt {N}^3 GMRES(100) tol 1e-10", meth, G, h, led, fl, dt))
    if a.big:
        for name, meths in (("laplace3d256.npz", ("one_sync_mgs",)),
                            ("laplace3d256_two_sync_cgs2.npz", ("two_sync_cgs2",)),
                            ("laplace3d256_cgs2.npz", ("cgs2",)),
                            ("laplace3d256_mgs_l1.npz", ("mgs_l1",))):
            path = os.path.join(GOLD, name)
            if not os.path.exists(path):
                continue
            G = np.load(path)
            A = P.gen_laplace3d(256)
            b = P.gen_rhs("random", A, 42)
            for meth in meths:
                h, led, dt = run(A, b, meth, 50, 100, 1e-6)
                rows.append(row("C2 3D 7-pt 256^3 GMRES(50)", meth, G, h, led, 1.3e-12, dt))
    lines = ["| case | method | iterations (ref) | max rel. deviation | reorder floor | dev / floor "
             "| ledger equal | solve s |", "|---|---|---:|---:|---:|---:|---|---:|"]
    for r in rows:
        fl = r["floor"]
        ratio = f"{r['max_rel_dev'] / fl:.2f}" if fl else ""
        lines.append(f"| {r['case']} | {r['method']} | {r['iterations']} ({r['ref_iterations']}) | "
                     f"{r['max_rel_dev']:.3g} | {fl if fl is None else f'{fl:.3g}'} | {ratio} | "
                     f"{r['ledger_equal']} | {r['seconds']:.3f} |")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(a.out[:-3] + ".jsonl", "w") as fh:
        for r in rows:
            fh.write(json.dumps(r) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
