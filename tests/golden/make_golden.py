"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py small     # seconds: kernel + C1 + Simoncini + 3D N=32 + 27pt N=16
    python tests/golden/make_golden.py c2        # ~30 min: 3D 7-point 256^3 one-sync GMRES(50) to 1e-6
    python tests/golden/make_golden.py c5        # 27-point N=64 GMRES(100) to 1e-10

The reference is imported read-only from /root/reference/pkg/src
(OPENBLAS_NUM_THREADS pinned to 1 for reproducibility).  The
fixtures are small .npz files committed beside this script; nothing at test
or bench time reads /root/reference.
"""

import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import lowsync as ls  # noqa: E402
from oracle import lowsync_oracle as orc  # noqa: E402  (generators only: builds the same CSR for 3D)


def _ref_csr(O):
    """Wrap an oracle-built CSR into the reference CsrMatrix (runs its validate)."""
    return ls.CsrMatrix(O.n_rows, O.n_cols, O.row_ptr, O.col_idx, O.values)


def _run(A, b, method, m, restarts, tol, diag=0, btf=1.0):
    led = ls.ReductionLedger()
    cfg = ls.GmresConfig(restart_m=m, max_restarts=restarts, rel_tol=tol, method=method,
                         breakdown_tol_factor=btf)
    t0 = time.perf_counter()
    x, h = ls.solve(A, b, config=cfg, ledger=led, diagnostics_every=diag)
    dt = time.perf_counter() - t0
    ev = led.events
    out = dict(
        x=x,
        curve=h.implicit_curve(),
        iters=np.array([r.iteration for r in h.records]),
        reductions=np.array([r.reductions for r in h.records]),
        true_rel=np.array([np.nan if r.true_rel_res is None else r.true_rel_res for r in h.records]),
        s_norm=np.array([np.nan if r.s_norm is None else r.s_norm for r in h.records]),
        orth_loss=np.array([np.nan if r.orth_loss is None else r.orth_loss for r in h.records]),
        cycle_starts=np.array(h.cycle_starts),
        outcome=np.array(h.outcome),
        final_true_rel_res=np.array(h.final_true_rel_res),
        k=np.array(h.k),
        ev_iter=np.array([e.iteration for e in ev]),
        ev_kind=np.array([e.kind for e in ev]),
        ev_count=np.array([e.scalar_count for e in ev]),
        ev_elig=np.array([e.overlap_eligible for e in ev]),
        seconds=np.array(dt),
    )
    if h.basis is not None and h.basis.shape[1] <= 128:
        k = h.k
        cols = h.basis[:, : k + 1]
        nz = np.any(cols != 0, axis=0)
        out["final_orth_loss"] = np.array(ls.orthogonality_loss(cols[:, nz]))
        out["hessenberg"] = h.hessenberg
    return out


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, f"{os.path.getsize(path) / 1024:.1f} KiB")


def small():
    # ---- primitives on seeded inputs (kernels.py:256-362)
    rng = np.random.default_rng(1234)
    prims = {}
    for tag, (n, p) in {"a": (1000, 7), "b": (4099, 33), "c": (257, 1)}.items():
        X = np.asfortranarray(rng.standard_normal((n, p)))
        u, w = rng.standard_normal(n), rng.standard_normal(n)
        alpha = rng.standard_normal(p)
        led = ls.ReductionLedger()
        prims[f"{tag}_X"], prims[f"{tag}_u"], prims[f"{tag}_w"], prims[f"{tag}_alpha"] = X, u, w, alpha
        prims[f"{tag}_mdot_pair"] = ls.mdot_pair(X, u, w, led)
        prims[f"{tag}_mass"] = ls.mass_inner_product(X, w, led)
        prims[f"{tag}_maxpy"] = ls.maxpy(w, X, alpha)
        prims[f"{tag}_norm"] = np.array(ls.norm2(w, led))
        prims[f"{tag}_dot"] = np.array(ls.dot(u, w, led))
    # SpMV on random sparse rows incl. empty rows and long rows (pairwise path)
    n = 600
    lens = rng.integers(0, 300, size=n)
    lens[::17] = 0
    rows = np.repeat(np.arange(n), lens)
    cols = np.concatenate([np.sort(rng.choice(n, size=L, replace=False)) for L in lens])
    vals = rng.standard_normal(rows.size) * np.exp(rng.standard_normal(rows.size) * 3)
    A = ls.CsrMatrix.from_coo(n, n, rows, cols, vals)
    xs = rng.standard_normal(n)
    prims.update(sp_row_ptr=A.row_ptr, sp_col_idx=A.col_idx, sp_values=A.values, sp_x=xs,
                 sp_y=ls.spmv(A, xs))
    # generators
    L2 = ls.gen_laplace2d(64)
    prims.update(l2_row_ptr=L2.row_ptr, l2_col_idx=L2.col_idx, l2_values=L2.values,
                 rhs42_4096=ls.gen_rhs("random", L2, 42))
    # 3D generators pinned against a loop-built reference from_coo at small N
    for tag, offs, N in (("l3", None, 6), ("c27", orc.convdiff27_offsets(0.5), 5)):
        if offs is None:
            offs = [((0, 0, 0), 6.0)] + [(tuple(s if a == ax else 0 for a in range(3)), -1.0)
                                         for ax in range(3) for s in (-1, 1)]
        r_, c_, v_ = [], [], []
        for iz in range(N):
            for iy in range(N):
                for ix in range(N):
                    i = (iz * N + iy) * N + ix
                    for (dx, dy, dz), val in offs:
                        jx, jy, jz = ix + dx, iy + dy, iz + dz
                        if 0 <= jx < N and 0 <= jy < N and 0 <= jz < N:
                            r_.append(i); c_.append((jz * N + jy) * N + jx); v_.append(val)
        R = ls.CsrMatrix.from_coo(N ** 3, N ** 3, r_, c_, v_)
        prims.update({f"{tag}_N": np.array(N), f"{tag}_row_ptr": R.row_ptr,
                      f"{tag}_col_idx": R.col_idx, f"{tag}_values": R.values})
    # ---- orthogonalizers through qr_factorize (gram_schmidt.py:305-358)
    sys.path.insert(0, "/root/reference/pkg/tests")
    from helpers import conditioned_matrix
    for kappa in (8.0, 1e6, 1e10):
        M = conditioned_matrix(60, 20, kappa, seed=22)
        prims[f"qr_M_{kappa:g}"] = M
        for meth in ("mgs", "cgs1", "cgs2", "mgs_wy", "cgs2_wy"):
            Q, R = ls.qr_factorize(M, method=meth)
            prims[f"qr_{meth}_{kappa:g}_Q"] = Q
            prims[f"qr_{meth}_{kappa:g}_R"] = R
    _save("kernels.npz", **prims)

    methods = ("one_sync_mgs", "two_sync_cgs2", "mgs_l1", "cgs2", "pipeline2")
    # ---- C1: 2D 5-point 64^2, GMRES(30), tol 1e-6, seed 42
    A = ls.gen_laplace2d(64)
    b = ls.gen_rhs("random", A, 42)
    out = {}
    for meth in methods:
        r = _run(A, b, meth, 30, 200, 1e-6)
        out.update({f"{meth}__{k}": v for k, v in r.items()})
        print("C1", meth, len(r["curve"]), r["outcome"], r["final_true_rel_res"])
    _save("c1_laplace2d64.npz", **out)

    # ---- Simoncini n=100, m=100, tol 1e-14, diagnostics every iteration
    A = ls.gen_simoncini(100)
    b = ls.gen_rhs("random", A, 42)
    out = {}
    for meth in methods:
        r = _run(A, b, meth, 100, 1, 1e-14, diag=1)
        out.update({f"{meth}__{k}": v for k, v in r.items()})
        print("simoncini", meth, len(r["curve"]), r["outcome"])
    _save("simoncini100.npz", **out)

    # ---- 3D 7-point N=32, GMRES(50), tol 1e-6 (C2 at small scale)
    A = _ref_csr(orc.laplace3d(32))
    b = ls.gen_rhs("random", A, 42)
    out = {}
    for meth in methods:
        r = _run(A, b, meth, 50, 50, 1e-6)
        out.update({f"{meth}__{k}": v for k, v in r.items()})
        print("L3D32", meth, len(r["curve"]), r["outcome"])
    _save("laplace3d32.npz", **out)

    # ---- 27-point convection-diffusion N=16, GMRES(100), tol 1e-10 (C5 small)
    A = _ref_csr(orc.convdiff27(16))
    b = ls.gen_rhs("random", A, 42)
    out = {}
    for meth in ("one_sync_mgs", "two_sync_cgs2", "mgs_l1", "cgs2"):
        r = _run(A, b, meth, 100, 20, 1e-10)
        out.update({f"{meth}__{k}": v for k, v in r.items()})
        print("C27_16", meth, len(r["curve"]), r["outcome"], r.get("final_orth_loss"))
    _save("convdiff27_16.npz", **out)


def ghysels():
    """cgs1_ghysels runs: the stall problem (cancellation failure), a
    well-conditioned system, the identity (exact-zero radicand), C1."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from helpers import spread_system
    out = {}
    cases = {
        "sim": (ls.gen_simoncini(100), None, 100, 1, 1e-14, 1),
        "spread": spread_system(10, seed=10)[0::2] + (10, 10, 1e-12, 0),
        "eye": (ls.CsrMatrix.diagonal(np.ones(5)), np.ones(5), 5, 10, 1e-10, 0),
        "c1": (ls.gen_laplace2d(64), None, 30, 200, 1e-6, 0),
    }
    for tag, (A, b, m, R, tol, diag) in cases.items():
        if b is None:
            b = ls.gen_rhs("random", A, 42)
        r = _run(A, b, "cgs1_ghysels", m, R, tol, diag=diag)
        out.update({f"{tag}__{k}": v for k, v in r.items()})
        out[f"{tag}__b"] = b
        if hasattr(A, "to_dense") and A.n_rows <= 100:
            out[f"{tag}__A"] = A.to_dense()
        print("ghysels", tag, len(r["curve"]), r["outcome"])
    _save("ghysels.npz", **out)


def ghysels3d():
    """cgs1_ghysels on the 3D 7-point N=32 problem of laplace3d32.npz
    (GMRES(50), tol 1e-6): the case where the device fuses the Ghysels
    step's SpMV and norm into its reduction (7-point stencil)."""
    A = _ref_csr(orc.laplace3d(32))
    b = ls.gen_rhs("random", A, 42)
    r = _run(A, b, "cgs1_ghysels", 50, 50, 1e-6)
    print("L3D32 cgs1_ghysels", len(r["curve"]), r["outcome"])
    _save("laplace3d32_ghysels.npz", **{f"cgs1_ghysels__{k}": v for k, v in r.items()})


def extras():
    """true_residual_every probes (gmres.py:273-283)."""
    out = {}
    A = ls.gen_simoncini(100)
    b = ls.gen_rhs("random", A, 42)
    for meth in ("mgs_l1", "one_sync_mgs"):
        led = ls.ReductionLedger()
        cfg = ls.GmresConfig(restart_m=100, max_restarts=1, rel_tol=1e-14, method=meth)
        _, h = ls.solve(A, b, config=cfg, ledger=led, diagnostics_every=1, true_residual_every=1)
        out[f"sim_{meth}_true"] = np.array([np.nan if r.true_rel_res is None else r.true_rel_res
                                            for r in h.records])
        out[f"sim_{meth}_curve"] = h.implicit_curve()
    A = ls.gen_laplace2d(64)
    b = ls.gen_rhs("random", A, 42)
    for meth, te in (("one_sync_mgs", 5), ("two_sync_cgs2", 3), ("cgs2", 7)):
        led = ls.ReductionLedger()
        cfg = ls.GmresConfig(restart_m=30, max_restarts=200, rel_tol=1e-6, method=meth)
        _, h = ls.solve(A, b, config=cfg, ledger=led, diagnostics_every=0, true_residual_every=te)
        out[f"c1_{meth}_true"] = np.array([np.nan if r.true_rel_res is None else r.true_rel_res
                                           for r in h.records])
        out[f"c1_{meth}_curve"] = h.implicit_curve()
        out[f"c1_{meth}_every"] = np.array(te)
    _save("extras.npz", **out)


def jacobi():
    """Right Jacobi preconditioning (gmres.py:106-126, 254, 264-265, 277, 297)
    on a 2D 5-point matrix whose diagonal varies in [4, 10] (so M^-1 is not a
    multiple of the identity), several restarts, every method."""
    O = orc.laplace2d(24)
    rng = np.random.default_rng(8)
    vals = O.values.copy()
    rows = np.repeat(np.arange(O.n_rows), np.diff(O.row_ptr))
    vals[O.col_idx == rows] += rng.uniform(0.0, 6.0, O.n_rows)
    A = ls.CsrMatrix(O.n_rows, O.n_cols, O.row_ptr, O.col_idx, vals)
    b = ls.gen_rhs("random", A, 5)
    out = dict(row_ptr=A.row_ptr, col_idx=A.col_idx, values=A.values, b=b)
    for meth in ("one_sync_mgs", "two_sync_cgs2", "mgs_l1", "cgs2", "pipeline2", "cgs1_ghysels"):
        led = ls.ReductionLedger()
        cfg = ls.GmresConfig(restart_m=10, max_restarts=200, rel_tol=1e-10, method=meth,
                             precond="jacobi")
        x, h = ls.solve(A, b, config=cfg, ledger=led, diagnostics_every=0)
        ev = led.events
        out.update({f"{meth}__x": x, f"{meth}__curve": h.implicit_curve(),
                    f"{meth}__cycle_starts": np.array(h.cycle_starts),
                    f"{meth}__outcome": np.array(h.outcome),
                    f"{meth}__final_true_rel_res": np.array(h.final_true_rel_res),
                    f"{meth}__ev_kind": np.array([e.kind for e in ev]),
                    f"{meth}__ev_count": np.array([e.scalar_count for e in ev]),
                    f"{meth}__ev_iter": np.array([e.iteration for e in ev]),
                    f"{meth}__ev_elig": np.array([e.overlap_eligible for e in ev])})
        print("jacobi", meth, len(h.implicit_curve()), h.outcome, h.final_true_rel_res)
    _save("jacobi.npz", **out)


def big_c2(N=256, methods=("one_sync_mgs",), tag=""):
    t0 = time.perf_counter()
    A = _ref_csr(orc.laplace3d(N))
    b = ls.gen_rhs("random", A, 42)
    print("built", time.perf_counter() - t0, flush=True)
    out = {}
    for meth in methods:
        r = _run(A, b, meth, 50, 100, 1e-6)
        r.pop("x")
        out.update({f"{meth}__{k}": v for k, v in r.items()})
        print(f"L3D{N}", meth, len(r["curve"]), r["outcome"], r["seconds"], flush=True)
    _save(f"laplace3d{N}{tag}.npz", **out)


def big_c5(N=64):
    A = _ref_csr(orc.convdiff27(N))
    b = ls.gen_rhs("random", A, 42)
    out = {}
    for meth in ("one_sync_mgs", "two_sync_cgs2", "mgs_l1"):
        r = _run(A, b, meth, 100, 30, 1e-10)
        r.pop("x")
        out.update({f"{meth}__{k}": v for k, v in r.items()})
        print(f"C27_{N}", meth, len(r["curve"]), r["outcome"], r.get("final_orth_loss"), flush=True)
    _save(f"convdiff27_{N}.npz", **out)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        small()
    elif what == "extras":
        extras()
    elif what == "ghysels":
        ghysels()
    elif what == "ghysels3d":
        ghysels3d()
    elif what == "c2":
        big_c2(int(sys.argv[2]) if len(sys.argv) > 2 else 256)
    elif what == "l3d64":
        # P = 8 slab tests (8 planes per rank): 3D 7-point 64^3, GMRES(50), tol 1e-6
        big_c2(64, ("one_sync_mgs", "two_sync_cgs2"))
    elif what == "c2m":
        # one further C2 variant per process, so they can run side by side:
        #   python tests/golden/make_golden.py c2m two_sync_cgs2   (-> laplace3d256_two_sync_cgs2.npz)
        big_c2(256, (sys.argv[2],), tag="_" + sys.argv[2])
    elif what == "jacobi":
        jacobi()
    elif what == "c5":
        big_c5(int(sys.argv[2]) if len(sys.argv) > 2 else 64)
