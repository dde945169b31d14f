"""Pin the CPU oracle against fixtures produced by the reference itself.

The oracle (oracle/lowsync_oracle.py) restates the reference with the same
numpy/BLAS calls, so inside one process it matches the reference bit for
bit.  Across processes OpenBLAS's dgemv result depends on buffer alignment
(the reference itself drifts ~1e-12 between two runs of the 3D problem), so
solver histories are compared at the 1e-10 parity bar and iteration
counts, outcomes and ledger events exactly.
"""

import os

import numpy as np
import pytest

from oracle import lowsync_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


@pytest.fixture(scope="module")
def K():
    return _load("kernels.npz")


def test_primitives_match_reference(K):
    for tag in ("a", "b", "c"):
        X, u, w, al = K[f"{tag}_X"], K[f"{tag}_u"], K[f"{tag}_w"], K[f"{tag}_alpha"]
        X = np.asfortranarray(X)
        led = orc.Ledger()
        G = orc.mdot_pair(X, u, w, led)
        np.testing.assert_allclose(G, K[f"{tag}_mdot_pair"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(orc.mass_ip(X, w, led), K[f"{tag}_mass"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(orc.maxpy(w, X, al), K[f"{tag}_maxpy"], rtol=0, atol=1e-13)
        assert abs(orc.norm2(w, led) - float(K[f"{tag}_norm"])) <= 4 * orc.EPS * float(K[f"{tag}_norm"])
        assert [e[1] for e in led.events] == ["mdot", "mdot", "norm"]
        assert led.events[0][2] == 2 * X.shape[1]


def test_spmv_bitwise(K):
    A = orc.Csr(600, 600, K["sp_row_ptr"], K["sp_col_idx"], K["sp_values"])
    assert np.array_equal(orc.spmv(A, K["sp_x"]), K["sp_y"])


def test_generators_bitwise(K):
    L2 = orc.laplace2d(64)
    assert np.array_equal(L2.row_ptr, K["l2_row_ptr"])
    assert np.array_equal(L2.col_idx, K["l2_col_idx"])
    assert np.array_equal(L2.values, K["l2_values"])
    assert np.array_equal(orc.rhs_random(4096, 42), K["rhs42_4096"])
    for tag, gen in (("l3", orc.laplace3d), ("c27", orc.convdiff27)):
        N = int(K[f"{tag}_N"])
        A = gen(N)
        assert np.array_equal(A.row_ptr, K[f"{tag}_row_ptr"])
        assert np.array_equal(A.col_idx, K[f"{tag}_col_idx"])
        assert np.array_equal(A.values, K[f"{tag}_values"])


@pytest.mark.parametrize("kappa", ["8", "1e+06", "1e+10"])
@pytest.mark.parametrize("meth", ["mgs", "cgs1", "cgs2", "mgs_wy", "cgs2_wy"])
def test_qr_kernels_match_reference(K, meth, kappa):
    M = K[f"qr_M_{kappa}"]
    Q, R, _ = orc.qr_columns(M, meth)
    np.testing.assert_allclose(Q, K[f"qr_{meth}_{kappa}_Q"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(R, K[f"qr_{meth}_{kappa}_R"], rtol=0,
                               atol=1e-12 * np.abs(R).max())


def _check_run(run, G, meth, exact_curve_tol=1e-10):
    p = meth + "__"
    curve = G[p + "curve"]
    assert len(run.curve) == len(curve), (meth, len(run.curve), len(curve))
    rel = np.abs(np.array(run.curve) - curve) / np.abs(curve)
    assert rel.max() <= exact_curve_tol, (meth, rel.max())
    assert run.outcome == str(G[p + "outcome"])
    assert run.cycle_starts == list(G[p + "cycle_starts"])
    assert run.reductions == list(G[p + "reductions"])
    ev = run.ledger.events
    assert [e[0] for e in ev] == list(G[p + "ev_iter"])
    assert [e[1] for e in ev] == list(G[p + "ev_kind"])
    assert [e[2] for e in ev] == list(G[p + "ev_count"])
    assert [e[3] for e in ev] == list(G[p + "ev_elig"])
    f = float(G[p + "final_true_rel_res"])
    assert abs(run.final_true_rel_res - f) <= 1e-10 * f


METHODS = ["one_sync_mgs", "two_sync_cgs2", "mgs_l1", "cgs2", "pipeline2"]


@pytest.mark.parametrize("meth", METHODS)
def test_c1_laplace2d_history(meth):
    G = _load("c1_laplace2d64.npz")
    A = orc.laplace2d(64)
    b = orc.rhs_random(A.n_rows, 42)
    run = orc.gmres(A, b, meth, 30, 200, 1e-6)
    _check_run(run, G, meth)
    if meth == "one_sync_mgs":
        assert len(run.curve) == 365 and len(run.cycle_starts) == 13
        assert len(run.ledger.events) == 392


@pytest.mark.parametrize("meth", METHODS)
def test_simoncini_history_with_diagnostics(meth):
    G = _load("simoncini100.npz")
    A = orc.simoncini(100)
    b = orc.rhs_random(100, 42)
    run = orc.gmres(A, b, meth, 100, 1, 1e-14, diag_every=1)
    _check_run(run, G, meth, exact_curve_tol=1e-9)
    s = np.array(run.s_norm, dtype=float)
    np.testing.assert_allclose(s, G[meth + "__s_norm"], rtol=1e-6, atol=1e-14)


@pytest.mark.parametrize("meth", METHODS)
def test_laplace3d_small_history(meth):
    G = _load("laplace3d32.npz")
    A = orc.laplace3d(32)
    b = orc.rhs_random(A.n_rows, 42)
    run = orc.gmres(A, b, meth, 50, 50, 1e-6)
    _check_run(run, G, meth)


def test_laplace3d_small_ghysels_history():
    G = _load("laplace3d32_ghysels.npz")
    A = orc.laplace3d(32)
    b = orc.rhs_random(A.n_rows, 42)
    run = orc.gmres(A, b, "cgs1_ghysels", 50, 50, 1e-6)
    # the Pythagorean residual sqrt(|z|^2 - |y|^2) loses digits as the
    # radicand shrinks (1.7e-9 here; the device bar for Ghysels is 1e-7)
    _check_run(run, G, "cgs1_ghysels", exact_curve_tol=1e-8)


@pytest.mark.parametrize("meth", ["one_sync_mgs", "two_sync_cgs2", "mgs_l1", "cgs2"])
def test_convdiff27_small_history(meth):
    G = _load("convdiff27_16.npz")
    A = orc.convdiff27(16)
    b = orc.rhs_random(A.n_rows, 42)
    run = orc.gmres(A, b, meth, 100, 20, 1e-10, cycle_orth=True)
    _check_run(run, G, meth)
    ref = float(G[meth + "__final_orth_loss"])
    assert 0.1 * ref <= run.cycle_orth_loss[-1] <= 10 * ref


@pytest.mark.parametrize("tag", ["sim", "spread", "eye", "c1"])
def test_ghysels_matches_reference(tag):
    G = _load("ghysels.npz")
    p = tag + "__"
    if tag == "c1":
        A = orc.laplace2d(64)
        m, R, tol, diag = 30, 200, 1e-6, 0
    else:
        A = orc.dense_to_csr(G[p + "A"])
        m, R, tol, diag = {"sim": (100, 1, 1e-14, 1), "spread": (10, 10, 1e-12, 0),
                           "eye": (5, 10, 1e-10, 0)}[tag]
    run = orc.gmres(A, G[p + "b"], "cgs1_ghysels", m, R, tol, diag_every=diag)
    curve = G[p + "curve"]
    assert len(run.curve) == len(curve) and run.outcome == str(G[p + "outcome"])
    assert np.max(np.abs(np.array(run.curve) - curve) / np.maximum(curve, 1e-300)) <= 1e-9
    assert [e[1] for e in run.ledger.events] == list(G[p + "ev_kind"])


JACOBI_METHODS = ["one_sync_mgs", "two_sync_cgs2", "mgs_l1", "cgs2", "pipeline2", "cgs1_ghysels"]


@pytest.mark.parametrize("meth", JACOBI_METHODS)
def test_jacobi_matches_reference(meth):
    """The oracle's right-Jacobi branch (oracle/lowsync_oracle.py, gmres.py:106-126,
    264-265, 277, 297) against the reference run on a varying-diagonal matrix
    (tests/golden/make_golden.py jacobi)."""
    G = _load("jacobi.npz")
    A = orc.Csr(int(G["row_ptr"].size - 1), int(G["row_ptr"].size - 1), G["row_ptr"], G["col_idx"],
                G["values"])
    run = orc.gmres(A, G["b"], meth, 10, 200, 1e-10, jacobi=True)
    p = meth + "__"
    curve = G[p + "curve"]
    assert len(run.curve) == len(curve) and run.outcome == str(G[p + "outcome"])
    assert run.cycle_starts == list(G[p + "cycle_starts"])
    np.testing.assert_allclose(run.curve, curve, rtol=1e-10, atol=0)
    ev = run.ledger.events
    assert [e[1] for e in ev] == list(G[p + "ev_kind"])
    assert [e[2] for e in ev] == list(G[p + "ev_count"])
    assert [e[0] for e in ev] == list(G[p + "ev_iter"])
    np.testing.assert_allclose(run.x, G[p + "x"], rtol=1e-9, atol=1e-12)
