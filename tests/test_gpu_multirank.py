"""Multi-rank path with the real kernels on one GPU: P ranks run as threads
(parallel.ThreadComm), each on its own stream, exchanging the per-iteration
partials (all-gather + fixed-order sum) and the ghost z-planes through
device memory exactly as the NCCL communicator does across GPUs.  The
row-partitioned solve must reproduce the reference's golden history."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1809_05805_b200 as P
    return P


def _rank(comm, dims, meth, m, restarts, tol):
    import paper_1809_05805_b200 as P
    from paper_1809_05805_b200.parallel import local_rhs, slab_problem
    op, ng = slab_problem(dims, comm)
    b = local_rhs(dims, comm, 42)
    led = P.ReductionLedger()
    cfg = P.GmresConfig(restart_m=m, max_restarts=restarts, rel_tol=tol, method=meth)
    x, h = P.gmres.solve_distributed(op, b, comm, ng, config=cfg, ledger=led)
    ev = [(e.iteration, e.kind, e.scalar_count, e.overlap_eligible) for e in led.events]
    return x, h.implicit_curve(), h.outcome, ev, h.final_true_rel_res, list(h.cycle_starts)


@pytest.mark.parametrize("ranks,meth", [(2, "one_sync_mgs"), (4, "one_sync_mgs"),
                                        (2, "two_sync_cgs2"), (2, "mgs_l1"), (2, "cgs2"),
                                        (3, "pipeline2")])
def test_slab_partition_reproduces_reference(P, ranks, meth):
    from paper_1809_05805_b200.parallel import run_threads
    G = np.load(os.path.join(GOLD, "laplace3d32.npz"))
    out = run_threads(ranks, _rank, (32, 32, 32), meth, 50, 50, 1e-6)
    c0 = out[0][1]
    for r in range(1, ranks):   # replicated small state: identical on every rank
        assert np.array_equal(out[r][1], c0)
        assert out[r][3] == out[0][3]
    cr = G[meth + "__curve"]
    assert len(c0) == len(cr)
    assert np.max(np.abs(c0 - cr) / cr) <= 1e-10
    assert out[0][2] == str(G[meth + "__outcome"])
    assert out[0][5] == list(G[meth + "__cycle_starts"])
    assert [e[1] for e in out[0][3]] == list(G[meth + "__ev_kind"])
    assert [e[2] for e in out[0][3]] == list(G[meth + "__ev_count"])
    x = np.concatenate([o[0] for o in out])
    xr = G[meth + "__x"]
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)


def _rank_scaled(comm, dims, scale):
    import paper_1809_05805_b200 as P
    from paper_1809_05805_b200.parallel import local_rhs, slab_problem
    op, ng = slab_problem(dims, comm)
    b = local_rhs(dims, comm, 42) * scale
    cfg = P.GmresConfig(restart_m=50, max_restarts=50, rel_tol=1e-6, method="one_sync_mgs")
    x, h = P.gmres.solve_distributed(op, b, comm, ng, config=cfg)
    return x, h.implicit_curve(), h.outcome


@pytest.mark.parametrize("scale", [2.0 ** 600, 2.0 ** -600])
def test_slab_partition_restart_norm_out_of_range(P, scale):
    """|b| ~ 2^±600: the restart norm's sum of squares over- or underflows
    unless rescaled; across ranks the exact power-of-two rescale needs the
    global max|r| (second all-gather).  Scaling b by a power of two scales
    every quantity exactly, so the history equals the unscaled golden one."""
    from paper_1809_05805_b200.parallel import run_threads
    G = np.load(os.path.join(GOLD, "laplace3d32.npz"))
    out = run_threads(2, _rank_scaled, (32, 32, 32), scale)
    c0 = out[0][1]
    assert np.array_equal(out[1][1], c0)
    cr = G["one_sync_mgs__curve"]
    assert len(c0) == len(cr) and np.max(np.abs(c0 - cr) / cr) <= 1e-10
    assert out[0][2] == str(G["one_sync_mgs__outcome"])
    x = np.concatenate([o[0] for o in out]) / scale
    xr = G["one_sync_mgs__x"]
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)
