"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path's host
logic: z-slab bounds, ghost-plane exchange, the all-gather + fixed-order sum
that replaces each reduction, and an end-to-end row-partitioned one-sync
GMRES built from those pieces (numpy per rank, as the checker) that must
reproduce the single-process oracle's iteration count and residual history.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lowsync_oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, world=2, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q, args)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = [q.get() for _ in range(world)]
    for r in res:
        if isinstance(r, BaseException) or (isinstance(r, tuple) and r and r[0] == "error"):
            raise AssertionError(r)
    return sorted(res, key=lambda t: t[0])


def _entry(fn, rank, world, port, q, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        from paper_1809_05805_b200.parallel import Comm
        comm = Comm.init("gloo")
        out = fn(comm, *args)
        q.put((rank, out))
        comm.close()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(("error", rank, traceback.format_exc()))


# ---------------------------------------------------------------- pieces
def _halo_and_gather(comm):
    from paper_1809_05805_b200.parallel import slab_bounds
    nx = ny = 3
    nz = 7
    plane = nx * ny
    z0, nzl = slab_bounds(nz, comm.size, comm.rank)
    n = nzl * plane
    off = plane + (plane % 2)
    vec = torch.full((off + n + plane + 2,), -1.0, dtype=torch.float64)
    glob = torch.arange(nz * plane, dtype=torch.float64)
    vec[off:off + n] = glob[z0 * plane:(z0 + nzl) * plane]
    comm.halo(vec, off, n, plane)
    lo = vec[off - plane:off].tolist() if z0 > 0 else None
    hi = vec[off + n:off + n + plane].tolist() if z0 + nzl < nz else None
    loc = torch.tensor([comm.rank + 0.5, 10.0 * comm.rank], dtype=torch.float64)
    out = torch.zeros(2 * comm.size, dtype=torch.float64)
    comm.allgather(loc, out)
    return (z0, nzl, lo, hi, out.tolist())


def test_halo_exchange_and_allgather_order():
    res = _spawn(_halo_and_gather)
    plane = 9
    (r0, (z0a, na, loa, hia, ga)), (r1, (z0b, nb, lob, hib, gb)) = res
    assert (z0a, na, z0b, nb) == (0, 4, 4, 3)
    glob = np.arange(63.0)
    assert loa is None and hib is None
    assert hia == glob[4 * plane:5 * plane].tolist()       # first plane of rank 1
    assert lob == glob[3 * plane:4 * plane].tolist()       # last plane of rank 0
    assert ga == gb == [0.5, 0.0, 1.5, 10.0]


def _rhs_slice(comm):
    from paper_1809_05805_b200.parallel import local_rhs
    return local_rhs((4, 3, 5), comm, 42).tolist()


def test_local_rhs_slices_reassemble_global():
    res = _spawn(_rhs_slice)
    b = np.concatenate([np.array(r[1]) for r in res])
    assert np.array_equal(b, orc.rhs_random(60, 42))


# ---------------------------------------------------------------- partitioned solve
def _partitioned_one_sync(comm, N, m, restarts, tol):
    """Row-partitioned one-sync GMRES(m) with exactly the device path's
    communication schedule: per iteration one halo exchange (SpMV input) and
    ONE all-gather of the local [Q^T u, Q^T w] partials, summed in rank
    order; small state replicated.  numpy stands in for the kernels."""
    from paper_1809_05805_b200.parallel import local_rhs, slab_bounds
    dims = (N, N, N)
    A = orc.laplace3d(N)
    plane = N * N
    z0, nzl = slab_bounds(N, comm.size, comm.rank)
    r0, r1 = z0 * plane, (z0 + nzl) * plane
    n = r1 - r0
    lo = r0 - plane if z0 > 0 else r0
    rows = slice(r0, r1)
    ptr = A.row_ptr[r0:r1 + 1] - A.row_ptr[r0]
    cols = A.col_idx[A.row_ptr[r0]:A.row_ptr[r1]] - lo
    vals = A.values[A.row_ptr[r0]:A.row_ptr[r1]]
    Aloc = orc.Csr(n, 0, ptr, cols, vals)
    off = r0 - lo

    def spmv(v):
        ext = torch.zeros(off + n + plane + 2, dtype=torch.float64)
        ext[off:off + n] = torch.as_tensor(v)
        comm.halo(ext, off, n, plane)
        return orc.spmv(Aloc, ext.numpy()[: off + n + (plane if z0 + nzl < N else 0)])

    def allsum(vec):
        loc = torch.as_tensor(np.ascontiguousarray(vec, dtype=np.float64))
        out = torch.zeros(loc.numel() * comm.size, dtype=torch.float64)
        comm.allgather(loc, out)
        parts = out.view(comm.size, -1).numpy()
        acc = parts[0].copy()
        for q in range(1, comm.size):
            acc = acc + parts[q]
        return acc

    def gnorm(v):
        return float(np.sqrt(allsum(np.array([np.dot(v, v)]))[0]))

    b = local_rhs(dims, comm, 42)
    x = np.zeros(n)
    r = b - spmv(x)
    beta = gnorm(r)
    denom, target = beta, tol * beta
    curve, cycles = [], 0
    n_global = N ** 3
    for _ in range(restarts):
        cycles += 1
        V = np.zeros((n, m + 2), order="F")
        F = orc.Factors(m + 2)
        st = orc.Rotations(m, beta)
        V[:, 0] = r / beta
        stop = None

        def lagged(p):
            Q, u, w = V[:, :p], V[:, p - 1], V[:, p]
            G = allsum(np.concatenate([Q.T @ u, Q.T @ w])).reshape(2, p).T
            bsq = G[p - 1, 0]
            bt = np.sqrt(bsq) if bsq > 0 else 0.0
            orc.breakdown_check(n_global, bt, F.R[: p - 1, p - 1], 1.0, p - 1)
            V[:, p - 1] = u / bt
            F.R[p - 1, p - 1] = bt
            if p >= 2:
                F.T[: p - 1, p - 1] = -(F.T[: p - 1, : p - 1] @ (G[: p - 1, 0] / bt))
            F.T[p - 1, p - 1] = 1.0
            y = G[:, 1].copy()
            y[p - 1] /= bt
            c = F.T[:p, :p].T @ y / bt
            V[:, p] = V[:, p] / bt - V[:, :p] @ c
            F.R[:p, p] = c

        V[:, 1] = spmv(V[:, 0])
        lagged(1)
        k = m
        for i in range(1, m + 1):
            V[:, i + 1] = spmv(V[:, i])
            lagged(i + 1)
            res = orc.givens(st, F.R[: i + 1, i], i)
            curve.append(res / denom)
            if res <= target:
                stop, k = i, i
                break
        y = orc.back_substitute(st, k)
        x = x + V[:, :k] @ y
        r = b - spmv(x)
        beta = gnorm(r)
        if stop is not None or beta <= target:
            break
    return curve, cycles


def test_partitioned_one_sync_matches_single_process_oracle():
    N, m, restarts, tol = 12, 20, 20, 1e-8
    res = _spawn(_partitioned_one_sync, 2, N, m, restarts, tol)
    c0, c1 = np.array(res[0][1][0]), np.array(res[1][1][0])
    assert np.array_equal(c0, c1)          # replicated small state: identical bits on all ranks
    ref = orc.gmres(orc.laplace3d(N), orc.rhs_random(N ** 3, 42), "one_sync_mgs", m, restarts, tol)
    cr = np.array(ref.curve)
    assert len(c0) == len(cr)
    assert np.max(np.abs(c0 - cr) / cr) <= 1e-10
