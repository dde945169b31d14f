"""Row-partitioned (z-slab) multi-GPU plumbing: one process per GPU,
torch.distributed (NCCL on GPUs, gloo on CPU for tests).

The paper's model: rows of A, of every basis vector and
of x/b are split into contiguous blocks; each reduction-shaped operation
becomes one global collective.  Here every per-iteration reduction is ONE
all-gather of the ranks' local partial vectors followed by a fixed-order sum
on device (so every rank holds bit-identical small state, independent of the
collective's algorithm), and the stencil SpMV needs one ghost z-plane from
each neighbour (NCCL send/recv, batched).
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


class Comm:
    """The two collectives the solver needs, plus timing helpers."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    @classmethod
    def init(cls, backend=None):
        if not dist.is_initialized():
            backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
            kw = {}
            if backend == "nccl":
                kw["device_id"] = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
            dist.init_process_group(backend=backend, **kw)
        return cls()

    def allgather(self, local, out):
        """out[q*len(local):(q+1)*len(local)] = rank q's `local` (one collective)."""
        dist.all_gather_into_tensor(out, local, group=self.group)

    def halo(self, vec, off, n, plane):
        """Fill the ghost planes around vec[off:off+n] from the z-neighbours:
        vec[off-plane:off] <- last plane of rank-1, vec[off+n:off+n+plane]
        <- first plane of rank+1 (one batched send/recv group)."""
        ops = []
        r, s = self.rank, self.size
        if r > 0:
            ops.append(dist.P2POp(dist.isend, vec[off:off + plane], r - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, vec[off - plane:off], r - 1, self.group))
        if r < s - 1:
            ops.append(dist.P2POp(dist.isend, vec[off + n - plane:off + n], r + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, vec[off + n:off + n + plane], r + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def max_scalar(self, v):
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def barrier(self):
        dist.barrier(group=self.group)

    def close(self):
        if dist.is_initialized():
            dist.destroy_process_group()


class ThreadGroup:
    """Shared state of P in-process ranks (one Python thread per rank)."""

    def __init__(self, size):
        import threading
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = [None] * size
        self.done = [None] * size


class ThreadComm:
    """Single-process communicator: P ranks = P threads, each issuing its
    kernels on its own CUDA stream (same or different devices).  A
    collective publishes the rank's buffer with a CUDA event, meets the
    other ranks at a host barrier, copies the peers' data device-to-device
    after waiting on their events, and fences again so no rank overwrites a
    published buffer before every peer has copied it.  Same interface and
    data movement as Comm, so the engine runs unchanged; used to exercise
    the multi-rank kernels (g_parts > 1, ghost planes, slab operators) on a
    single GPU, and usable as a one-process multi-GPU driver."""

    def __init__(self, group, rank):
        self.g = group
        self.rank = rank
        self.size = group.size

    def _exchange(self, publish, consume):
        g, r = self.g, self.rank
        ev = torch.cuda.Event()
        ev.record()
        g.slots[r] = (publish, ev)
        g.barrier.wait()
        st = torch.cuda.current_stream()
        for q in range(self.size):
            st.wait_event(g.slots[q][1])
        consume(g.slots)
        ev2 = torch.cuda.Event()
        ev2.record()
        g.done[r] = ev2
        g.barrier.wait()
        for q in range(self.size):
            st.wait_event(g.done[q])
        g.barrier.wait()   # slots may be reused only after everyone fenced

    def allgather(self, local, out):
        L = local.numel()

        def consume(slots):
            for q in range(self.size):
                out[q * L:(q + 1) * L].copy_(slots[q][0], non_blocking=True)
        self._exchange(local, consume)

    def halo(self, vec, off, n, plane):
        r, s = self.rank, self.size
        pub = (vec[off:off + plane], vec[off + n - plane:off + n])

        def consume(slots):
            if r > 0:
                vec[off - plane:off].copy_(slots[r - 1][0][1], non_blocking=True)
            if r < s - 1:
                vec[off + n:off + n + plane].copy_(slots[r + 1][0][0], non_blocking=True)
        self._exchange(pub, consume)

    def max_scalar(self, v):
        g = self.g
        g.slots[self.rank] = (float(v), None)
        g.barrier.wait()
        m = max(x[0] for x in g.slots)
        g.barrier.wait()
        return m

    def barrier(self):
        self.g.barrier.wait()

    def close(self):
        pass


def run_threads(size, fn, *args):
    """Run fn(comm, *args) on `size` in-process ranks; returns per-rank results."""
    import threading
    grp = ThreadGroup(size)
    out = [None] * size
    err = []

    def body(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(ThreadComm(grp, r), *args)
            s.synchronize()
        except BaseException as e:  # pragma: no cover
            err.append(e)
            grp.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


def slab_bounds(nz, size, rank):
    """Planes [z0, z0+nzl) of rank `rank` (contiguous, as equal as possible)."""
    base, extra = divmod(nz, size)
    z0 = rank * base + min(rank, extra)
    return z0, base + (1 if rank < extra else 0)


def slab_problem(dims, comm, kind="laplace3d", pe=0.5):
    """This rank's z-slab of the global stencil operator -> (operator, n_global)."""
    from .operators import StencilOperator, convdiff27, laplace3d
    nx, ny, nz = dims
    S = laplace3d(0, dims) if kind == "laplace3d" else convdiff27(0, pe, dims)
    z0, nzl = slab_bounds(nz, comm.size, comm.rank)
    return StencilOperator(S, z0=z0, nz_local=nzl), nx * ny * nz


def local_rhs(dims, comm, seed):
    """This rank's rows of gen_rhs('random', A_global, seed): the global
    unit-norm seeded Gaussian, sliced (identical bits to the 1-GPU b)."""
    nx, ny, nz = dims
    n = nx * ny * nz
    b = np.random.default_rng(seed).standard_normal(n)
    b /= np.linalg.norm(b)
    z0, nzl = slab_bounds(nz, comm.size, comm.rank)
    plane = nx * ny
    return np.ascontiguousarray(b[z0 * plane:(z0 + nzl) * plane])
