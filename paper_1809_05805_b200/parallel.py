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
