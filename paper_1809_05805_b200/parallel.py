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

import ctypes as C
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

    def _staged(self):
        """gloo moves CPU tensors only: CUDA buffers are staged through host
        copies (validation of this class with the real kernels on one GPU;
        NCCL takes the device buffers directly)."""
        return dist.get_backend(self.group) == "gloo"

    def allgather(self, local, out):
        """out[q*len(local):(q+1)*len(local)] = rank q's `local` (one collective)."""
        if self._staged() and local.is_cuda:
            h = out.cpu()
            dist.all_gather_into_tensor(h, local.cpu(), group=self.group)
            out.copy_(h)
            return
        dist.all_gather_into_tensor(out, local, group=self.group)

    def halo(self, vec, off, n, plane):
        """Fill the ghost planes around vec[off:off+n] from the z-neighbours:
        vec[off-plane:off] <- last plane of rank-1, vec[off+n:off+n+plane]
        <- first plane of rank+1 (one batched send/recv group)."""
        ops = []
        r, s = self.rank, self.size
        staged = self._staged() and vec.is_cuda
        bufs = []

        def sbuf(t):
            if not staged:
                return t
            h = t.cpu()
            bufs.append((h, t))
            return h
        if r > 0:
            ops.append(dist.P2POp(dist.isend, sbuf(vec[off:off + plane]), r - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, sbuf(vec[off - plane:off]), r - 1, self.group))
        if r < s - 1:
            ops.append(dist.P2POp(dist.isend, sbuf(vec[off + n - plane:off + n]), r + 1,
                                  self.group))
            ops.append(dist.P2POp(dist.irecv, sbuf(vec[off + n:off + n + plane]), r + 1,
                                  self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for h, t in bufs:
            t.copy_(h)

    def exchange(self, obj):
        """Host-side all-gather of a picklable object (setup only)."""
        out = [None] * self.size
        dist.all_gather_object(out, obj, group=self.group)
        return out

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

    def exchange(self, obj):
        g = self.g
        g.barrier.wait()
        g.slots[self.rank] = (obj, None)
        g.barrier.wait()
        out = [x[0] for x in g.slots]
        g.barrier.wait()
        return out

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


def run_threads(size, fn, *args, peer=False):
    """Run fn(comm, *args) on `size` in-process ranks; returns per-rank
    results.  peer=True hands each rank a PeerComm over the ThreadComm (the
    device-side exchange kernels, peers' buffers as plain pointers).  On one
    device the ranks' streams must not share a hardware work queue (a
    spinning exchange kernel would block the kernels it waits for): set
    CUDA_DEVICE_MAX_CONNECTIONS=32 before CUDA initialises (tests/conftest.py
    does)."""
    if peer and size > 1 and int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8")) < 2 * size:
        import warnings
        warnings.warn("run_threads(peer=True) on one device wants CUDA_DEVICE_MAX_CONNECTIONS >= "
                      "2 x ranks set before CUDA initialises; exchanges may time out")
    if peer and torch.cuda.is_available():
        # ranks sharing the device must not hit a device-wide synchronisation
        # while a peer's exchange kernel spins: cudaFree (the caching
        # allocator releasing cached segments to satisfy a new allocation) is
        # one.  Start from an empty cache so the ranks' allocations are fresh
        # cudaMallocs, and drop a cached single-rank solver engine.
        import gc
        from . import gmres as _gm
        _gm.clear_engine_cache()
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    import threading
    grp = ThreadGroup(size)
    out = [None] * size
    err = []

    def body(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                c = ThreadComm(grp, r)
                if peer:
                    c = PeerComm(c, ipc=False)
                out[r] = fn(c, *args)
                if peer:
                    c.close()
            s.synchronize()
        except BaseException as e:  # pragma: no cover
            if os.environ.get("LSB_RANK_ERRORS"):
                import sys
                import traceback
                sys.stderr.write(f"rank {r}: " + traceback.format_exc())
                sys.stderr.flush()
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


class PeerUnavailable(RuntimeError):
    """Peer mappings (CUDA IPC / P2P) are not available on every rank."""


class _Reg:
    __slots__ = ("base", "span", "ld", "off", "n", "ptrs")


class PeerComm:
    """The solver's two exchange steps as device kernels over peer memory
    (csrc/peer.cu, lsb_peer_allgather / lsb_peer_halo): every rank's
    mailbox, signal words and halo target vectors are mapped into every
    rank (CUDA IPC between processes -- NVLink/NVSwitch P2P between GPUs --
    or plain pointers between ranks sharing a process), the exchanges signal
    with epochs kept on the device, so a multi-rank cycle needs no host
    call per iteration and is captured in a CUDA graph like the one-GPU
    cycle.  The host communicator `host` (Comm over torch.distributed, or
    ThreadComm) is used only at setup and for host-side scalars/barriers.

    Same interface as Comm for the engine: allgather(local, out) and
    halo(vec, off, n, plane); plus register(...) so that halo() can address
    the neighbours' copy of a vector, and check() to raise on a timeout."""

    graph_safe = True

    def __init__(self, host, ipc=True, slot=None, timeout_s=None):
        from . import _abi
        self.host = host
        self.rank, self.size = host.rank, host.size
        if self.size > _abi.PEER_MAX:
            raise ValueError(f"at most {_abi.PEER_MAX} ranks")
        self.ipc = bool(ipc)
        self.lib = _abi.load()
        self._opened = {}
        dev = torch.device("cuda", torch.cuda.current_device())
        self.slot = int(slot or 2 * 130 + 8)          # 2 cap + nonfinite word, cap <= 130
        self.mbox = torch.zeros(2 * self.size * self.slot, dtype=torch.float64, device=dev)
        self.sig = torch.zeros(self.size + 2, dtype=torch.int64, device=dev)
        self.ctr = torch.zeros(4, dtype=torch.int64, device=dev)
        self.counter = torch.zeros(8, dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        mb, sg = self._share_checked(self.mbox), self._share_checked(self.sig)
        P = _abi.Peer()
        P.rank, P.size, P.slot = self.rank, self.size, self.slot
        if timeout_s is None:
            timeout_s = float(os.environ.get("LSB_PEER_TIMEOUT_S", "60"))
        P.timeout_ns = int(timeout_s * 1e9)
        for q in range(self.size):
            P.mbox[q], P.sig[q] = mb[q], sg[q]
        P.epoch, P.counter = self.ctr.data_ptr(), self.counter.data_ptr()
        self.P = P
        self.Pref = C.byref(P)
        self._regs = []
        self.flags = None          # the current engine's flag block (error reporting)
        self.host.barrier()

    # ------------------------------------------------------------ setup
    def _share_checked(self, t):
        """_share with failures made collective: if any rank cannot export
        or map, every rank raises PeerUnavailable at the same step (so a
        caller can fall back to the NCCL communicator consistently)."""
        err = None
        try:
            out = self._share(t)
        except Exception as e:   # noqa: BLE001 -- reported below on every rank
            out, err = None, f"rank {self.rank}: {e}"
        errs = [e for e in self.host.exchange(err) if e]
        if errs:
            self._close_mappings()
            raise PeerUnavailable("; ".join(errs))
        return out

    def selftest(self):
        """One all-gather of the rank ids (collective); raises PeerUnavailable
        on every rank if any rank's exchange failed or timed out."""
        loc = torch.full((4,), float(self.rank), dtype=torch.float64, device=self.mbox.device)
        out = torch.zeros(4 * self.size, dtype=torch.float64, device=self.mbox.device)
        self.allgather(loc, out)
        torch.cuda.current_stream().synchronize()
        want = torch.arange(self.size, dtype=torch.float64).repeat_interleave(4)
        ok = bool(torch.equal(out.cpu(), want)) and int(self.ctr[2].item()) == 0
        if not all(self.host.exchange(ok)):
            raise PeerUnavailable("peer all-gather self-test failed")

    def _share(self, t):
        """Per-rank device pointers of the peers' copies of `t` (valid here)."""
        if not self.ipc:
            return self.host.exchange(t.data_ptr())
        from . import _abi
        h = (C.c_char * 64)()
        off = C.c_int64()
        _abi.check(self.lib.lsb_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off)),
                   "lsb_ipc_export")
        allh = self.host.exchange((bytes(h), off.value))
        out = []
        for q, (hb, o) in enumerate(allh):
            if q == self.rank:
                out.append(t.data_ptr())
                continue
            base = self._opened.get(hb)
            if base is None:
                # a failed exchange on any rank raises on every rank (the
                # handles were all published before anyone maps them)
                bp = C.c_void_p()
                _abi.check(self.lib.lsb_ipc_open(C.create_string_buffer(hb, 64), C.byref(bp)),
                           "lsb_ipc_open")
                base = self._opened[hb] = bp.value
            out.append(base + o)
        return out

    def register(self, t, off, n, ld=0):
        """Collective: make `t` (a vector with ghost padding around
        t[off:off+n], or a 2-D array of such rows ld doubles apart) a halo
        target.  Every rank registers the same buffers in the same order."""
        r = _Reg()
        r.base = t.data_ptr()
        r.span = 8 * t.numel()
        r.ptrs = self._share(t)
        info = self.host.exchange((int(ld), int(off), int(n)))
        r.ld = [i[0] for i in info]
        r.off = [i[1] for i in info]
        r.n = [i[2] for i in info]
        self._regs.append(r)
        return r

    def unregister_all(self):
        self._regs = []

    def _find(self, p):
        for r in reversed(self._regs):
            if r.base <= p < r.base + r.span:
                me = r.ld[self.rank]
                j = (p - r.base) // (8 * me) if me else 0
                return r, j
        raise KeyError("halo on a buffer that was not registered with PeerComm.register")

    # ------------------------------------------------------------ exchanges
    def allgather(self, local, out):
        L = local.numel()
        rc = self.lib.lsb_peer_allgather(self.Pref, C.c_void_p(local.data_ptr()), L,
                                         C.c_void_p(out.data_ptr()), L, self.flags,
                                         C.c_void_p(torch.cuda.current_stream().cuda_stream))
        if rc:
            from . import _abi
            _abi.check(rc, "lsb_peer_allgather")

    def halo(self, vec, off, n, plane):
        p = vec.data_ptr()
        r, j = self._find(p)
        q = self.rank
        lo_dst = hi_dst = None
        if q > 0:
            lo_dst = C.c_void_p(r.ptrs[q - 1] + 8 * (j * r.ld[q - 1] + r.off[q - 1] + r.n[q - 1]))
        if q < self.size - 1:
            hi_dst = C.c_void_p(r.ptrs[q + 1] + 8 * (j * r.ld[q + 1] + r.off[q + 1] - plane))
        rc = self.lib.lsb_peer_halo(self.Pref, C.c_void_p(p + 8 * off), lo_dst,
                                    C.c_void_p(p + 8 * (off + n - plane)), hi_dst, int(plane),
                                    self.flags, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        if rc:
            from . import _abi
            _abi.check(rc, "lsb_peer_halo")

    # ---- the ghost exchange fused into K2 / the fused K1+SpMV (one-sync)
    def halo_push(self, vec, off, n, plane):
        """lsb_halo_push for the column/vector `vec` (registered): the K2 that
        finishes it stores its first/last `plane` rows straight into the
        neighbours' ghost rows and signals them."""
        from . import _abi
        r, j = self._find(vec.data_ptr())
        q = self.rank
        hp = _abi.HaloPush()
        hp.plane = int(plane)
        if q > 0:
            hp.lo_dst = r.ptrs[q - 1] + 8 * (j * r.ld[q - 1] + r.off[q - 1] + r.n[q - 1])
            hp.sig_lo = self.P.sig[q - 1] + 8 * (self.size + 1)
        if q < self.size - 1:
            hp.hi_dst = r.ptrs[q + 1] + 8 * (j * r.ld[q + 1] + r.off[q + 1] - plane)
            hp.sig_hi = self.P.sig[q + 1] + 8 * self.size
        hp.epoch = self.ctr.data_ptr() + 8
        hp.counter = self.counter.data_ptr()
        return hp

    def halo_wait(self):
        """lsb_halo_wait: this rank's own halo signal words and epoch."""
        from . import _abi
        hw = _abi.HaloWait()
        base = self.sig.data_ptr()
        if self.rank > 0:
            hw.sig_lo = base + 8 * self.size
        if self.rank < self.size - 1:
            hw.sig_hi = base + 8 * (self.size + 1)
        hw.epoch = self.ctr.data_ptr() + 8
        hw.timeout_ns = self.P.timeout_ns
        hw.flags = self.flags.value if self.flags is not None else None
        return hw

    def check(self):
        """Raise if an exchange kernel timed out (a peer died or diverged)."""
        if int(self.ctr[2].item()):
            raise RuntimeError("peer exchange timed out (a rank stopped participating)")

    # ------------------------------------------------------------ host side
    def exchange(self, obj):
        return self.host.exchange(obj)

    def max_scalar(self, v):
        return self.host.max_scalar(v)

    def barrier(self):
        torch.cuda.current_stream().synchronize()
        self.host.barrier()

    def _close_mappings(self):
        for base in self._opened.values():
            self.lib.lsb_ipc_close(C.c_void_p(base))
        self._opened = {}

    def close(self):
        torch.cuda.synchronize()
        self.host.barrier()
        self._close_mappings()
        self._regs = []


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


def csr_row_block(A, comm):
    """This rank's contiguous row block of a global CSR matrix (SURVEY
    §8(e): CSR SpMV partitions by rows) -> (operator,
    n_global, row0).  Ghost columns are the `halo` rows just below and above
    the block -- halo = the farthest any rank's columns reach outside its own
    block, agreed by all ranks -- which the engine's halo exchange copies
    from the neighbouring blocks (banded matrices: stencils in CSR form,
    their 27-point convection-diffusion of config 5).  Raises ValueError on
    every rank if the band reaches past a neighbouring block."""
    from .operators import CsrOperator
    n = int(A.n_rows)
    r0, nl = slab_bounds(n, comm.size, comm.rank)
    rp = np.asarray(A.row_ptr, dtype=np.int64)
    lo, hi = int(rp[r0]), int(rp[r0 + nl])
    cols = np.asarray(A.col_idx[lo:hi], dtype=np.int64)
    reach = 0
    if cols.size:
        reach = max(0, r0 - int(cols.min()), int(cols.max()) - (r0 + nl - 1))
    halo = int(comm.max_scalar(float(reach)))
    smallest = -comm.max_scalar(-float(nl))
    if comm.size > 1 and halo > smallest:
        raise ValueError(f"matrix band ({halo} rows) reaches past a neighbouring row block "
                         f"({int(smallest)} rows): use fewer ranks")
    op = CsrOperator.row_block(rp[r0:r0 + nl + 1] - lo, cols, np.asarray(A.values[lo:hi]), r0,
                               halo if comm.size > 1 else 0)
    return op, n, r0
