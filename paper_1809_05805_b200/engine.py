"""Device-resident GMRES(m) cycle engine.

One restart cycle of the reference driver (gmres.py:309-466) is enqueued as
a fixed sequence of liblsb200 launches per Arnoldi iteration:

  one_sync_mgs / pipeline2   SpMV -> K1 lagged_reduce -> [allgather] -> K5 -> K2
  two_sync_cgs2              SpMV -> K1 -> [ag] -> K5a -> K3 (= K2 + K1') -> [ag] -> K5b -> K4
  mgs_l1                     SpMV -> (p+1) x K8 pass -> [ag each] -> norm -> K5d -> scale
  cgs2                       SpMV -> K1' -> coef -> project -> K1' -> coef -> project+norm -> K5d -> scale

Convergence, breakdown, the Givens fold and the back-substitution are
device-side (flags block), so a whole cycle -- including the x update and
the restart residual/norm -- is launch-only: no host synchronisation inside
a cycle.  On one GPU the cycle is captured once as a CUDA graph and
replayed; with a communicator (multi-GPU) it is issued eagerly.  The host
reads one small report (flags, residuals, scalars) per cycle.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import threading

import numpy as np
import torch

from . import _abi
from . import _dev as D
from .operators import device_operator

LAGGED = ("one_sync_mgs", "two_sync_cgs2", "pipeline2")
K3_MAX_COLS = 110   # lsb_lagged_update_reduce stages p + 1 <= 110 columns
# one-cluster persistent cycle (lsb_cycle_persistent): launch-bound sizes
# whose basis fits the cluster's shared memory (lsb_cycle_persistent_fits)
PERSIST_METHODS = ("one_sync_mgs", "pipeline2")
DIRECT = ("mgs_l1", "cgs2")


class CycleReport:
    """Host copy of what one cycle produced."""

    __slots__ = ("stop_iter", "status", "broke_iter", "k", "nonfinite", "restart_ok",
                 "comm_error", "res", "scal", "true_res")

    def __init__(self, flags, res, scal, true_res=None):
        self.stop_iter, self.status, self.broke_iter, self.k, self.nonfinite, self.restart_ok = (
            int(v) for v in flags[:6])
        self.comm_error = int(flags[6]) if len(flags) > 6 else 0
        self.res = res
        self.scal = scal
        self.true_res = true_res


_CANON7 = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]


def _canonical7(op):
    """7-point stencil in laplace3d's column order, nx even, unscaled:
    eligible for the fused K1+SpMV kernel (tile.cuh canonical7)."""
    c = getattr(op, "c", None)
    if not isinstance(c, _abi.Stencil) or c.noff != 7 or c.col_scale or c.nx % 2 or c.nx < 4:
        return False
    return [(c.dx[k], c.dy[k], c.dz[k]) for k in range(7)] == _CANON7


def _timing_event():
    """Timing event that also works inside the captured cycle graph: an
    external record becomes an event-record node, re-recorded on every
    replay (a plain record under capture is only a dependency marker)."""
    return torch.cuda.Event(enable_timing=True, external=True)


_REPORT = {}

# capture_begin registers the graph with the device's default RNG generator,
# whose graph-safe state tensors are created lazily; ranks emulated as
# threads that begin their captures at the same moment raced on that
# creation ("Expected a proper Tensor but got None", seen once in ~20 runs
# of the threaded row-block tests).  The registration is serialised; the
# captures themselves still run concurrently (thread-local capture mode).
_CAPTURE_BEGIN_LOCK = threading.Lock()


def _report_buffers(m):
    import threading
    key = (m, threading.get_ident())
    if key not in _REPORT:
        _REPORT[key] = (torch.zeros(_abi.FLAGS_INTS, dtype=torch.int32).pin_memory(),
                        torch.zeros(m + 1, dtype=D.F64).pin_memory(),
                        torch.zeros(_abi.S_COUNT, dtype=D.F64).pin_memory())
    return _REPORT[key]


class Engine:
    def __init__(self, A, m, method, rel_tol, btf=1.0, inv_diag=None, comm=None,
                 diagnostics=False, use_graph=True, n_global=None, op=None, fuse=True,
                 true_residual=False, persistent=None):
        self.dev = D.require_cuda()
        self.lib = _abi.load()
        base_op = op if op is not None else device_operator(A)
        self.method = method
        self.lagged = method in LAGGED
        self.comm = comm
        self.m = int(m)
        self.n = int(base_op.n_rows)
        self.n_global = int(n_global or self.n)
        self.cap = self.m + 2 if self.lagged else self.m + 1
        self.halo = int(getattr(base_op, "halo", 0))
        self.off = D.round_up(self.halo, 2)
        self.ld = D.round_up(self.off + self.n + self.halo, 32)
        f64 = dict(dtype=D.F64, device=self.dev)
        self.inv_diag = None
        self._peer = comm is not None and hasattr(comm, "register")
        if inv_diag is not None:
            self.inv_diag = self._vec_with_halo()
            if self._peer and self.halo:
                comm.register(self.inv_diag, self.off, self.n)
            self.inv_diag_view().copy_(torch.as_tensor(np.asarray(inv_diag), **f64)
                                       if not isinstance(inv_diag, torch.Tensor) else inv_diag)
            # the ghost entries of the scaling are exchanged by setup_exchange(),
            # once every rank's engine exists (no rank may spin on an exchange
            # while a peer still allocates: allocation can synchronise a
            # device the ranks share)
            self._setup_halo = comm is not None and self.halo
            self.op = base_op.with_scale(self.inv_diag[self.off:])
        else:
            self.op = base_op
        # true residuals use A itself (gmres.py:472, 498, 511: b - spmv(A, x));
        # only the Krylov products see the right preconditioner (gmres.py:264-265)
        self.rop = base_op
        # storage: every basis column is written before it is read; only the
        # ghost-plane padding must start at zero (Dirichlet planes never read)
        self.Vstore = torch.empty((self.cap, self.ld), **f64)
        if self.halo:
            self.Vstore[:, : self.off].zero_()
            self.Vstore[:, self.off + self.n:].zero_()
        cap, m = self.cap, self.m
        parts = comm.size if comm is not None else 1
        # the small state lives in one zeroed arena (one fill instead of a
        # dozen allocations + fills: launch-bound solves pay per call)
        sizes = [("R", (cap, cap)), ("T", (cap, cap)), ("L", (cap, cap)), ("rot", (2 * m,)),
                 ("g", (m + 1,)), ("tri", ((m + 1) * m,)), ("coef", (cap,)), ("coef2", (cap,)),
                 ("Gloc", (2 * cap,)), ("scal", (_abi.S_COUNT,)), ("res", (m + 1,)),
                 ("flags", ((_abi.FLAGS_INTS + 1) // 2,))]
        if parts > 1:
            sizes += [("G", (parts * 2 * cap,)), ("Gloc2", (2,)), ("G2", (parts * 2,))]
        if diagnostics:
            sizes.append(("gram", (cap, cap)))
        if true_residual:
            sizes += [("ytrial", (cap,)), ("true_res", (m + 1,))]
        offs, tot = [], 0
        for _, shp in sizes:
            offs.append(tot)
            tot += D.round_up(math.prod(shp), 2)
        self._arena = torch.zeros(tot, **f64)
        for (name, shp), o in zip(sizes, offs):
            setattr(self, name, self._arena[o:o + math.prod(shp)].view(shp))
        self.flags = self.flags.view(torch.int32)[:_abi.FLAGS_INTS]
        if parts == 1:
            self.G = self.Gloc
        if not diagnostics:
            self.gram = None
        self.ws = D.Workspace(cap, self.dev)
        self.x = self._vec_with_halo()
        if self._peer:
            comm.flags = C.c_void_p(self.flags.data_ptr())
            if self.halo:
                comm.register(self.Vstore, self.off, self.n, ld=self.ld)
                comm.register(self.x, self.off, self.n)
        self.b = torch.empty(self.n, **f64)       # uploaded before every read
        self.rbuf = torch.empty(self.n, **f64)    # residual: written before read
        self.diagnostics = diagnostics
        # true-residual probe buffers (true_residual_every > 0)
        self.true_residual = bool(true_residual)
        if self.true_residual:
            self.xt = self._vec_with_halo()
            if self._peer and self.halo:
                comm.register(self.xt, self.off, self.n)
            self.rtrial = torch.zeros(self.n, **f64)
            self.h_true = torch.zeros(m + 1, dtype=D.F64).pin_memory()
        self.S = _abi.Arnoldi(
            V=self.Vstore.data_ptr() + 8 * self.off, ld=self.ld, n=self.n, n_global=self.n_global,
            cap=cap, m=m, R=self.R.data_ptr(), T=self.T.data_ptr(), L=self.L.data_ptr(),
            rot=self.rot.data_ptr(), g=self.g.data_ptr(), tri=self.tri.data_ptr(),
            coef=self.coef.data_ptr(), coef2=self.coef2.data_ptr(), G=self.G.data_ptr(),
            g_parts=parts, g_stride=2 * cap, Gloc=self.Gloc.data_ptr(), scal=self.scal.data_ptr(),
            res=self.res.data_ptr(), flags=self.flags.data_ptr(),
            ws=_abi.Workspace(self.ws.partial.data_ptr(), self.ws.counter.data_ptr(), 0, 0))
        self.Sref = C.byref(self.S)
        self.scal[_abi.S_RELTOL] = float(rel_tol)
        self.scal[_abi.S_BTF] = float(btf)
        # host report buffers (pinned, cached across engines of the same m)
        self.h_flags, self.h_res, self.h_scal = _report_buffers(m)
        # multi-rank: capturable when the exchanges are device kernels (PeerComm)
        self.use_graph = use_graph and (comm is None or getattr(comm, "graph_safe", False))
        self.graph = None
        self.cycles_run = 0
        self.launches_per_cycle = 0
        self._count = 0
        self.timer = None   # list -> CUDA events around K1/K2/SpMV launches (bench.py)
        # fuse the 7-point SpMV into K1 when the operator allows it
        self.fused7 = bool(fuse) and self.lagged and _canonical7(self.op) and self.n % 2 == 0 \
            and self.cap - 1 <= 128
        # classical CGS2: z = A v_{i-1} and the first pass's Q^T z in one pass
        # (the lagged kernel with u = v_{i-1}, the last column of Q = V[:, :i])
        self.fused7_direct = bool(fuse) and method == "cgs2" and _canonical7(self.op) \
            and self.n % 2 == 0 and self.cap <= 128 \
            and os.environ.get("LSB_FUSE_DIRECT", "1") != "0"
        # cgs1_ghysels: z = A v_{i-1} and Q^T z in one pass the same way
        self.fused7_ghysels = bool(fuse) and method == "cgs1_ghysels" and _canonical7(self.op) \
            and self.n % 2 == 0 and self.cap <= 128 \
            and os.environ.get("LSB_FUSE_DIRECT", "1") != "0"
        # two-sync: fuse the first projection with the second reduction (K3)
        self.fuse_k3 = bool(fuse)
        # launch-bound sizes: the whole lagged cycle as one cluster launch
        self.pcsr = None
        env = os.environ.get("LSB_PERSISTENT")
        want = persistent if persistent is not None else (None if env is None else env != "0")
        if want is not False and method in PERSIST_METHODS and comm is None \
                and not diagnostics and not self.true_residual \
                and self.lib.lsb_cycle_persistent_fits(self.n, self.cap):
            self.pcsr = self._persist_csr(base_op)
        self.persistent = self.pcsr is not None
        # above one cluster, while the basis still sits in L2: the whole
        # cycle's iterations as one cooperative launch over every SM
        # (lsb_cycle_grid; LSB_GRID_CYCLE=0 or LSB_PERSISTENT=0 disables)
        self.gcsr = None
        if not self.persistent and want is not False and method in PERSIST_METHODS \
                and comm is None and not diagnostics and not self.true_residual \
                and os.environ.get("LSB_GRID_CYCLE", "1") != "0" \
                and self.lib.lsb_cycle_grid_fits(self.n, self.cap):
            self.gcsr = self._persist_csr(base_op)
        self.grid_cycle = self.gcsr is not None
        # multi-rank fused path: the ghost exchange rides on K2 (push) and the
        # fused K1+SpMV (interior tiles first, wait before boundary tiles)
        # (one_sync_mgs only: with pipeline2's side-stream settle the gate of
        # an iteration closes at a different point of the kernel sequence on
        # each rank; the separate halo kernel, never gated, keeps it simple)
        self.push_halo = bool(self._peer and self.halo and self.fused7
                              and method == "one_sync_mgs"
                              and not self.true_residual
                              and os.environ.get("LSB_HALO_PUSH", "1") != "0")
        self._keep = []
        self._hwait = comm.halo_wait() if self.push_halo else None

    def reset(self, rel_tol, btf):
        """Fresh small state for another solve on the same operator (the
        engine cache in gmres.py): one fill of the arena, the tolerances;
        storage, registrations and the captured cycle graph are kept."""
        self._arena.zero_()
        self.scal[_abi.S_RELTOL] = float(rel_tol)
        self.scal[_abi.S_BTF] = float(btf)
        if self._peer:
            self.comm.flags = C.c_void_p(self.flags.data_ptr())

    def setup_exchange(self):
        """Exchanges the engine needs before its first cycle (multi-rank:
        the ghost entries of the Jacobi scaling); call on every rank after
        all ranks have built their engines."""
        if getattr(self, "_setup_halo", False):
            self.comm.halo(self.inv_diag, self.off, self.n, self.halo)
            self._setup_halo = False

    def _persist_csr(self, base_op):
        """The operator as device CSR (bitwise the same SpMV), column-scaled
        like self.op under the Jacobi preconditioner; None if unavailable."""
        from .operators import CsrOperator, StencilOperator
        if isinstance(base_op, StencilOperator) and not base_op.halo:
            csr = base_op.stencil.device_csr()
        elif isinstance(base_op, CsrOperator) and base_op.c.x_lo == 0:
            csr = base_op
        else:
            return None
        if self.inv_diag is not None:
            csr = csr.with_scale(self.inv_diag[self.off:])
        return csr

    # ---------------------------------------------------------------- helpers
    def _vec_with_halo(self):
        return torch.zeros(self.off + self.n + self.halo + 2, dtype=D.F64, device=self.dev)

    def inv_diag_view(self):
        return self.inv_diag[self.off:self.off + self.n]

    def x_view(self):
        return self.x[self.off:self.off + self.n]

    def col_ptr(self, j):
        return C.c_void_p(self.Vstore.data_ptr() + 8 * (self.off + self.ld * j))

    def col(self, j):
        return self.Vstore[j, self.off:self.off + self.n]

    # kernel -> (bench label, index of p in the argument list)
    _TIMED = {"lsb_lagged_reduce": ("lagged_reduce", 2),
              "lsb_lagged_reduce_spmv7": ("lagged_reduce_spmv", 3),
              "lsb_lagged_update": ("lagged_update", 2),
              "lsb_lagged_update_reduce": ("lagged_update_reduce", 2)}

    def _call(self, name, *args):
        self._count += 1
        tm = self.timer is not None and name in self._TIMED
        if tm:
            e0, e1 = _timing_event(), _timing_event()
            e0.record()
        rc = getattr(self.lib, name)(*args)
        if rc:
            _abi.check(rc, name)
        if tm:
            e1.record()
            label, ip = self._TIMED[name]
            self.timer.append((label, int(args[ip]), e0, e1))

    def _gather(self, count):
        """All ranks' local reduction results -> G (one collective)."""
        if self.comm is not None:
            self.comm.allgather(self.Gloc, self.G)

    def _apply_op(self, src_tensor_base, src_ptr, dst_ptr, b_ptr, it, op=None):
        if self.comm is not None and self.halo:
            self.comm.halo(src_tensor_base[0], src_tensor_base[1], self.n, self.halo)
        self._count += 1
        tm = self.timer is not None and b_ptr is None
        if tm:
            e0, e1 = _timing_event(), _timing_event()
            e0.record()
        (op or self.op).apply_ptr(src_ptr, dst_ptr, b_ptr, C.c_void_p(self.flags.data_ptr()), it,
                                  D.stream())
        if tm:
            e1.record()
            self.timer.append(("spmv", 0, e0, e1))

    def _op_col(self, src_j, dst_j, it):
        self._apply_op((self.Vstore[src_j], self.off), self.col_ptr(src_j), self.col_ptr(dst_j),
                       None, it)

    # ---------------------------------------------------------------- phases
    def load(self, b, x0=None):
        """Place b and x0 in device memory (H2D when they live on the host)."""
        self.b.copy_(torch.as_tensor(b) if not isinstance(b, torch.Tensor) else b,
                     non_blocking=True)
        xv = self.x_view()
        if x0 is None:
            xv.zero_()
        else:
            xv.copy_(torch.as_tensor(x0) if not isinstance(x0, torch.Tensor) else x0,
                     non_blocking=True)

    def _residual_and_norm(self):
        """rbuf = b - A x; scal[RNORM] = ||rbuf|| (gmres.py:472-473 / 498-500)."""
        st = D.stream()
        xp = C.c_void_p(self.x.data_ptr() + 8 * self.off)
        self._apply_op((self.x, self.off), xp, D.ptr(self.rbuf), D.ptr(self.b), -1, op=self.rop)
        self._call("lsb_norm_partial", D.ptr(self.rbuf), self.n, D.ptr(self.Gloc), self.ws.ref(),
                   None, -1, st)
        self._gather(2)
        rn = C.c_void_p(self.scal.data_ptr() + 8 * _abi.S_RNORM)
        if self.comm is None:
            self._call("lsb_norm_finish", D.ptr(self.G), 1, self.S.g_stride, D.ptr(self.rbuf),
                       self.n, rn, self.ws.ref(), None, -1, st)
            return
        # ranks > 1: the overflow-safe rescaled pass needs the global max|r|,
        # so it is a second (2-double) all-gather; the restart norm runs
        # once per cycle
        self._call("lsb_norm_scaled_partial", D.ptr(self.G), self.S.g_parts, self.S.g_stride,
                   D.ptr(self.rbuf), self.n, D.ptr(self.Gloc2), self.ws.ref(), st)
        self.comm.allgather(self.Gloc2, self.G2)
        self._call("lsb_norm_finish_scaled", D.ptr(self.G), D.ptr(self.G2), self.S.g_parts,
                   self.S.g_stride, 2, rn, st)

    def enqueue_prologue(self):
        self._residual_and_norm()
        self._call("lsb_restart_check", self.Sref, 1, D.stream())

    def enqueue_cycle(self):
        st = D.stream()
        S = self.Sref
        self._count = 0
        self._keep = []     # launch arguments are copied at launch / capture
        # V[:,0] = r / beta (gmres.py:396 / 313), fresh small state (392-395)
        self._call("lsb_scale_div", D.ptr(self.rbuf), self.n,
                   C.c_void_p(self.scal.data_ptr() + 8 * _abi.S_RNORM), self.col_ptr(0), None, -1, st)
        self._call("lsb_cycle_begin", S, st)
        if self.persistent:       # iterations 0..m in one cluster launch
            self._call("lsb_cycle_persistent", S, C.byref(self.pcsr.c), 1, st)
        elif self.grid_cycle:     # iterations 0..m in one cooperative grid launch
            self._call("lsb_cycle_grid", S, C.byref(self.gcsr.c), 1, D.ptr(self.ws.partial),
                       int(self.ws.partial.numel()), st)
        elif self.lagged:
            self._lagged_body(st)
        else:
            self._direct_body(st)
        self._call("lsb_cycle_lsq", S, st)
        xp = C.c_void_p(self.x.data_ptr() + 8 * self.off)
        self._call("lsb_cycle_extract", S, xp,
                   None if self.inv_diag is None else C.c_void_p(self.inv_diag.data_ptr() + 8 * self.off),
                   st)
        self._residual_and_norm()
        self._call("lsb_restart_check", S, 0, st)
        self.launches_per_cycle = self._count

    def _lagged_body(self, st):
        S, m = self.Sref, self.m
        two = self.method == "two_sync_cgs2"
        # pipeline2 (gmres.py:444-462) as real overlap: the Givens fold of
        # column i-1 runs on a side stream while iteration i+1's basis passes
        # proceed; iteration i+2 waits for it (depth-2 schedule).  Arithmetic
        # identical to one_sync_mgs (tests: bitwise-equal histories).
        defer = self.method == "pipeline2" and not self.true_residual
        main = torch.cuda.current_stream()
        if defer:
            if not hasattr(self, "_side") or self._side.device != main.device:
                self._side = torch.cuda.Stream()
                self._ev_front = [torch.cuda.Event() for _ in range(m + 1)]
                self._ev_settled = [torch.cuda.Event() for _ in range(m + 1)]
            side = self._side
            side_ptr = C.c_void_p(side.cuda_stream)
        for i in range(0, m + 1):
            p = i + 1
            if defer and i >= 3:
                main.wait_event(self._ev_settled[i - 2])
            if self.fused7:                                  # w = A u and [Q^T u, Q^T w], one pass
                if self.push_halo and i >= 1:
                    # column i's ghost rows were pushed by K2 of iteration
                    # i-1; interior tiles run before the wait on the signals
                    self._call("lsb_lagged_reduce_spmv7_halo", S, C.byref(self.op.c), i, p,
                               C.byref(self._hwait), st)
                else:
                    if self.comm is not None and self.halo:
                        self.comm.halo(self.Vstore[i], self.off, self.n, self.halo)
                    self._call("lsb_lagged_reduce_spmv7", S, C.byref(self.op.c), i, p, st)
            else:
                self._op_col(i, i + 1, i)                    # V.push(A v_i)
                self._call("lsb_lagged_reduce", S, i, p, st)  # one pass: [Q^T u, Q^T w]
            self._gather(2 * p)
            if not two and defer and i >= 1:
                self._call("lsb_mgs_lvl2_small", S, i, p, 1, -i, st)
                self._ev_front[i].record(main)
                side.wait_event(self._ev_front[i])
                self._call("lsb_settle", S, i, i, side_ptr)
                self._ev_settled[i].record(side)
                self._k2(i, p, st)
            elif not two:
                self._call("lsb_mgs_lvl2_small", S, i, p, 1, i, st)
                self._k2(i, p, st)
            else:
                self._call("lsb_cgs2_lvl2_small_a", S, i, p, 1, i, st)
                if self.fuse_k3 and p + 1 <= K3_MAX_COLS:   # K2 + 2nd mdot, Q read once
                    self._call("lsb_lagged_update_reduce", S, i, p, 1, st)
                else:
                    self._call("lsb_lagged_update", S, i, p, 1, st)
                    self._call("lsb_mdot", self.col_ptr(0), self.ld, self.n, p, self.col_ptr(p),
                               None, D.ptr(self.Gloc), self.ws.ref(), D.ptr(self.flags), i, st)
                self._gather(p)
                self._call("lsb_cgs2_lvl2_small_b", S, i, p, st)
                self._call("lsb_lagged_correct", S, i, p, st)
            if self.diagnostics:
                self._gram_row(i, i, i + 1, st)
            if self.true_residual and i >= 1:
                self._trial(i, st)
        if defer:   # join: the least squares needs every fold
            main.wait_event(self._ev_settled[m])
            if m >= 2:
                main.wait_event(self._ev_settled[m - 1])

    def _gram_row(self, it, row, ncols, st):
        """gram[row, :ncols] = Q^T q_row (diagnostics.py:47-69); on several
        ranks the local partial rows are all-gathered and summed in rank
        order (lsb_sum_parts), so every rank holds the same global Gram."""
        if self.comm is None:
            self._call("lsb_gram_row", self.Sref, it, row, ncols, D.ptr(self.gram), self.cap, st)
            return
        self._call("lsb_mdot", self.col_ptr(0), self.ld, self.n, ncols, self.col_ptr(row), None,
                   D.ptr(self.Gloc), self.ws.ref(), D.ptr(self.flags), it, st)
        self._gather(ncols)
        self._call("lsb_sum_parts", D.ptr(self.G), self.S.g_parts, self.S.g_stride, ncols,
                   C.c_void_p(self.gram.data_ptr() + 8 * row * self.cap), D.ptr(self.flags), it,
                   st)

    def _k2(self, i, p, st):
        """K2; with the fused ghost exchange it also pushes the boundary rows
        of the column it finishes (the next SpMV's input) to the neighbours."""
        if self.push_halo and i < self.m:
            hp = self.comm.halo_push(self.Vstore[p], self.off, self.n, self.halo)
            self._keep.append(hp)       # the struct outlives graph capture
            self._call("lsb_lagged_update_push", self.Sref, i, p, 1, C.byref(hp), st)
        else:
            self._call("lsb_lagged_update", self.Sref, i, p, 1, st)

    def _trial(self, i, st):
        """||b - A (x + Mi V_i y_i)|| of iteration i into true_res[i]
        (gmres.py:273-283), gated like every other kernel of iteration i."""
        S = self.Sref
        xo = 8 * self.off
        self._call("lsb_trial_lsq", S, i, D.ptr(self.ytrial), st)
        self._call("lsb_trial_combine", S, i, C.c_void_p(self.x.data_ptr() + xo),
                   D.ptr(self.ytrial), C.c_void_p(self.xt.data_ptr() + xo),
                   None if self.inv_diag is None else C.c_void_p(self.inv_diag.data_ptr() + xo),
                   st)
        self._apply_op((self.xt, self.off), C.c_void_p(self.xt.data_ptr() + xo),
                       D.ptr(self.rtrial), D.ptr(self.b), i, op=self.rop)
        self._call("lsb_norm_partial", D.ptr(self.rtrial), self.n, D.ptr(self.Gloc),
                   self.ws.ref(), D.ptr(self.flags), i, st)
        self._gather(2)
        self._call("lsb_norm_finish", D.ptr(self.G), self.S.g_parts, self.S.g_stride,
                   D.ptr(self.rtrial), self.n, C.c_void_p(self.true_res.data_ptr() + 8 * i),
                   self.ws.ref(), D.ptr(self.flags), i, st)

    # ---- host-driven pieces of the cgs1_ghysels cancellation arbitration
    def _ensure_trial_buffers(self):
        if not hasattr(self, "xt"):
            f64 = dict(dtype=D.F64, device=self.dev)
            self.ytrial = torch.zeros(self.cap, **f64)
            self.xt = self._vec_with_halo()
            if self._peer and self.halo:
                self.comm.register(self.xt, self.off, self.n)
            self.rtrial = torch.zeros(self.n, **f64)
            self.true_res = torch.zeros(self.m + 1, **f64)

    def trial_residual(self, k):
        """(||b - A (x + Mi V_k y_k)||, singular?) for iteration k, eagerly
        (gmres.py:338-348); the trial iterate stays in self.xt."""
        self._ensure_trial_buffers()
        st = D.stream()
        self._call("lsb_trial_lsq", self.Sref, k, D.ptr(self.ytrial), st)
        if bool(torch.isnan(self.ytrial[0])):
            return float("inf"), True
        self._trial(k, st)
        return float(self.true_res[k].item()), False

    def accept_trial(self):
        self.x_view().copy_(self.xt[self.off:self.off + self.n])

    def extract_k(self, k):
        """x <- x + Mi V_k y_k with the first k rotated columns (_extract)."""
        if k < 1:
            return
        self._ensure_trial_buffers()
        st = D.stream()
        xo = 8 * self.off
        self._call("lsb_trial_lsq", self.Sref, k, D.ptr(self.ytrial), st)
        self._call("lsb_trial_combine", self.Sref, k, C.c_void_p(self.x.data_ptr() + xo),
                   D.ptr(self.ytrial), C.c_void_p(self.xt.data_ptr() + xo),
                   None if self.inv_diag is None else C.c_void_p(self.inv_diag.data_ptr() + xo),
                   st)
        self.accept_trial()

    def refresh_residual(self):
        """Restart residual + norm for the current x, then a fresh report."""
        self._residual_and_norm()
        self._call("lsb_restart_check", self.Sref, 0, D.stream())
        return self.report()

    def _direct_body(self, st):
        S, m = self.Sref, self.m
        if self.diagnostics:
            self._gram_row(0, 0, 1, st)
        for i in range(1, m + 1):
            p = i
            if self.fused7_direct:
                # z = A v_{i-1} into V[:, i] and [Q^T v_{i-1}, Q^T z] in one pass;
                # the first CGS pass takes the Q^T z half (odd entries)
                if self.comm is not None and self.halo:
                    self.comm.halo(self.Vstore[i - 1], self.off, self.n, self.halo)
                self._call("lsb_lagged_reduce_spmv7", S, C.byref(self.op.c), i, p, st)
                self._gather(2 * p)
                self._call("lsb_collect_coef_pairs", S, i, p, st)
                fused = p + 1 <= K3_MAX_COLS
                if fused:   # z -= Q s and the 2nd pass's Q^T z in one read of Q
                    self._call("lsb_cgs_project_reduce", S, i, i, p, st)
                else:
                    self._call("lsb_cgs_project", S, i, i, p, 0, st)
                    self._call("lsb_mdot", self.col_ptr(0), self.ld, self.n, p, self.col_ptr(i),
                               None, D.ptr(self.Gloc), self.ws.ref(), D.ptr(self.flags), i, st)
                self._gather(p)
                self._call("lsb_collect_coef", S, i, p, 1, st)
                self._call("lsb_cgs_project", S, i, i, p, 1, st)
                self._gather(2)
                self._finish_direct(i, p, st)
                continue
            if self.fused7_ghysels:
                # [Q^T v_{i-1}, Q^T z] pairs with z = A v_{i-1} (one pass), then
                # (max|z|, sum z^2) after them: fused_mdot_norm's reduction
                if self.comm is not None and self.halo:
                    self.comm.halo(self.Vstore[i - 1], self.off, self.n, self.halo)
                self._call("lsb_lagged_reduce_spmv7_norm", S, C.byref(self.op.c), i, p, st)
                self._gather(2 * p + 2)
                self._call("lsb_ghysels_small_pairs", S, i, i, p, st)
                self._call("lsb_cgs_project", S, i, i, p, 2, st)   # + q = z / h
                if self.diagnostics:
                    self._gram_row(i, i, i + 1, st)
                if self.true_residual:
                    self._trial(i, st)
                continue
            self._op_col(i - 1, i, i)                        # z = A v_{i-1}, in place in V[:, i]
            if self.method == "cgs1_ghysels":
                # one fused reduction: [Q^T z, max|z|, sum z^2] (fused_mdot_norm)
                self._call("lsb_mdot", self.col_ptr(0), self.ld, self.n, p, self.col_ptr(i), None,
                           D.ptr(self.Gloc), self.ws.ref(), D.ptr(self.flags), i, st)
                self._call("lsb_norm_partial", self.col_ptr(i), self.n,
                           C.c_void_p(self.Gloc.data_ptr() + 8 * p), self.ws.ref(),
                           D.ptr(self.flags), i, st)
                self._gather(p + 2)
                self._call("lsb_ghysels_small", S, i, i, p, st)
                self._call("lsb_cgs_project", S, i, i, p, 2, st)   # + q = z / h
                if self.diagnostics:
                    self._gram_row(i, i, i + 1, st)
                if self.true_residual:
                    self._trial(i, st)
                continue
            if self.method == "mgs_l1":
                if self.comm is None:     # all passes in one cooperative launch
                    self._call("lsb_mgs1_passes", S, i, i, p, st)
                else:
                    for k in range(p + 1):
                        self._call("lsb_mgs1_pass", S, i, i, k, p, st)
                        self._gather(2)
            else:
                fused = self.fuse_k3 and p + 1 <= K3_MAX_COLS
                for accumulate in (0, 1):
                    if not (fused and accumulate):
                        self._call("lsb_mdot", self.col_ptr(0), self.ld, self.n, p,
                                   self.col_ptr(i), None, D.ptr(self.Gloc), self.ws.ref(),
                                   D.ptr(self.flags), i, st)
                    self._gather(p)
                    self._call("lsb_collect_coef", S, i, p, accumulate, st)
                    if fused and not accumulate:   # z -= Q s and the 2nd pass's Q^T z, one read of Q
                        self._call("lsb_cgs_project_reduce", S, i, i, p, st)
                    else:
                        self._call("lsb_cgs_project", S, i, i, p, accumulate, st)
                self._gather(2)
            self._finish_direct(i, p, st)

    def _finish_direct(self, i, p, st):
        """r_diag = ||z|| from the gathered (max, ssq) pair, K5d (breakdown,
        Hessenberg column, Givens fold), q = z / r_diag, diagnostics."""
        S = self.Sref
        self._call("lsb_norm_finish", D.ptr(self.G), self.S.g_parts, self.S.g_stride,
                   self.col_ptr(i), self.n, C.c_void_p(self.scal.data_ptr() + 8 * _abi.S_BETA),
                   self.ws.ref(), D.ptr(self.flags), i, st)
        self._call("lsb_direct_small", S, i, i, p, st)
        self._call("lsb_direct_normalize", S, i, i, st)
        if self.diagnostics:
            self._gram_row(i, i, i + 1, st)
        if self.true_residual:
            self._trial(i, st)

    # ---------------------------------------------------------------- driving
    def prologue(self):
        self.enqueue_prologue()
        return self.report()

    def cycle(self):
        self.launch_cycle()
        return self.report()

    def launch_cycle(self):
        """Enqueue one restart cycle (graph replay from the second on) without
        waiting for it; report() collects it."""
        if self.use_graph and self.cycles_run >= 1:
            if self.graph is None:
                self.graph = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    if self.comm is None:
                        with torch.cuda.graph(self.graph, stream=side):
                            self.enqueue_cycle()
                    else:
                        # ranks sharing a device (in-process emulation) spin
                        # on each other's exchange kernels: no device-wide
                        # synchronize (torch.cuda.graph's entry does one), and
                        # capture errors only for this thread.  Every rank
                        # captures and instantiates between two barriers: the
                        # instantiation may wait for the device, which must
                        # not hold a kernel spinning on a rank still capturing
                        self.comm.barrier()
                        with _CAPTURE_BEGIN_LOCK:
                            self.graph.capture_begin(capture_error_mode="thread_local")
                        try:
                            self.enqueue_cycle()
                        finally:
                            self.graph.capture_end()
                        self.comm.barrier()
                torch.cuda.current_stream().wait_stream(side)
            self.graph.replay()
        else:
            self.enqueue_cycle()
        self.cycles_run += 1

    def report(self):
        self.h_flags.copy_(self.flags, non_blocking=True)
        self.h_res.copy_(self.res, non_blocking=True)
        self.h_scal.copy_(self.scal, non_blocking=True)
        if self.true_residual:
            self.h_true.copy_(self.true_res, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return CycleReport(self.h_flags.tolist(), self.h_res.numpy().copy(),
                           self.h_scal.numpy().copy(),
                           self.h_true.numpy().copy() if self.true_residual else None)

    def solve_cycles(self, max_cycles):
        """Every restart cycle of the solve on the device in one cluster launch
        (lsb_solve_persistent; needs self.persistent): the first cycle's
        prologue as enqueue_cycle, then cycles + epilogues + restart tests
        until the restart shell would stop.  Yields one CycleReport per cycle
        run, as cycle() would have, in order -- each as soon as the device
        has written it into the mapped pinned log, so the host's per-cycle
        bookkeeping overlaps the cycles that follow."""
        st = D.stream()
        S = self.Sref
        self._call("lsb_scale_div", D.ptr(self.rbuf), self.n,
                   C.c_void_p(self.scal.data_ptr() + 8 * _abi.S_RNORM), self.col_ptr(0), None, -1, st)
        self._call("lsb_cycle_begin", S, st)
        stride = self.m + 22
        log = torch.zeros(max_cycles * stride, dtype=D.F64, pin_memory=True)
        self._call("lsb_solve_persistent", S, C.byref(self.pcsr.c), 1,
                   C.c_void_p(self.x.data_ptr() + 8 * self.off), D.ptr(self.b),
                   C.c_void_p(log.data_ptr()), int(max_cycles), st)
        done = torch.cuda.Event()
        done.record()
        host = log.numpy()
        for c in range(max_cycles):
            mark = c * stride + stride - 1
            spins = 0
            while host[mark] == 0.0:
                spins += 1
                if spins % 256 == 0 and done.query() and host[mark] == 0.0:
                    raise RuntimeError("lsb_solve_persistent ended without report %d" % c)
            if host[mark] < 0.0:
                raise _abi.LsbError("persistent cycle: a cluster handoff exceeded its wait limit "
                                    "(LSB_TUNE_PERSIST_TIMEOUT_S); the kernel aborted")
            rec = host[c * stride:(c + 1) * stride].copy()
            self.cycles_run += 1
            yield CycleReport(rec[:4].view(np.int32).tolist(), rec[4:5 + self.m],
                              rec[5 + self.m:5 + self.m + _abi.S_COUNT])
            if rec[-1] != 2.0:
                return

    def hessenberg(self, k):
        """Hbar_k from the R columns (R[:, j+1] rows 0..j+1 = H[:, j])."""
        R = self.R.cpu().numpy()
        H = np.zeros((k + 1, k))
        for j in range(k):
            H[: j + 2, j] = R[: j + 2, j + 1]
        return H

    def basis(self, k, ncols):
        B = np.zeros((self.n, k + 1))
        c = min(ncols, k + 1)
        if c > 0:
            B[:, :c] = self.Vstore[:c, self.off:self.off + self.n].t().cpu().numpy()
        return B
