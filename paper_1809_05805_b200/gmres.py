"""Drop-in GMRES drivers of lowsync.gmres (reference gmres.py), on B200.

The restart shell, history and ledger stay on the host exactly as in the
reference (gmres.py:470-516); each restart cycle runs on the device
(engine.Engine) with one host synchronisation per cycle.  The ledger is
reconstructed from the cycle report with the reference's exact event
schedule (kind, scalar_count, iteration attribution, overlap_eligible),
including pipeline2's depth-2 look-ahead.
"""

from __future__ import annotations

import os

from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _abi
from . import _dev as D
from .diagnostics import gram_orthogonality_loss, gram_paige_metric
from .engine import Engine
from .errors import HappyBreakdown, NonFiniteError, SingularHessenberg
from .kernels import DOT, FUSED, MDOT, NORM, ReductionLedger

CONVERGED = "converged"
STALLED_MAXITER = "stalled_maxiter"
BREAKDOWN = "breakdown"
CANCELLATION_FAILURE = "cancellation_failure"

METHODS = ("mgs_l1", "cgs1_ghysels", "cgs2", "two_sync_cgs2", "one_sync_mgs", "pipeline2")
_ALIASES = {
    "mgs-l1": "mgs_l1", "mgs": "mgs_l1",
    "cgs1-ghysels": "cgs1_ghysels", "ghysels": "cgs1_ghysels",
    "two-sync": "two_sync_cgs2", "two_sync": "two_sync_cgs2",
    "one-sync": "one_sync_mgs", "one_sync": "one_sync_mgs",
}
DEVICE_METHODS = METHODS


def canonical_method(name):
    """gmres.py:78-84."""
    key = name.strip().lower()
    key = _ALIASES.get(key, key)
    if key not in METHODS:
        raise ValueError(f"unknown method {name!r}; choose from {METHODS}")
    return key


@dataclass
class GmresConfig:
    """gmres.py:87-103."""
    restart_m: int = 50
    max_restarts: int = 10
    rel_tol: float = 1e-6
    method: str = "one_sync_mgs"
    precond: str = "none"
    breakdown_tol_factor: float = 1.0

    def __post_init__(self):
        if self.restart_m < 1:
            raise ValueError("restart_m must be >= 1")
        if not self.rel_tol > 0.0:
            raise ValueError("rel_tol must be positive")
        self.method = canonical_method(self.method)
        if self.precond not in ("none", "jacobi"):
            raise ValueError("precond must be 'none' or 'jacobi'")


class Preconditioner:
    """Right preconditioner: identity or Jacobi (gmres.py:106-118)."""

    def __init__(self, kind, A=None, comm=None):
        if kind not in ("none", "jacobi"):
            raise ValueError("precond must be 'none' or 'jacobi'")
        self.kind = kind
        self.inv_diag = None
        if kind == "jacobi":
            # row-partitioned: this rank's rows; the zero test is global
            # (every rank raises together)
            d = np.asarray(A.diagonal_values(), dtype=np.float64)
            zero = bool(np.any(d == 0.0))
            if comm is not None:
                zero = comm.max_scalar(1.0 if zero else 0.0) > 0.0
            if zero:
                raise ValueError("jacobi preconditioner requires a zero-free diagonal")
            self.inv_diag = 1.0 / d


def apply_preconditioner(precond, v):
    """M^{-1} v (gmres.py:121-126); elementwise product on the device."""
    host = D.is_host(v)
    vv = D.to_device_vector(v)
    if precond is None or precond.kind == "none":
        return D.out_like(vv, host)
    d = D.to_device_vector(precond.inv_diag, vv.shape[0])
    out = torch.empty_like(vv)
    # v * inv_diag (one rounding) through K6's column-scaling path: a
    # one-point identity stencil computes 1.0 * (v[r] * d[r]) exactly.
    from .operators import StencilMatrix
    S = StencilMatrix((vv.shape[0], 1, 1), [((0, 0, 0), 1.0)])
    S.device_op().with_scale(d).apply(vv, out)
    return D.out_like(out, host)


class GivensState:
    """Rotations, rotated triangle and rhs (gmres.py:129-140).  Default:
    numpy arrays like the reference (g, tri, the rotations list; the device
    kernels run on staged copies and write them back); ``device="cuda"``:
    kept on the device (rotations read back on access)."""

    def __init__(self, m, beta, device=None):
        self.m = int(m)
        self.host = device is None
        if self.host:
            self.rotations = []
            self.g = np.zeros(m + 1)
            self.g[0] = beta
            self.tri = np.zeros((m + 1, m))
            return
        dev = D.require_cuda()
        self._rot = torch.zeros(2 * max(m, 1), dtype=D.F64, device=dev)
        self.g = torch.zeros(m + 1, dtype=D.F64, device=dev)
        self.g[0] = float(beta)
        self.tri = torch.zeros((m + 1, m), dtype=D.F64, device=dev)
        self._count = 0

    def __getattr__(self, name):
        if name == "rotations":      # device mode
            r = self._rot[: 2 * self._count].cpu().numpy()
            return [(float(r[2 * k]), float(r[2 * k + 1])) for k in range(self._count)]
        raise AttributeError(name)

    def _staged(self):
        """(rot, g, tri, count) as device tensors."""
        if not self.host:
            return self._rot, self.g, self.tri, self._count
        dev = D.require_cuda()
        rot = np.zeros(2 * max(self.m, 1))
        for k, (c, s_) in enumerate(self.rotations):
            rot[2 * k], rot[2 * k + 1] = c, s_
        return (torch.as_tensor(rot).to(dev), torch.as_tensor(np.array(self.g)).to(dev),
                torch.as_tensor(np.ascontiguousarray(self.tri)).to(dev), len(self.rotations))


def givens_update(state, h_col, i):
    """Fold Hessenberg column i (1-based, i+1 entries); returns |g[i]|
    (gmres.py:153-177) -- the same device code the solver cycle runs."""
    rot, g, tri, count = state._staged()
    if count != i - 1:
        raise ValueError(f"expected {i - 1} prior rotations, have {count}")
    h = D.to_device_vector(h_col)
    if h.shape[0] != i + 1:
        raise ValueError(f"column {i} must have {i + 1} entries")
    res = torch.empty(1, dtype=D.F64, device=h.device)
    _abi.call("lsb_givens_update", D.ptr(rot), D.ptr(g), D.ptr(tri), state.m, D.ptr(h), i,
              D.ptr(res), D.stream())
    if state.host:
        r = rot.cpu().numpy()
        state.rotations.append((float(r[2 * (i - 1)]), float(r[2 * (i - 1) + 1])))
        state.g[...] = g.cpu().numpy()
        state.tri[...] = tri.cpu().numpy()
    else:
        state._count += 1
    return float(res.item())


def solve_least_squares(state, k):
    """Back-substitution of the rotated k x k triangle (gmres.py:184-192)."""
    _, g, tri, _ = state._staged()
    y = torch.zeros(max(k, 1), dtype=D.F64, device=g.device)
    st = torch.zeros(1, dtype=torch.int32, device=g.device)
    _abi.call("lsb_back_substitute", D.ptr(tri.contiguous()), D.ptr(g), state.m, k,
              D.ptr(y), D.ptr(st), D.stream())
    bad = int(st.item())
    if bad >= 0:
        raise SingularHessenberg(f"zero diagonal at {bad}")
    return y[:k].cpu().numpy()


@dataclass
class IterationRecord:
    iteration: int
    implicit_rel_res: float
    true_rel_res: float | None = None
    s_norm: float | None = None
    orth_loss: float | None = None
    reductions: int = 0


class ConvergenceHistory:
    """Per-iteration records (gmres.py:205-236).  ``basis`` / ``hessenberg``
    are materialised from the device on first access (the reference copies
    V every cycle, 5.5 s/cycle at 256^3; here it costs nothing unless read)."""

    def __init__(self):
        self.records: list[IterationRecord] = []
        self.outcome: str | None = None
        self.denom = 1.0
        self.cycle_starts: list[int] = []
        self.k = 0
        self.final_true_rel_res = None
        self.method = None
        self._stash = None
        self._basis = None
        self._hess = None

    @property
    def iterations(self):
        return len(self.records)

    def implicit_curve(self):
        return np.array([r.implicit_rel_res for r in self.records])

    def stall_iteration(self, level=0.99):
        for rec in self.records:
            if rec.s_norm is not None and rec.s_norm >= level:
                return rec.iteration
        return None

    @property
    def basis(self):
        if self._basis is None and self._stash is not None:
            eng, k, ncols = self._stash
            self._basis = eng.basis(k, ncols)
        return self._basis

    @basis.setter
    def basis(self, v):
        self._basis = v

    @property
    def hessenberg(self):
        if self._hess is None and self._stash is not None:
            eng, k, _ = self._stash
            self._hess = eng.hessenberg(k)
        return self._hess

    @hessenberg.setter
    def hessenberg(self, v):
        self._hess = v

    def release(self):
        """Drop the device basis kept alive for lazy ``basis`` access
        (without copying it: unread attachments are simply discarded)."""
        self._stash = None


# One engine (basis storage, small-state arena, captured cycle graph) kept
# across solve() calls on the same operator object and configuration: a
# service solving many right-hand sides pays the allocation and the graph
# capture once (the e2e path).  Reused only when the previous solve's
# history no longer holds the engine for its lazy `basis` (released,
# collected or already materialised), so no history ever sees its basis
# overwritten.  clear_engine_cache() drops it (frees the device memory).
_ENGINE_CACHE = {}


def clear_engine_cache():
    _ENGINE_CACHE.clear()


class _BasisSnapshot:
    """Device copy of what a history's lazy ``basis`` / ``hessenberg`` read
    from its engine (the basis columns and R), so the engine can be reused
    by the next solve while that history is still alive (a solve loop
    `x, h = solve(...)` keeps the previous h until the call returns).  Same
    interface as Engine.basis / Engine.hessenberg."""

    def __init__(self, eng, ncols):
        c = max(0, min(ncols, eng.Vstore.shape[0]))
        self.n = eng.n
        self.V = eng.Vstore[:c, eng.off:eng.off + eng.n].clone()
        self.R = eng.R.clone()

    def hessenberg(self, k):
        R = self.R.cpu().numpy()
        H = np.zeros((k + 1, k))
        for j in range(k):
            H[: j + 2, j] = R[: j + 2, j + 1]
        return H

    def basis(self, k, ncols):
        B = np.zeros((self.n, k + 1))
        c = min(ncols, k + 1, self.V.shape[0])
        if c > 0:
            B[:, :c] = self.V[:c].t().cpu().numpy()
        return B


# a live history's basis up to this size is copied on the device (a few
# microseconds) so the cached engine is reused; above it a new engine is
# built instead (its allocation and graph capture are then noise next to
# the solve itself, and a second basis copy would double the footprint)
_SNAPSHOT_MAX_BYTES = 1 << 28


def _cached_engine(key, A):
    ent = _ENGINE_CACHE.get(key)
    if ent is None:
        return None
    eng, a_ref, h_ref = ent
    if a_ref() is not A:
        return None
    h = h_ref() if h_ref is not None else None
    if h is not None and h._stash is not None and h._basis is None:
        src, k, ncols = h._stash
        if src is not eng:
            return eng
        if (min(ncols, k + 1) * eng.n + eng.R.numel()) * 8 > _SNAPSHOT_MAX_BYTES:
            return None
        h._stash = (_BasisSnapshot(eng, min(ncols, k + 1)), k, ncols)
    return eng


class _DeviceSolve:
    """One solve: host restart shell over device cycles (gmres.py:239-516)."""

    def __init__(self, A, b, x0, config, ledger, diagnostics_every, true_residual_every,
                 use_graph=True, comm=None, n_global=None):
        if A.n_rows != A.n_cols:
            raise ValueError("GMRES needs a square matrix")
        if config.method not in DEVICE_METHODS:
            raise NotImplementedError(
                f"method {config.method!r} is outside the B200 hot path (SURVEY §8f)")
        self.true_every = int(true_residual_every or 0)
        import os
        import time
        self._trace = [("start", time.perf_counter())] if os.environ.get("LSB_TRACE") else None
        self.A = A
        self.comm = comm
        self.n = A.n_rows
        self.n_global = int(n_global or self.n)
        self.host = D.is_host(b)
        self.b = D.to_device_vector(b, self.n)
        if comm is None and not bool((self.b != 0).any()):
            raise ValueError("right-hand side must be nonzero")
        self.x0 = None if x0 is None else D.to_device_vector(x0, self.n)
        self.config = config
        self.ledger = ledger if ledger is not None else ReductionLedger()
        self.pc = Preconditioner(config.precond, A, comm=comm)
        self.m = min(config.restart_m, self.n_global)
        self.diag_every = diagnostics_every
        self.history = ConvergenceHistory()
        self.history.method = config.method
        self.global_it = 0
        self.use_graph = use_graph
        self._mark("setup")

    def _events_lagged(self, base, k, stop, broke_iter, two, pipeline):
        """Ledger events + per-iteration reduction counts of one lagged cycle
        (gmres.py:397-462)."""
        led = self.ledger
        led.iteration = base
        led.record(FUSED, 2)
        if two:
            led.record(MDOT, 1)
        nred = {}

        def advance(i, eligible):
            led.iteration = base + i
            mark = len(led)
            led.record(FUSED, 2 * (i + 1), eligible)
            if two and broke_iter != i:
                led.record(MDOT, i + 1, eligible)
            nred[i] = len(led) - mark
            return broke_iter == i

        if not pipeline:
            for i in range(1, k + 1):
                advance(i, False)
        else:
            i, done = 1, False
            while i <= self.m and not done:
                pair = [i] if i == self.m else [i, i + 1]
                for t in pair:
                    br = advance(t, True)
                    if br:
                        break
                if stop is not None and stop in pair:
                    done = True
                i += len(pair)
        return nred

    def _events_direct(self, i, two_pass):
        led = self.ledger
        mark = len(led)
        if two_pass:
            led.record(MDOT, i)
            led.record(MDOT, i)
        else:
            for _ in range(i):
                led.record(DOT, 1)
        led.record(NORM, 1)
        return len(led) - mark

    def run(self):
        cfg = self.config
        led = self.ledger
        hist = self.history
        inv = self.pc.inv_diag
        key = (id(self.A), self.m, cfg.method, cfg.precond, bool(self.diag_every),
               bool(self.true_every), id(self.comm), self.n_global, self.use_graph,
               os.environ.get("LSB_PERSISTENT"))
        # (single-rank only: reuse must be a collective decision across ranks)
        cache = self.comm is None and os.environ.get("LSB_ENGINE_CACHE", "1") != "0"
        eng = _cached_engine(key, self.A) if cache else None
        if eng is not None:
            eng.reset(cfg.rel_tol, cfg.breakdown_tol_factor)
        else:
            if cache:
                _ENGINE_CACHE.clear()    # at most one engine (its basis) kept alive
            eng = Engine(self.A, self.m, cfg.method, cfg.rel_tol, cfg.breakdown_tol_factor,
                         inv_diag=inv, diagnostics=bool(self.diag_every),
                         use_graph=self.use_graph, comm=self.comm, n_global=self.n_global,
                         true_residual=bool(self.true_every))
        if cache:
            import weakref
            try:
                _ENGINE_CACHE[key] = (eng, weakref.ref(self.A), weakref.ref(self.history))
            except TypeError:            # operator without weakref support: no reuse
                pass
        self.engine = eng
        self._mark("engine")
        eng.load(self.b, self.x0)
        if self.comm is not None:
            # every rank's buffers exist (and are registered) before any
            # exchange kernel can spin on them
            self.comm.barrier()
            eng.setup_exchange()
        # the host result buffer is faulted in while the device iterates
        self._xhost = D.HostBuffer(eng.n) if (self.host and eng.n >= D._STAGE_MIN
                                              and not D._PINNED_RESULTS) else None
        led.iteration = 0
        rep = eng.prologue()
        self._mark("prologue")
        self._comm_check(rep)
        if rep.nonfinite:
            raise NonFiniteError("spmv result contains NaN or Inf")
        beta = float(rep.scal[_abi.S_RNORM])
        if np.isnan(beta):
            raise NonFiniteError("norm2 input contains NaN")
        led.record(NORM, 1)
        hist.denom = beta if beta > 0.0 else 1.0
        if beta == 0.0:
            hist.outcome = CONVERGED
            hist.final_true_rel_res = 0.0
            return self._result(eng)
        target = cfg.rel_tol * beta
        outcome = None
        saw_cancellation = False
        lagged = cfg.method in ("one_sync_mgs", "two_sync_cgs2", "pipeline2")
        # launch-bound sizes: the whole restarted solve is one cluster launch
        # that logs every cycle's report; the shell below replays them
        whole = eng.persistent and cfg.max_restarts >= 1 \
            and os.environ.get("LSB_PERSISTENT_SOLVE", "1") != "0"
        device_reports = eng.solve_cycles(cfg.max_restarts) if whole else None
        # the next cycle is launched as soon as a report says the restart
        # shell will continue -- before this cycle's ledger/history
        # bookkeeping, which then overlaps the device (not for Ghysels, whose
        # arbitration is host-driven, nor with diagnostics, read from the
        # device state the next cycle overwrites)
        ahead = cfg.method != "cgs1_ghysels" and not self.diag_every \
            and os.environ.get("LSB_CYCLE_AHEAD", "1") != "0"
        pending = False
        for _cycle in range(cfg.max_restarts):
            hist.cycle_starts.append(self.global_it)
            if device_reports is None:
                rep = eng.report() if pending else eng.cycle()
                pending = False
                if ahead and _cycle + 1 < cfg.max_restarts and not rep.nonfinite \
                        and not rep.comm_error and rep.status == _abi.RUNNING \
                        and rep.stop_iter == _abi.NO_STOP \
                        and not float(rep.scal[_abi.S_RNORM]) <= target:
                    eng.launch_cycle()
                    pending = True
            else:
                rep = next(device_reports, None)
                if rep is None:
                    raise RuntimeError("device solve stopped before the restart shell")
            self._mark("cycle")
            self._comm_check(rep)
            if rep.nonfinite:
                raise NonFiniteError("spmv result contains NaN or Inf")
            if rep.status == _abi.STARTUP_BREAKDOWN:
                raise HappyBreakdown(0, float(rep.scal[_abi.S_BETA]), float(rep.scal[_abi.S_TOL]),
                                     r_col=np.zeros(0))
            if rep.status == _abi.SINGULAR:
                raise SingularHessenberg(f"zero diagonal at {rep.k}")
            stopped = rep.stop_iter != _abi.NO_STOP
            k = rep.stop_iter if stopped else self.m
            broke = rep.broke_iter if rep.broke_iter >= 1 else None
            gram = eng.gram.cpu().numpy() if self.diag_every else None
            base = self.global_it
            decided = None
            if lagged:
                nred = self._events_lagged(base, k, k if stopped else None, broke,
                                           cfg.method == "two_sync_cgs2",
                                           cfg.method == "pipeline2")
                for i in range(1, k + 1):
                    self.global_it = base + i
                    ncols = i if broke == i else i + 1
                    self._record(rep.res[i], nred[i], gram, ncols, rep, i)
            elif cfg.method == "cgs1_ghysels":
                check = rep.status == _abi.GHYSELS_CHECK
                last = k - 1 if check else k
                stop_col = k
                for i in range(1, last + 1):
                    self.global_it += 1
                    led.iteration = self.global_it
                    led.record(FUSED, i + 1)
                    self._record(rep.res[i], 1, gram, i + 1, rep, i)
                if check:
                    # gmres.py:333-360: the Pythagorean radicand lost its
                    # digits -- arbitrate with the true residual of the trial
                    i = k
                    self.global_it += 1
                    led.iteration = self.global_it
                    mark = len(led)
                    led.record(FUSED, i + 1)
                    true_abs, singular = eng.trial_residual(i)
                    if not singular:
                        led.record(NORM, 1)
                    rad = float(rep.scal[_abi.S_RAD])
                    if not singular and (true_abs <= target or rad == 0.0):
                        self._record(rep.res[i], len(led) - mark, gram, i, rep, i)
                        eng.accept_trial()
                        decided = CONVERGED if true_abs <= target else BREAKDOWN
                    else:
                        k = i - 1                  # aborted attempt: nothing recorded
                        eng.extract_k(k)
                        decided = CANCELLATION_FAILURE
                    rep = eng.refresh_residual()
            else:
                for i in range(1, k + 1):
                    self.global_it += 1
                    led.iteration = self.global_it
                    nr = self._events_direct(i, cfg.method == "cgs2")
                    ncols = i if broke == i else i + 1
                    self._record(rep.res[i], nr, gram, ncols, rep, i)
            if decided is not None:
                status = decided
            elif stopped:
                status = CONVERGED if rep.status == _abi.CONVERGED else BREAKDOWN
            else:
                status = "full"
            if lagged:
                ncols_norm = k + (0 if status == BREAKDOWN else 1)
            elif cfg.method == "cgs1_ghysels":
                ncols_norm = stop_col if decided is not None else k + 1
            else:
                ncols_norm = k if broke == k else k + 1
            hist.k = k
            hist._stash = (eng, k, ncols_norm)
            hist._basis = hist._hess = None
            if status in (CONVERGED, BREAKDOWN):
                outcome = status
                break
            if status == CANCELLATION_FAILURE:
                saw_cancellation = True
            led.iteration = self.global_it
            led.record(NORM, 1)
            beta = float(rep.scal[_abi.S_RNORM])
            rel = beta / hist.denom
            if hist.records:
                hist.records[-1].true_rel_res = rel
            if beta <= target:
                outcome = CONVERGED
                break
        if device_reports is not None and next(device_reports, None) is not None:
            raise RuntimeError("device solve ran past the restart shell")
        if outcome is None:
            outcome = CANCELLATION_FAILURE if saw_cancellation else STALLED_MAXITER
        led.iteration = self.global_it
        led.record(NORM, 1)
        final_rel = float(rep.scal[_abi.S_RNORM]) / hist.denom
        hist.final_true_rel_res = final_rel
        if hist.records:
            hist.records[-1].true_rel_res = final_rel
        hist.outcome = outcome
        return self._result(eng)

    def _comm_check(self, rep):
        if rep.comm_error:
            if self.comm is not None and hasattr(self.comm, "check"):
                self.comm.check()
            raise RuntimeError("peer exchange timed out (a rank stopped participating)")

    def _record(self, res, nred, gram, ncols, rep=None, i=0):
        """gmres.py:280-292: diagnostics from the device Gram rows, the
        true-residual probe from the device trial of iteration i."""
        s = o = None
        if self.diag_every and self.global_it % self.diag_every == 0:
            Gm = gram[:ncols, :ncols]
            Gm = np.triu(Gm.T, 0) + np.triu(Gm.T, 1).T  # rows hold Q^T q_row: symmetrise
            s, o = gram_paige_metric(Gm), gram_orthogonality_loss(Gm)
        true_rel = None
        if self.true_every and self.global_it % self.true_every == 0 and i >= 1:
            v = float(rep.true_res[i])
            if np.isnan(v):
                raise SingularHessenberg("zero diagonal in the trial least-squares solve")
            true_rel = v / self.history.denom
        self.history.records.append(IterationRecord(
            iteration=self.global_it, implicit_rel_res=float(res) / self.history.denom,
            true_rel_res=true_rel, s_norm=s, orth_loss=o, reductions=nred))

    def _result(self, eng):
        x = eng.x_view().clone()
        hb = getattr(self, "_xhost", None)
        out = D.out_like(x, self.host, hb), self.history
        self._mark("result")
        if self._trace is not None:
            import sys
            t0 = self._trace[0][1]
            sys.stderr.write("lsb trace: " + ", ".join(
                f"{k} {1e3 * (t - t0):.1f}ms" for k, t in self._trace[1:]) + "\n")
        return out

    def _mark(self, label):
        """LSB_TRACE=1: synchronised phase timestamps of one solve."""
        if self._trace is not None:
            import time
            torch.cuda.synchronize()
            self._trace.append((label, time.perf_counter()))


def _run(method, A, b, x0, config, ledger, diagnostics_every, true_residual_every):
    config = replace(config, method=method) if config is not None else GmresConfig(method=method)
    return _DeviceSolve(A, b, x0, config, ledger, diagnostics_every, true_residual_every).run()


def gmres_mgs_l1(A, b, x0=None, config=None, ledger=None, diagnostics_every=1,
                 true_residual_every=0):
    """Level-1 MGS GMRES: i + 1 reductions at iteration i (gmres.py:526-530)."""
    return _run("mgs_l1", A, b, x0, config, ledger, diagnostics_every, true_residual_every)


def gmres_cgs2(A, b, x0=None, config=None, ledger=None, diagnostics_every=1,
               true_residual_every=0):
    """Two-pass classical GS GMRES: 3 reductions per iteration (gmres.py:533-537)."""
    return _run("cgs2", A, b, x0, config, ledger, diagnostics_every, true_residual_every)


def gmres_cgs1_ghysels(A, b, x0=None, config=None, ledger=None, diagnostics_every=1,
                       true_residual_every=0):
    """Single-pass classical GS with the Pythagorean norm substitute, one
    fused reduction per iteration; cancellation is arbitrated with the true
    residual exactly as gmres.py:325-360 (gmres.py:540-548)."""
    return _run("cgs1_ghysels", A, b, x0, config, ledger, diagnostics_every, true_residual_every)


def gmres_two_sync(A, b, x0=None, config=None, ledger=None, diagnostics_every=1,
                   true_residual_every=0):
    """Lagged two-pass classical GMRES: 2 reductions per iteration (gmres.py:551-555)."""
    return _run("two_sync_cgs2", A, b, x0, config, ledger, diagnostics_every, true_residual_every)


def gmres_one_sync(A, b, x0=None, config=None, ledger=None, diagnostics_every=1,
                   true_residual_every=0):
    """Lagged compact-WY MGS GMRES: 1 reduction per iteration (gmres.py:558-562)."""
    return _run("one_sync_mgs", A, b, x0, config, ledger, diagnostics_every, true_residual_every)


def gmres_pipeline2(A, b, x0=None, config=None, ledger=None, diagnostics_every=1,
                    true_residual_every=0):
    """Depth-2 schedule of one_sync; bitwise-identical history, reductions
    tagged overlap_eligible (gmres.py:565-576)."""
    return _run("pipeline2", A, b, x0, config, ledger, diagnostics_every, true_residual_every)


_DISPATCH = {
    "mgs_l1": gmres_mgs_l1,
    "cgs2": gmres_cgs2,
    "cgs1_ghysels": gmres_cgs1_ghysels,
    "two_sync_cgs2": gmres_two_sync,
    "one_sync_mgs": gmres_one_sync,
    "pipeline2": gmres_pipeline2,
}


def solve(A, b, x0=None, config=None, ledger=None, diagnostics_every=1, true_residual_every=0):
    """Dispatch on config.method (gmres.py:589-594)."""
    config = config if config is not None else GmresConfig()
    return _DISPATCH[config.method](A, b, x0, config, ledger, diagnostics_every,
                                    true_residual_every)


def solve_distributed(op, b_local, comm, n_global, x0_local=None, config=None, ledger=None,
                      diagnostics_every=0):
    """Row-partitioned solve (one rank per GPU): `op` is this rank's row
    block -- a stencil z-slab (parallel.slab_problem) or a CSR row block
    (parallel.csr_row_block) -- and b_local/x0_local its rows.  Every rank
    runs the same host restart shell on bit-identical device reports, so
    histories, ledgers and diagnostics agree across ranks (the Gram rows of
    the diagnostics are all-gathered like the solver's reductions);
    returns (x_local, history)."""
    config = config if config is not None else GmresConfig()
    return _DeviceSolve(op, b_local, x0_local, config, ledger, diagnostics_every, 0,
                        use_graph=True, comm=comm, n_global=n_global).run()
