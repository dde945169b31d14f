"""Benchmark: Arnoldi iterations/s of one-sync MGS-CWY GMRES(50) on the 3D
7-point Laplacian (BASELINE.json config 2: 256^3, n = 16.7M) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

A step is one GMRES(50) restart cycle = 50 Arnoldi iterations (SpMV + K1
one-pass [Q^T u, Q^T w] + K5 small state + K2 lagged update, then the
cycle's least squares, x update and restart residual), all resident in HBM.
`value` = whole-job iterations/s, device-timed with CUDA events; `e2e` = the
same metric through the public drop-in call `solve(A, b_host, ...)` with the
host->device copy of b and the device->host copy of x inside each step.

--gpus N > 1 runs the row-partitioned (z-slab) solve, one process per GPU:
launched under torchrun by the driver, or re-executed under
torch.distributed.run by this script when WORLD_SIZE is unset (it exits
non-zero if the world size then differs from N).  The per-iteration
exchanges -- one all-gather of the 2p-vector per iteration plus the ghost
z-planes -- are peer-memory kernels over NVLink (parallel.PeerComm, CUDA
IPC mappings, captured in the cycle graph); NCCL (NCCL_DEBUG=INFO) carries
setup and host scalars, and is the fallback transport when peer mappings
are unavailable (--comm nccl forces it).  Default: weak scaling, 256^3 rows
per GPU, the global grid doubled x -> y -> z (N=8 is the 512^3 cube of
config 4); `value` counts 16.7M-row slab iterations/s (global it/s x N, the
unit the driver's weak-scaling efficiency needs) and `global_it_per_s` is
the solve's own rate.  --strong runs config 4 as stated (512^3 split over
N GPUs, value = global it/s).

--impl reference times the reference algorithm on the host cores: the
numpy oracle port (oracle/lowsync_oracle.py, same numpy/OpenBLAS calls as
lowsync) on the same C2 solve -- after an untimed prefix of 23 iterations,
each step is a window of 3 consecutive Arnoldi iterations (p = 24, 25, ...
continuing through the restart), so the timed steps sample a
representative mix of p.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Arnoldi iters/sec (n=16.7M, m=50); ortho HBM GB/s vs peak; 1/2/4/8 B200"
UNIT = "Arnoldi iterations/s"
N_SLAB = 256
M = 50
C4_ONE_GPU = 104.6   # it/s, 512^3 one-sync GMRES(50) cycle on one B200 (round 1)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _dims(n_gpus, slab=N_SLAB):
    """Global grid for N GPUs: slab^3 (256^3) per GPU, doubling x, y, z in
    turn (N=8 -> 512^3 = config 4); slabs along z."""
    nx = ny = nz = slab
    k = 0
    g = n_gpus
    while g > 1:
        if k % 3 == 0:
            nx *= 2
        elif k % 3 == 1:
            ny *= 2
        else:
            nz *= 2
        g //= 2
        k += 1
    return nx, ny, nz


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, enabled=True):
        self.index = index
        self.enabled = enabled
        self.proc = None
        self.lines = []

    def __enter__(self):
        if not self.enabled:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU side
PREFIX = 23        # untimed Arnoldi iterations before the first CPU window
PER_WINDOW = 3     # Arnoldi iterations per CPU step


def _blas_threads(threads):
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(threads)
    except Exception:   # noqa: BLE001 -- env var then governs a fresh numpy
        os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
        return None


def cpu_windows(n_windows, per=PER_WINDOW, prefix=PREFIX, threads=None):
    """The reference algorithm (numpy oracle port, same numpy/OpenBLAS calls
    as lowsync) on the host cores: ONE run of the C2 solve; after `prefix`
    untimed iterations, `n_windows` consecutive windows of `per` Arnoldi
    iterations (continuing through the restart at 50, whose extract and
    restart residual belong to the cycle the GPU step times too).
    Returns (seconds per window, threads)."""
    threads = threads or os.cpu_count()
    lim = _blas_threads(threads)
    from oracle import lowsync_oracle as orc
    A = orc.laplace3d(N_SLAB)
    b = orc.rhs_random(A.n_rows, 42)
    total = prefix + n_windows * per
    run = orc.gmres(A, b, "one_sync_mgs", M, total // M + 2, 1e-14, max_iters=total)
    t = run.iter_t
    assert len(t) == total
    out = [t[prefix + (w + 1) * per - 1] - t[prefix + w * per - 1] for w in range(n_windows)]
    del lim
    return out, threads


def _config(world, slab, strong=False):
    nx, ny, nz = (512, 512, 512) if strong else _dims(world, slab)
    n_global = nx * ny * nz
    return {"workload": f"3D 7-point Laplacian {nx}x{ny}x{nz} (n={n_global:,}), "
                        "one-sync MGS-CWY GMRES(50), seed-42 unit Gaussian b, x0=0",
            "n_per_gpu": n_global // world, "m": M, "method": "one_sync_mgs",
            "step": "one GMRES(50) restart cycle = 50 Arnoldi iterations",
            "rel_tol": 1e-14, "l2": "inputs larger than L2 (basis 7.0 GB per GPU)"
            if not strong or world >= 8 else "inputs larger than L2",
            "partition": "z-slabs" if world > 1 else "none",
            "value_units": ("global Arnoldi iterations/s of the 512^3 solve" if strong else
                            f"Arnoldi iterations/s of {slab}^3-row slabs (global it/s x N)")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = args.gpus
    steps = args.warmup + args.steps
    secs, threads = cpu_windows(steps)
    timed = secs[args.warmup:]
    tot = sum(timed)
    value = PER_WINDOW * len(timed) / tot
    first = PREFIX + args.warmup * PER_WINDOW + 1
    sample = (f"one run of the 256^3 one-sync GMRES(50) solve (numpy oracle port, same "
              f"numpy/OpenBLAS calls as lowsync): {PREFIX} untimed iterations, {args.warmup} "
              f"warm-up windows, then each step = {PER_WINDOW} consecutive Arnoldi iterations "
              f"(timed: iterations {first}..{first + PER_WINDOW * len(timed) - 1}, through the "
              f"restart at {M})")
    if world > 1:
        sample += ("; the CPU's cost is linear in rows, so its rate on one 256^3 slab is its "
                   "rate in the GPU arm's unit (slab iterations/s = global it/s x N)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(world, N_SLAB),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- GPU side
def _ortho_bytes(n, p, kind):
    """Algorithmic HBM bytes per launch."""
    if kind == "lagged_reduce":      # K1: reads Q (p cols, u = col p-1) and w
        return 8 * n * (p + 1)
    if kind == "lagged_reduce_spmv":  # K1+K6 fused: reads Q (incl. u), writes w = A u
        return 8 * n * (p + 1)
    if kind == "lagged_update":      # K2: reads Q[:p-1], u, w; writes u, w
        return 8 * n * (p + 3)
    if kind == "spmv":               # K6 stencil: read x, write y
        return 16 * n
    return 0


def _reexec_torchrun(args):
    """--gpus N > 1 without a launcher: start N ranks under torch.distributed.run."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execvpe(sys.executable, cmd, env)


def _make_comm(args, rank):
    """Host communicator over NCCL, and the peer-memory exchange on top of it
    (falls back to NCCL collectives if peer mappings are unavailable)."""
    from paper_1809_05805_b200.parallel import Comm, PeerComm, PeerUnavailable
    # NCCL refuses two ranks on one device: --shared-gpu validation uses gloo
    host = Comm.init("gloo" if args.shared_gpu else None)
    if args.comm == "nccl":
        return host, "nccl"
    try:
        pc = PeerComm(host, ipc=True)
        pc.selftest()
        return pc, "peer-ipc"
    except PeerUnavailable as e:
        if rank == 0:
            sys.stderr.write(f"bench: peer exchange unavailable ({e}); using NCCL collectives\n")
        return host, "nccl"


def run_gpu(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.emulate_ranks <= 1 and world != args.gpus:
        sys.stderr.write(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    need = 1 if (args.emulate_ranks > 1 or args.shared_gpu) else args.gpus
    if torch.cuda.device_count() < need:
        sys.stderr.write(f"bench: --gpus {args.gpus} but only {torch.cuda.device_count()} "
                         "CUDA devices are visible\n")
        sys.exit(2)
    if args.shared_gpu:
        local = 0    # validation: every rank process on GPU 0 (gloo host comm, IPC peers)
    torch.cuda.set_device(local)
    if args.emulate_ranks > 1:
        # P ranks as threads on this one GPU (parallel.run_threads, peer
        # exchange kernels): exercises the multi-rank path end to end; the
        # number is NOT a scaling result
        from paper_1809_05805_b200.parallel import run_threads
        out = run_threads(args.emulate_ranks,
                          lambda c: _bench_core(args, c, args.emulate_ranks, c.rank, local,
                                                "peer-threads"),
                          peer=True)
        print(json.dumps(dict(out[0], emulated_ranks_on_one_gpu=args.emulate_ranks)), flush=True)
        return
    comm, kind = None, None
    if world > 1:
        # communicator creation logged (ranks per NCCL communicator), also
        # when the driver launches torchrun itself
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        comm, kind = _make_comm(args, rank)
    result = _bench_core(args, comm, world, rank, local, kind)
    if args.shared_gpu:
        result["shared_gpu_validation"] = "all ranks on GPU 0: NOT a scaling result"
    if rank == 0:
        print(json.dumps(result), flush=True)
    if comm is not None:
        if kind == "peer-ipc":
            comm.close()
            comm.host.close()
        else:
            comm.close()


def _bench_core(args, comm, world, rank, local, comm_kind=None):
    import numpy as np
    import torch

    import paper_1809_05805_b200 as P
    from paper_1809_05805_b200 import _abi
    from paper_1809_05805_b200.engine import Engine

    slab = args.slab
    nx, ny, nz = (512, 512, 512) if args.strong else _dims(world, slab)
    if comm is not None:
        from paper_1809_05805_b200.parallel import slab_problem
        A_local, n_global = slab_problem((nx, ny, nz), comm)
    else:
        A_local = P.gen_laplace3d(nx)
        n_global = A_local.n_rows
    n = A_local.n_rows
    if comm is None:
        b_local = np.random.default_rng(42).standard_normal(n)
        b_local /= np.linalg.norm(b_local)
    else:
        from paper_1809_05805_b200.parallel import local_rhs
        b_local = local_rhs((nx, ny, nz), comm, 42)

    # the production path: on one GPU the cycle is a CUDA graph (captured in
    # the second warm-up cycle).  The per-kernel timing events are captured
    # as event-record nodes into a second, instrumented copy of the cycle
    # graph; --kernel-timers last (default) replays it for the last timed
    # step only (event nodes cost ~3% of a cycle), "all" for every step.
    eng = Engine(A_local, M, "one_sync_mgs", 1e-14, comm=comm, n_global=n_global)
    eng.load(torch.as_tensor(b_local).cuda())
    rep = eng.prologue()

    timers = []
    eng.timer = timers

    def step():
        r = eng.cycle()
        assert r.stop_iter == _abi.NO_STOP, "bench cycles must run all m iterations"
        return r

    captured = None   # timers[a:b] = the event pairs inside the instrumented graph
    clean = timed = None
    for w in range(args.warmup):
        k0 = len(timers)
        step()
        if eng.graph is not None and captured is None:
            captured = (k0, len(timers))
            timed = eng.graph
            if args.kernel_timers == "last":   # capture the uninstrumented twin
                eng.timer, eng.graph = None, None
                step()
                clean, eng.timer = eng.graph, timers
    if captured is None:
        timers.clear()
    torch.cuda.synchronize()
    if comm is not None:
        comm.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, enabled=(rank == 0)) as clk:
        ev0.record()
        for s_i in range(args.steps):
            if clean is not None:
                eng.graph = timed if s_i == args.steps - 1 else clean
            step()
        ev1.record()
        torch.cuda.synchronize()
    if comm is not None:
        comm.barrier()
    ms = ev0.elapsed_time(ev1)
    if comm is not None:
        ms = comm.max_scalar(ms)
    iters = M * args.steps
    global_rate = iters / (ms / 1e3)       # Arnoldi iterations/s of the (global) solve
    # weak scaling: one global iteration = N slab iterations (16.7M rows each)
    value = global_rate if args.strong else global_rate * world
    # per-kernel device times: events around each launch in the timed region
    # (graph: the event nodes hold the last timed replay -- every replay runs
    # the identical 50-iteration cycle -- so one cycle's times x steps)
    agg = {}
    entries, rep_steps = (timers[captured[0]:captured[1]], args.steps) if captured else (timers, 1)
    for name, p, e0, e1 in entries:
        t = e0.elapsed_time(e1)
        a = agg.setdefault(name, [0.0, 0, 0])
        a[0] += t * rep_steps
        a[1] += rep_steps
        a[2] += _ortho_bytes(n, p, name) * rep_steps
    peak, peak_kind = _peaks()
    kern = {}
    for name, (t, cnt, byt) in agg.items():
        kern[name] = {"ms_total": t, "launches": cnt, "ms_avg": t / cnt,
                      "GBps": (byt / (t / 1e3) / 1e9) if byt and t > 0 else None}
    ortho = [k for k in ("lagged_reduce", "lagged_reduce_spmv", "lagged_update") if k in agg]
    dom = max(ortho, key=lambda k: agg[k][0])
    t_dom, c_dom, b_dom = agg[dom]
    achieved = b_dom / (t_dom / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        traffic = tr.get(dom)
    except Exception:
        pass
    ortho_t = sum(agg[k][0] for k in ortho)
    ortho_b = sum(agg[k][2] for k in ortho)
    cfg_json = _config(world, slab, args.strong)
    cfg_json["n_per_gpu"] = n
    if comm is not None:
        cfg_json["exchange"] = comm_kind
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg_json,
        "global_it_per_s": global_rate,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                     "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "bytes_per_launch_avg": b_dom / c_dom,
                     "ortho_GBps": ortho_b / (ortho_t / 1e3) / 1e9,
                     "ortho_frac": ortho_b / (ortho_t / 1e3) / 1e9 / peak},
        "kernels": kern,
        "gpu_launches": eng.launches_per_cycle * args.steps,   # every liblsb200 launch timed
        "clocks": clk.summary(),
    }
    if (nx, ny, nz) == (512, 512, 512) and world > 1:
        # config 4 as north_star states it: the same 512^3 solve on one B200
        # ran 104.6 it/s (profiles/r1_c4_512cube_single_gpu.txt)
        result["c4_vs_one_gpu_512cube"] = {
            "one_gpu_it_per_s": C4_ONE_GPU, "source": "profiles/r1_c4_512cube_single_gpu.txt",
            "speedup": global_rate / C4_ONE_GPU,
            "parallel_efficiency": global_rate / (world * C4_ONE_GPU)}
    del eng
    if comm_kind != "peer-threads":   # (device-wide sync: other in-process ranks may spin)
        torch.cuda.empty_cache()
    # e2e through the public API with host buffers: solve() on one GPU,
    # solve_distributed() per rank (each rank uploads its b rows, downloads x)
    cfg = P.GmresConfig(restart_m=M, max_restarts=1, rel_tol=1e-14, method="one_sync_mgs")
    # the step's input from pinned host memory (a numpy view of a page-locked
    # buffer, as a serving process would keep its request buffers)
    b_pin = torch.empty(len(b_local), dtype=torch.float64).pin_memory()
    b_host = b_pin.numpy()
    b_host[:] = b_local

    def e2e_once():
        if comm is None:
            x, h = P.solve(A_local, b_host, config=cfg, diagnostics_every=0)
        else:
            x, h = P.gmres.solve_distributed(A_local, b_host, comm, n_global, config=cfg)
        assert h.iterations == M and isinstance(x, np.ndarray)
        h.release()

    # two untimed calls: the first builds the solver engine, the second
    # captures its cycle graph (one-time costs of a (operator, config) that
    # every later call on the same operator reuses -- gmres._ENGINE_CACHE)
    e2e_once()
    e2e_once()
    torch.cuda.synchronize()
    if comm is not None:
        comm.barrier()
    t0 = time.perf_counter()
    e2e_steps = max(2, min(args.steps, 5))
    for _ in range(e2e_steps):
        e2e_once()
    dt = time.perf_counter() - t0
    if comm is not None:
        dt = comm.max_scalar(dt)
    result["e2e"] = {"value": M * e2e_steps / dt * (1 if args.strong else world), "unit": UNIT,
                     "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                     "steps": e2e_steps,
                     "what": "solve(A, b_host) -> x_host (per rank: solve_distributed), "
                             "b_host a numpy view of pinned host memory, x_host a fresh numpy "
                             "array; GmresConfig(50, 1 cycle); bytes per rank; after 2 untimed calls "
                             "(engine build, cycle-graph capture: reused by every later call "
                             "on the same operator)"}
    if world == 1 and not args.no_cpu and rank == 0 and not args.strong:
        secs, thr = cpu_windows(args.cpu_windows)
        v = PER_WINDOW * len(secs) / sum(secs)
        result["cpu_baseline"] = {
            "value": v, "unit": UNIT, "cores": thr, "kind": "port",
            "sample": f"iterations {PREFIX + 1}..{PREFIX + PER_WINDOW * len(secs)} (after "
                      f"{PREFIX} untimed) of the same 256^3 one-sync GMRES(50) solve, numpy "
                      f"oracle port ({sum(secs):.1f} s timed)"}
    return result


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-windows", type=int, default=4,
                    help="cpu_baseline: windows of 3 iterations after the 23-iteration prefix")
    ap.add_argument("--strong", action="store_true",
                    help="config 4 as stated: the 512^3 solve split over N GPUs (strong scaling)")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="validation only: run the N rank processes on GPU 0 (gloo host comm, "
                         "CUDA IPC peer exchange); not a scaling result")
    ap.add_argument("--comm", default="peer", choices=["peer", "nccl"],
                    help="N > 1: exchange transport (peer-memory kernels, or NCCL collectives)")
    ap.add_argument("--slab", type=int, default=N_SLAB, help="per-GPU cube edge (256 = config 2)")
    ap.add_argument("--kernel-timers", default="last", choices=["last", "all"],
                    help="per-kernel CUDA events in the last timed cycle only, or in every one")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="run the multi-rank path as K threads on one GPU (validation only)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.emulate_ranks > 1:
        # in-process ranks spin on each other's exchanges: one hardware queue
        # per rank stream (read at CUDA init; see parallel.run_threads)
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ \
            and args.emulate_ranks <= 1:
        _reexec_torchrun(args)
    if args.impl == "reference":
        if args.strong:
            print(json.dumps({"impl": "reference", "unavailable":
                              "--strong (512^3) exceeds a bounded CPU sample; use the default "
                              "weak-scaling arm"}), flush=True)
            return
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
