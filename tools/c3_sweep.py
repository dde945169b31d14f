"""Config C3: orthogonalization-only sweep, n = 2^20 .. 2^27,
k = 10, 20, 50, 100.  At each (n, k), p = k, one "step" is the per-column
kernel sequence of a variant, replayed as a CUDA graph as the engine runs its
cycles (`--eager`: launched from the host, round 1's protocol):

  one_sync  K1 lagged_reduce -> K5 mgs_lvl2_small -> K2 lagged_update
            (algorithmic 8n(2p+4))
  two_sync  K1 -> K5a -> K3 lagged_update_reduce -> K5b -> K4 lagged_correct
            (8n(3p+6); unfused K2 + K1' when p + 1 > 110)
  mgs_l1    p+1 fused K8 axpy+dot passes (one cooperative launch, grid
            barriers between passes) -> norm -> K5d -> scale
            (8n(4p+3))

V (cap k+2, Fortran-like column store) is filled from default_rng(0)-style
normals (torch generator seed 0) with unit columns, w from seed 1.  L2 is
flushed before every timed rep by READING a 256 MB buffer, so the step starts
with none of its data in L2 and no dirty lines to write back (round 1 wrote
the buffer instead: up to 126 MB of dirty-line write-back then landed inside
the timed step, ~15-30 us at n <= 2^22; `--dirty-flush` restores that).  Each
rep is bracketed by CUDA events on the launching stream.  Output: one JSON
object per line.

    python tools/c3_sweep.py [--ns 20,21,...,27] [--ks 10,20,50,100] [--reps 5]
"""

import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1809_05805_b200 import _abi  # noqa: E402
from paper_1809_05805_b200 import _dev as D  # noqa: E402

PEAK = 6551.4e9


def build(n, k):
    cap = k + 2
    ld = D.round_up(n, 32)
    dev = "cuda"
    f = dict(dtype=torch.float64, device=dev)
    V = torch.empty((cap, ld), **f)
    g = torch.Generator(device=dev).manual_seed(0)
    for j in range(cap):
        V[j, :n].normal_(generator=g)
        V[j, :n] /= torch.linalg.norm(V[j, :n])
    g1 = torch.Generator(device=dev).manual_seed(1)
    V[k, :n].normal_(generator=g1)
    st = dict(R=torch.zeros(cap * cap, **f), T=torch.zeros(cap * cap, **f),
              L=torch.zeros(cap * cap, **f), rot=torch.zeros(2 * cap, **f),
              g=torch.zeros(cap + 1, **f), tri=torch.zeros((cap + 1) * cap, **f),
              coef=torch.zeros(cap, **f), coef2=torch.zeros(cap, **f),
              G=torch.zeros(2 * cap + 4, **f), scal=torch.zeros(_abi.S_COUNT, **f),
              res=torch.zeros(cap + 1, **f),
              flags=torch.tensor([_abi.NO_STOP, 0, -1, 0, 0, 0, 0, 0], dtype=torch.int32,
                                 device=dev))
    st["scal"][_abi.S_BTF] = 1.0
    ws = D.Workspace(cap + 2)
    S = _abi.Arnoldi(V=V.data_ptr(), ld=ld, n=n, n_global=n, cap=cap, m=cap - 1,
                     R=st["R"].data_ptr(), T=st["T"].data_ptr(), L=st["L"].data_ptr(),
                     rot=st["rot"].data_ptr(), g=st["g"].data_ptr(), tri=st["tri"].data_ptr(),
                     coef=st["coef"].data_ptr(), coef2=st["coef2"].data_ptr(),
                     G=st["G"].data_ptr(), g_parts=1, g_stride=2 * cap, Gloc=st["G"].data_ptr(),
                     scal=st["scal"].data_ptr(), res=st["res"].data_ptr(),
                     flags=st["flags"].data_ptr(), ws=ws.c)
    return V, st, ws, S, ld


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="20,21,22,23,24,25,26,27")
    ap.add_argument("--ks", default="10,20,50,100")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="one_sync,two_sync,mgs_l1")
    ap.add_argument("--dirty-flush", action="store_true",
                    help="round-1 flush: write the 256 MB buffer, leaving L2 full of dirty "
                         "lines whose write-back lands inside the timed step")
    ap.add_argument("--eager", action="store_true",
                    help="issue each step's launches from the host (default: replay the "
                         "step as a CUDA graph, as the engine runs its cycles)")
    a = ap.parse_args()
    lib = _abi.load()
    cur = {"s": D.stream()}
    flush = torch.ones(1 << 25, dtype=torch.float64, device="cuda")   # 256 MB > L2
    sink = torch.empty((), dtype=torch.float64, device="cuda")

    def call(name, *args):
        _abi.check(getattr(lib, name)(*args), name)

    for e in [int(x) for x in a.ns.split(",")]:
        n = 1 << e
        for k in [int(x) for x in a.ks.split(",")]:
            V, st, ws, S, ld = build(n, k)
            ref = C.byref(S)
            p = k
            col = lambda j: C.c_void_p(V.data_ptr() + 8 * j * ld)  # noqa: E731

            def one_sync():
                stream = cur["s"]
                call("lsb_lagged_reduce", ref, 0, p, stream)
                call("lsb_mgs_lvl2_small", ref, 0, p, 1, 0, stream)
                call("lsb_lagged_update", ref, 0, p, 1, stream)

            def two_sync():
                stream = cur["s"]
                call("lsb_lagged_reduce", ref, 0, p, stream)
                call("lsb_cgs2_lvl2_small_a", ref, 0, p, 1, 0, stream)
                if p + 1 <= 110:
                    call("lsb_lagged_update_reduce", ref, 0, p, 1, stream)
                else:
                    call("lsb_lagged_update", ref, 0, p, 1, stream)
                    call("lsb_mdot", col(0), ld, n, p, col(p), None, D.ptr(st["G"]), ws.ref(),
                         None, -1, stream)
                call("lsb_cgs2_lvl2_small_b", ref, 0, p, stream)
                call("lsb_lagged_correct", ref, 0, p, stream)

            def mgs_l1():
                stream = cur["s"]
                call("lsb_mgs1_passes", ref, 0, p, p, stream)
                call("lsb_norm_finish", D.ptr(st["G"]), 1, 2 * (p + 2), col(p), n,
                     C.c_void_p(st["scal"].data_ptr() + 8 * _abi.S_BETA), ws.ref(), None, -1,
                     stream)
                call("lsb_direct_small", ref, 0, p, p, stream)
                call("lsb_direct_normalize", ref, 0, p, stream)

            byts = {"one_sync": 8 * n * (2 * p + 4), "two_sync": 8 * n * (3 * p + 6),
                    "mgs_l1": 8 * n * (4 * p + 3)}
            fns = {"one_sync": one_sync, "two_sync": two_sync, "mgs_l1": mgs_l1}
            for var in a.variants.split(","):
                fn = fns[var]
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                if not a.eager:
                    g = torch.cuda.CUDAGraph()
                    side = torch.cuda.Stream()
                    with torch.cuda.graph(g, stream=side):
                        cur["s"] = C.c_void_p(side.cuda_stream)
                        fn()
                    cur["s"] = D.stream()
                    g.replay()
                    torch.cuda.synchronize()
                    fn = g.replay
                tot = 0.0
                for _ in range(a.reps):
                    if a.dirty_flush:
                        flush.fill_(1.0)
                    else:
                        torch.sum(flush, dim=0, out=sink)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    fn()
                    e1.record()
                    torch.cuda.synchronize()
                    tot += e0.elapsed_time(e1)
                ms = tot / a.reps
                gbs = byts[var] / (ms / 1e3) / 1e9
                print(json.dumps({"n": n, "k": k, "variant": var, "graph": not a.eager,
                                  "flush": "write" if a.dirty_flush else "read",
                                  "ms": round(ms, 4),
                                  "alg_GBps": round(gbs, 1), "frac": round(gbs * 1e9 / PEAK, 3),
                                  "fits_L2": n * (k + 2) * 8 <= 126 * 2 ** 20}), flush=True)
            del V, st, ws, S
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
