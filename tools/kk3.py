"""K3 (lsb_lagged_update_reduce) against the unfused K2 + K1' pair at
n = 256^3: average launch time and algorithmic GB/s (8n(p+3) for K3;
8n(p+3) + 8n(p+1) for the pair).

    python tools/kk3.py [--ps 2,10,26,51,101] [--reps 20]
"""

import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1809_05805_b200 import _abi  # noqa: E402
from paper_1809_05805_b200 import _dev as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ps", default="2,10,26,51,101")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--rows", default="0", help="LSB_TUNE_K3_ROWS values to sweep (0 = auto)")
    ap.add_argument("--stages", default="0", help="LSB_TUNE_K3_STAGES values to sweep (0 = auto)")
    a = ap.parse_args()
    lib, st = _abi.load(), D.stream()
    n = a.n
    ld = D.round_up(n, 32)
    for p in [int(x) for x in a.ps.split(",")]:
        cap = p + 2
        V = torch.randn((cap, ld), device="cuda", dtype=torch.float64)
        coef = torch.randn(cap, device="cuda", dtype=torch.float64) * 1e-3
        scal = torch.zeros(_abi.S_COUNT, dtype=torch.float64, device="cuda")
        scal[_abi.S_BETA] = 1.0
        flags = torch.tensor([_abi.NO_STOP, 0, -1, 0, 0, 0, 0, 0], dtype=torch.int32,
                             device="cuda")
        Gloc = torch.zeros(2 * cap, dtype=torch.float64, device="cuda")
        ws = D.Workspace(cap)
        z = torch.zeros(cap * cap, dtype=torch.float64, device="cuda")
        S = _abi.Arnoldi(V=V.data_ptr(), ld=ld, n=n, n_global=n, cap=cap, m=cap - 2,
                         R=z.data_ptr(), T=z.data_ptr(), L=z.data_ptr(), rot=z.data_ptr(),
                         g=z.data_ptr(), tri=z.data_ptr(), coef=coef.data_ptr(),
                         coef2=z.data_ptr(), G=Gloc.data_ptr(), g_parts=1, g_stride=2 * cap,
                         Gloc=Gloc.data_ptr(), scal=scal.data_ptr(), res=z.data_ptr(),
                         flags=flags.data_ptr(), ws=ws.c)
        ref = C.byref(S)

        def k3():
            _abi.check(lib.lsb_lagged_update_reduce(ref, 0, p, 1, st), "k3")

        def pair():
            _abi.check(lib.lsb_lagged_update(ref, 0, p, 1, st), "k2")
            _abi.check(lib.lsb_mdot(C.c_void_p(V.data_ptr()), ld, n, p,
                                    C.c_void_p(V.data_ptr() + 8 * p * ld), None,
                                    C.c_void_p(Gloc.data_ptr()), ws.ref(), None, -1, st), "k1")

        res = {}
        arms = [(f"k3/{r}/{s}", k3, 8 * n * (p + 3), int(r), int(s))
                for r in a.rows.split(",") for s in a.stages.split(",")]
        arms.append(("pair", pair, 8 * n * (p + 3) + 8 * n * (p + 1), 0, 0))
        for name, fn, byt, rows, stages in arms:
            lib.lsb_set_tuning(4, rows)
            lib.lsb_set_tuning(5, stages)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            res[name] = (ms, byt / ms / 1e6)
        print(f"p={p:4d}  " + "  ".join(f"{k} {v[0]:.3f} ms {v[1]:5.0f} GB/s" for k, v in res.items()),
              flush=True)
        del V, S
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
