"""Small-n (C3 latency-bound cells) kernel probe: cold-L2 device time of K1,
K5 and K2 of the one-sync step at n = 2^20..2^22, per grid / part / row-CTA
override, to see where a 60 us step goes.

    python tools/ksmall.py [--ns 20,21,22] [--ps 10,50] [--reps 10]
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

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from c3_sweep import build  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="20,21,22")
    ap.add_argument("--ps", default="10,50")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    lib = _abi.load()
    flush = torch.ones(1 << 25, dtype=torch.float64, device="cuda")
    sink = torch.empty((), dtype=torch.float64, device="cuda")
    dirty = {"on": False}

    def call(name, *args):
        _abi.check(getattr(lib, name)(*args), name)

    def cold(fn, pre=None):
        tot = 0.0
        for _ in range(a.reps):
            if pre:
                pre()
            if dirty["on"]:
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
        return round(1e3 * tot / a.reps, 2)

    for e in [int(x) for x in a.ns.split(",")]:
        n = 1 << e
        for p in [int(x) for x in a.ps.split(",")]:
            V, st, ws, S, ld = build(n, p)
            ref = C.byref(S)
            s = D.stream()
            k1 = lambda: call("lsb_lagged_reduce", ref, 0, p, s)  # noqa: E731
            k5 = lambda: call("lsb_mgs_lvl2_small", ref, 0, p, 1, 0, s)  # noqa: E731
            k2 = lambda: call("lsb_lagged_update", ref, 0, p, 1, s)  # noqa: E731
            for f in (k1, k5, k2):
                f()
            torch.cuda.synchronize()
            out = {"n": e, "p": p, "K1": cold(k1), "K5": cold(k5, k1), "K2": cold(k2),
                   "step": cold(lambda: (k1(), k5(), k2()))}
            bytes1 = 8 * n * (p + 2)
            out["K1_TBps"] = round(bytes1 / out["K1"] / 1e6, 2)
            dirty["on"] = True
            out["K1_dirty"], out["K2_dirty"] = cold(k1), cold(k2)
            dirty["on"] = False
            for g in (148, 296, 444, 592, 888):
                ws.c.grid = g
                out[f"K1_g{g}"] = cold(k1)
            ws.c.grid = 0
            for r in (1, 2, 4):
                lib.lsb_set_tuning(_abi.TUNE_FORCE_PARTS, r)
                out[f"K1_R{r}"] = cold(k1)
            lib.lsb_set_tuning(_abi.TUNE_FORCE_PARTS, 0)
            for r in (1, 2, 3, 4):
                lib.lsb_set_tuning(_abi.TUNE_ROW_CTAS_PER_SM, r)
                out[f"K2_c{r}"] = cold(k2)
            lib.lsb_set_tuning(_abi.TUNE_ROW_CTAS_PER_SM, 0)
            # launch floor: an empty-ish step at the same grid (p = 1, n = 1024)
            print(json.dumps(out), flush=True)
            del V, st, ws, S
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
