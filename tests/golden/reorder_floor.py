"""Reference reorder-sensitivity floor (hard part 2).

Reruns the oracle (same algorithm and arithmetic as the reference) with only
the summation order of its reductions changed -- every inner product of
mdot_pair / mass_inner_product / dot summed in 148 row blocks (one per B200
SM) instead of one OpenBLAS call -- and reports the max relative deviation
of the implicit-residual curve from the reference's golden curve.  That is
how far the reference itself moves under a legitimate reordering; the GPU
parity tests use max(1e-10, 4x this floor).  Output: reorder_floor.json.

    python tests/golden/reorder_floor.py
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import lowsync_oracle as orc  # noqa: E402

NB = 148


def _blocked_T(X, y):
    n = X.shape[0]
    s = (n + NB - 1) // NB
    out = np.zeros(X.shape[1])
    for i in range(0, n, s):
        out += X[i:i + s].T @ y[i:i + s]
    return out


def mdot_pair(X, u, w, led, kind=orc.K_MDOT, eligible=False):
    p = X.shape[1]
    if p == 0:
        return np.zeros((0, 2))
    led.add(kind, 2 * p, eligible)
    return np.stack([_blocked_T(X, u), _blocked_T(X, w)], axis=1)


def mass_ip(X, y, led, eligible=False):
    p = X.shape[1]
    if p == 0:
        return np.zeros(0)
    led.add(orc.K_MDOT, p, eligible)
    return _blocked_T(X, y)


def dot(x, y, led):
    led.add(orc.K_DOT, 1)
    return float(_blocked_T(x[:, None], y)[0])


def main(N=64):
    orc.mdot_pair, orc.mass_ip, orc.dot = mdot_pair, mass_ip, dot
    G = np.load(os.path.join(HERE, f"convdiff27_{N}.npz"))
    A = orc.convdiff27(N)
    b = orc.rhs_random(A.n_rows, 42)
    out = {}
    for meth in ("one_sync_mgs", "two_sync_cgs2", "mgs_l1"):
        r = orc.gmres(A, b, meth, 100, 30, 1e-10)
        c, cr = np.array(r.curve), G[meth + "__curve"]
        n = min(len(c), len(cr))
        out[meth] = float(np.max(np.abs(c[:n] - cr[:n]) / cr[:n]))
        print(meth, len(c), len(cr), out[meth], flush=True)
    path = os.path.join(HERE, "reorder_floor.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data["_what"] = ("max relative per-iteration deviation of the reference algorithm's own "
                     "implicit-residual curve when only the summation order of its reductions "
                     "changes (148 row blocks), vs the golden run; tests/golden/reorder_floor.py")
    data[f"convdiff27_{N}"] = out
    with open(path, "w") as fh:
        json.dump(data, fh, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 64)
