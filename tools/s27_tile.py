"""27-point SpMV kernels side by side: the TMA plane-tile kernel (default
from 2^21 rows; forced with knob 5),
the z-march and the row-pair kernel -- bitwise check on ragged shapes and
slabs with ghost planes, then 256^3 timings (16n algorithmic bytes).

    python tools/s27_tile.py [--N 256] [--reps 20]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1809_05805_b200 import _abi  # noqa: E402
from paper_1809_05805_b200.operators import StencilMatrix, StencilOperator, convdiff27  # noqa: E402

MODES = {"auto": 0, "tile": 5, "pair": 2, "march_generic": 3, "march": 4}


def apply_all(op, xs, n, modes, b=None, zcs=(0,)):
    lib = _abi.load()
    outs = {}
    for name in modes:
        for zc in (zcs if name == "tile" else (0,)):
            lib.lsb_set_tuning(_abi.TUNE_S27_MARCH, MODES[name])
            lib.lsb_set_tuning(_abi.TUNE_S27_TILE_Z, zc)
            y = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
            op.apply(xs, y, b=b)
            outs[(name, zc)] = y.cpu().numpy()
    lib.lsb_set_tuning(_abi.TUNE_S27_MARCH, 0)
    lib.lsb_set_tuning(_abi.TUNE_S27_TILE_Z, 0)
    return outs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--skip-bitwise", action="store_true")
    ap.add_argument("--only", default="", help="comma list of timing cases, e.g. tile16,march")
    a = ap.parse_args()
    lib = _abi.load()
    rng = np.random.default_rng(3)
    res = {"bitwise": []}
    offs_rand = [((o % 3 - 1, (o // 3) % 3 - 1, o // 9 - 1), float(rng.standard_normal()))
                 for o in range(27)]
    for dims in [] if a.skip_bitwise else [(12, 10, 70), (34, 18, 33), (64, 48, 40), (6, 4, 5), (32, 16, 32), (66, 17, 97)]:
        for kind in ("convdiff", "random"):
            S = convdiff27(0, dims=dims) if kind == "convdiff" else StencilMatrix(dims, offs_rand, "r27")
            for halo in [(0, 0), (1, 1), (1, 0)]:
                nx, ny, nz = dims
                plane = nx * ny
                z0 = 1 if halo[0] else 0
                nzl = nz - z0 - (1 if halo[1] else 0)
                op = StencilOperator(S, z0=z0, nz_local=nzl)
                n = plane * nzl
                xpad = torch.as_tensor(rng.standard_normal(n + 2 * plane + 2)).cuda()
                xs = xpad[plane:plane + n]
                bb = torch.as_tensor(rng.standard_normal(n)).cuda() if halo == (1, 0) else None
                outs = apply_all(op, xs, n, ["tile", "pair", "march", "auto"], b=bb, zcs=(0, 7, 16))
                ref = outs[("pair", 0)]
                ok = all(np.array_equal(v, ref) for v in outs.values())
                res["bitwise"].append({"dims": dims, "kind": kind, "halo": halo, "ok": ok})
                print(dims, kind, halo, "bitwise" if ok else "MISMATCH", flush=True)
    S = convdiff27(a.N)
    n = S.n_rows
    op = StencilOperator(S)
    x = torch.as_tensor(np.random.default_rng(1).standard_normal(n)).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        "MEASURED_PEAKS.json") else 6551.4
    res["timing"] = {}
    cases = [("auto", 0), ("tile", 0), ("tile", 16), ("tile", 32), ("tile", 64), ("tile", 128), ("march", 0), ("pair", 0)]
    if a.only:
        cases = [c for c in cases if f"{c[0]}{c[1] or ''}" in a.only.split(",")]
    for name, zc in cases:
        lib.lsb_set_tuning(_abi.TUNE_S27_MARCH, MODES[name])
        lib.lsb_set_tuning(_abi.TUNE_S27_TILE_Z, zc)
        for _ in range(3):
            op.apply(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            op.apply(x, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        gbs = 16 * n / ms / 1e6
        res["timing"][f"{name}{zc or ''}"] = {"ms": ms, "GBps": gbs, "frac": gbs / pk}
        print(f"{name} zc={zc}: {ms:.4f} ms  {gbs:.0f} GB/s  frac {gbs / pk:.3f}", flush=True)
    lib.lsb_set_tuning(_abi.TUNE_S27_MARCH, 0)
    lib.lsb_set_tuning(_abi.TUNE_S27_TILE_Z, 0)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/s27_tile.json", "w"), indent=1, default=str)


if __name__ == "__main__":
    main()
