"""Config 5 throughput: 27-point convection-diffusion at N^3 (default 256^3,
n = 16.7M, 450M nonzeros), one-sync GMRES(100), in stencil (K6) and CSR (K7)
form.  Times the SpMV kernels alone (algorithmic bytes: 16n stencil,
12*nnz + 4(n+1) + 16n CSR, x read once) and whole graph-replayed cycles
against the cycle's HBM ceiling.  The CSR is built on the device
(StencilMatrix.device_csr); its y is checked bitwise against the stencil's.

    python tools/c5_rates.py [--N 256] [--m 100] [--cycles 2]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_05805_b200 as P  # noqa: E402
from paper_1809_05805_b200 import _abi  # noqa: E402
from paper_1809_05805_b200.engine import Engine  # noqa: E402
from paper_1809_05805_b200.operators import convdiff27, laplace3d  # noqa: E402


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]) * 1e9
    except Exception:
        return 6551.4e9


def time_spmv(op, x, y, reps=20):
    for _ in range(3):
        op.apply(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        op.apply(x, y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--m", type=int, default=100)
    ap.add_argument("--cycles", type=int, default=2)
    ap.add_argument("--no-cycles", action="store_true")
    a = ap.parse_args()
    PK = peak()
    lib = _abi.load()
    S = convdiff27(a.N)
    n = S.n_rows
    out = {"N": a.N, "n": n, "nnz": S.nnz, "peak_GBps": PK / 1e9}
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y0 = torch.empty_like(x)
    y1 = torch.empty_like(x)
    st = S.device_op()
    csr = S.device_csr()
    assert csr.values.shape[0] == S.nnz
    sp = {}
    ms = time_spmv(st, x, y0)
    sp["stencil27"] = {"ms": ms, "GBps": 16 * n / ms / 1e6}
    csr_bytes = 12 * S.nnz + 4 * (n + 1) + 16 * n
    dict_bytes = 2 * S.nnz + 4 * (n + 1) + 16 * n
    plain = csr.with_scale(None)
    plain.cd = None                      # the 12-byte-per-nonzero kernels
    if csr.cd is not None:
        for key, knob in (("csr_dict", 0), ("csr_dict_warp_staged", 1)):
            lib.lsb_set_tuning(_abi.TUNE_CSR_DICT, knob)
            ms = time_spmv(csr, x, y1)
            sp[key] = {"ms": ms, "GBps": dict_bytes / ms / 1e6,
                       "bitwise_eq_stencil": bool(torch.equal(y0, y1)),
                       "tables": [int(csr.cd.n_val), int(csr.cd.n_off)]}
        lib.lsb_set_tuning(_abi.TUNE_CSR_DICT, 0)
    for key, knob in (("csr_warp_u16", 0), ("csr_warp_u8_occ3", 2), ("csr_thread_row", 1)):
        lib.lsb_set_tuning(_abi.TUNE_CSR_THREAD_ROW, knob)
        ms = time_spmv(plain, x, y1)
        eq = bool(torch.equal(y0, y1))
        sp[key] = {"ms": ms, "GBps": csr_bytes / ms / 1e6, "bitwise_eq_stencil": eq}
    lib.lsb_set_tuning(_abi.TUNE_CSR_THREAD_ROW, 0)
    L = laplace3d(a.N).device_op()
    ms = time_spmv(L, x, y0)
    sp["stencil7_pair"] = {"ms": ms, "GBps": 16 * n / ms / 1e6}
    for k, v in sp.items():
        v["frac"] = v["GBps"] * 1e9 / PK
        print(k, {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()},
              flush=True)
    out["spmv"] = sp
    if not a.no_cycles:
        b = np.random.default_rng(42).standard_normal(n)
        b /= np.linalg.norm(b)
        bd = torch.as_tensor(b).cuda()
        ortho = sum(8 * n * (2 * (i + 1) + 4) for i in range(1, a.m + 1))
        cyc = {}
        forms = [("stencil", st, 16 * n), ("csr", plain, csr_bytes)]
        if csr.cd is not None:
            forms.append(("csr_dict", csr, dict_bytes))
        for form, op, sbytes in forms:
            eng = Engine(S, a.m, "one_sync_mgs", 1e-14, op=op, use_graph=True)
            eng.load(bd)
            eng.prologue()
            eng.cycle()
            eng.cycle()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.cycles):
                eng.cycle()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.cycles
            ceil = (ortho + a.m * sbytes) / PK * 1e3
            cyc[form] = {"ms_per_cycle": round(ms, 2), "it_s": round(a.m * 1e3 / ms, 1),
                         "hbm_ceiling_ms": round(ceil, 2), "frac": round(ceil / ms, 3)}
            print(form, cyc[form], flush=True)
            del eng
            torch.cuda.empty_cache()
        out["cycles"] = cyc
    print(json.dumps(out))


if __name__ == "__main__":
    main()
